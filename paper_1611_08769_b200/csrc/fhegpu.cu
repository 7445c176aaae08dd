// fhegpu.cu -- C ABI of the B200 engine (declared in include/fhegpu.h).
//
// Owns: the device ciphertext store, the context stream, levelised programs
// (op tables resident in HBM) and the kernel dispatch (tcgen05 kernel for the
// parameter sets it is instantiated for, CUDA-core kernel otherwise).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fhegpu.h"
#include "common.cuh"
#include "simt_nand.cuh"
#include "tc_nand.cuh"
#include "tc_nand_ws.cuh"
#include "tc_nand_resident.cuh"
#include "tc_nand_regfile.cuh"
#include "flow_nand.cuh"
#include "encrypt.cuh"
#include "bits.cuh"

using namespace fhegpu;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return fail(FHEGPU_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
  } while (0)

constexpr size_t kStagingCap = size_t(256) << 20;  // bytes per staged transfer chunk
constexpr int kStreamRegions = 3;                  // store regions rotated by fhegpu_prog_run_host

}  // namespace

struct fhegpu_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  DevParams p{};
  uint32_t n = 0, m = 0;
  int kernel_pref = FHEGPU_KERNEL_AUTO;
  bool tc_capable = false;  // sm_100 device and a kernel instantiated for (k, ell)
  int num_sms = 0;
  uint32_t *store = nullptr;
  uint64_t capacity = 0;  // ciphertexts
  uint64_t store_gen = 0; // bumped whenever the store moves (captured graphs bake its address)
  // staging
  uint32_t *d_stage = nullptr;
  size_t stage_bytes = 0;
  uint64_t *d_idx = nullptr;
  size_t idx_cap = 0;
  uint8_t *d_comp = nullptr;
  size_t comp_cap = 0;
  uint32_t *d_copy = nullptr;  // slot pairs of fhegpu_store_copy_slots (only written stream-ordered)
  size_t copy_cap = 0;
  OpRec *d_tmp_ops = nullptr;
  size_t tmp_ops_cap = 0;
  JumpTable *d_jump = nullptr;  // PCG64 jump-ahead constants (lazily uploaded)
  bool use_graphs = true;       // replay whole programs as CUDA graphs
  // host streaming (fhegpu_prog_run_host): copy-in / copy-out streams + per-region events
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_in[kStreamRegions] = {}, ev_done[kStreamRegions] = {}, ev_free[kStreamRegions] = {};
  uint32_t *d_hstage = nullptr;  // dense staging rows for contiguous host copies
  size_t hstage_bytes = 0;
};

struct fhegpu_prog {
  OpRec *d_ops = nullptr;
  std::vector<uint64_t> offsets;  // n_levels + 1
  uint64_t n_ops = 0;
  uint64_t n_slots = 0;           // 1 + the largest slot any op names
  int2 *d_deps = nullptr;         // dataflow mode: producing op of each operand (-1: ready)
  bool levels_valid = true;       // level launches are a valid fallback (no op depends on an op
                                  // of its own level); false for tiled programs
  uint32_t *d_progress = nullptr; // per-CTA completed-item counters
  // ready-queue launches (fhegpu_prog_set_queue): per-op pending counts, consumer lists, roots
  std::vector<int32_t> deps_host;
  bool use_queue = false;
  uint32_t *d_qmeta = nullptr;    // pend0[n_ops] | cons_off[n_ops + 1] | cons[n_edges] | roots[n_roots]
  uint64_t n_edges = 0;
  uint32_t n_roots = 0;
  uint32_t *d_qrun = nullptr;     // per run: counters[4] | pending[n_items] | queue[n_items]
  size_t qrun_cap = 0;
  // lane-resident launches (fhegpu_prog_set_resident): per-lane gate plan + program inputs
  bool use_resident = false;
  tc::ResOp *d_rplan = nullptr;
  uint32_t *d_rin = nullptr;
  uint32_t r_ops = 0, r_in = 0, r_local = 0, r_out = 0;
  uint64_t r_slots = 0;           // 1 + the largest store slot the plan reads or writes
  bool r_deps = true;             // the slot order has operands produced < 5 slots back
  // register-file launches (fhegpu_prog_set_regfile): per-lane slot table + fill list
  bool use_regfile = false;
  fhegpu_rf_slot *d_rfslots = nullptr;
  fhegpu_rf_fill *d_rffills = nullptr;
  uint32_t rf_ops = 0, rf_fills = 0, rf_buf = 0, rf_spill = 0;
  uint64_t rf_spill_base = 0;
  uint64_t rf_slots = 0;          // 1 + the largest store slot the plan reads or writes
  // warp-dataflow launches (fhegpu_prog_set_flow): per-worker gate lists + tagged scratch
  bool use_flow = false;
  uint4 *d_flow_ents = nullptr;
  uint32_t *d_flow_off = nullptr;
  uint4 *d_flow_scratch = nullptr;
  uint32_t flow_ctas = 0, flow_epoch = 0;
  double flow_makespan = 0;
  uint32_t flow_stats[4] = {0, 0, 0, 0};   // ring / scratch / store operands, max gates per worker
  // CUDA graph of one full run (all level launches), captured on first use per
  // (lanes, stream, kernel choice, debug bits); replayed with a single cudaGraphLaunch
  cudaGraphExec_t graph = nullptr;
  uint32_t graph_lanes = 0;
  cudaStream_t graph_stream = nullptr;
  int graph_kernel = -1;
  uint32_t graph_dbg = 0;
  uint64_t graph_store_gen = 0;
};

namespace {

int ensure(void **ptr, size_t *cap, size_t need) {
  if (*cap >= need) return FHEGPU_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  size_t sz = std::max(need, size_t(1) << 20);
  cudaError_t e = cudaMalloc(ptr, sz);
  if (e != cudaSuccess) return fail(FHEGPU_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  *cap = sz;
  return FHEGPU_OK;
}

bool tc_instantiated(uint32_t k, uint32_t ell) {
  return (k == 9 && ell == 29) || (k == 3 && ell == 17);
}

// Pseudo-Mersenne epilogue applies when the folded sum of finish_value stays < 2q.
bool pm_ok(uint32_t q, uint32_t ell) {
  if (ell < 17 || ell > 31) return false;
  const uint64_t c = (1ull << ell) - q;
  const uint64_t bh_max = ((1ull << 26) - 1) >> (ell - 16);
  const uint64_t t_max = ((1ull << 26) - 1) + (((1ull << (ell - 16)) - 1) << 16) + c * bh_max;
  return c * bh_max < (1ull << 32) && t_max < 2ull * q && t_max < (1ull << 32);
}

template <int K, int ELL, bool PM>
int launch_tc_impl(fhegpu_ctx *c, uint32_t *store, const OpRec *ops, uint32_t n_ops, uint32_t lanes) {
  using G = tc::Geo<K, ELL>;
  static bool attr_done = false;
  // 100 KB requested so at most two CTAs (2 x 256 TMEM columns) share an SM
  const int smem = std::max(G::SMEM, 100 * 1024);
  if (!attr_done) {
    CUDA_TRY(cudaFuncSetAttribute(tc::level_tc_kernel<K, ELL, PM>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_done = true;
  }
  const uint64_t items = (uint64_t)n_ops * lanes;
  const uint64_t grid = std::min<uint64_t>(items, (uint64_t)c->num_sms * 2);
  // programmatic dependent launch as for the warp-specialised kernel (dbg bit 13 disables)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(G::THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (c->p.dbg & 8192u) ? 0 : 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, tc::level_tc_kernel<K, ELL, PM>, store, ops, n_ops, lanes, c->p));
  return FHEGPU_OK;
}

template <int K, int ELL, bool PM, int ENC, bool Q = false>
int launch_tc_ws_enc(fhegpu_ctx *c, uint32_t *store, const OpRec *ops, uint32_t n_ops, uint32_t lanes,
                      const int2 *deps, uint32_t *progress, const tc::QueueArgs &qa = tc::QueueArgs{}) {
  using G = tc::GeoWS<K, ELL, PM, ENC, Q>;
  static bool attr_done = false;
  // > half of the SM's shared memory: exactly one CTA (512 TMEM columns) per SM
  const int smem = std::max(G::SMEM, 120 * 1024);
  if (!attr_done) {
    CUDA_TRY(cudaFuncSetAttribute(tc::level_tc_ws_kernel<K, ELL, PM, ENC, Q>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_done = true;
  }
  const uint64_t items = (uint64_t)n_ops * lanes;
  if (items >= (1ull << 32)) return fail(FHEGPU_EINVAL, "level too large (>= 2^32 gate items)");
  const uint64_t grid = std::min<uint64_t>(items, (uint64_t)c->num_sms);
  DevParams p = c->p;
  p.lanes_magic = (uint32_t)(0xFFFFFFFFu / lanes);
  // programmatic dependent launch (dbg bit 13 disables): consecutive levels overlap the
  // launch gap and prologue; the kernel's griddepcontrol.wait keeps the data dependence
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(G::THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (c->p.dbg & 8192u) ? 0 : 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, tc::level_tc_ws_kernel<K, ELL, PM, ENC, Q>, store, ops, n_ops, lanes, p,
                              deps, progress, qa));
  return FHEGPU_OK;
}

// Level launches and dataflow launches use different A encodings (tc_nand_ws.cuh, AEnc).
template <int K, int ELL, bool PM>
int launch_tc_ws_impl(fhegpu_ctx *c, uint32_t *store, const OpRec *ops, uint32_t n_ops, uint32_t lanes,
                      const int2 *deps = nullptr, uint32_t *progress = nullptr) {
  if (deps == nullptr)
    return launch_tc_ws_enc<K, ELL, PM, FHEGPU_ENC_LEVELS>(c, store, ops, n_ops, lanes, deps, progress);
  return launch_tc_ws_enc<K, ELL, PM, FHEGPU_ENC_FLOW>(c, store, ops, n_ops, lanes, deps, progress);
}

template <int K, int ELL>
int launch_tc(fhegpu_ctx *c, uint32_t *store, const OpRec *ops, uint32_t n_ops, uint32_t lanes) {
  if constexpr ((ELL + 7) / 8 == 4 && tc::Geo<K, ELL>::MT >= 1 &&
                tc::Geo<K, ELL>::D_COLS + tc::Geo<K, ELL>::A_COLS <= 256) {
    if (!(c->p.dbg & 4u)) {  // dbg bit 2 selects the two-CTA (v2) kernel
      if (pm_ok(c->p.q, c->p.ell) && !(c->p.dbg & 2u))
        return launch_tc_ws_impl<K, ELL, true>(c, store, ops, n_ops, lanes);
      return launch_tc_ws_impl<K, ELL, false>(c, store, ops, n_ops, lanes);
    }
  }
  if constexpr ((ELL + 7) / 8 == 4) {
    if (pm_ok(c->p.q, c->p.ell) && !(c->p.dbg & 2u))  // dbg bit 1 forces the generic epilogue
      return launch_tc_impl<K, ELL, true>(c, store, ops, n_ops, lanes);
  }
  return launch_tc_impl<K, ELL, false>(c, store, ops, n_ops, lanes);
}

int launch_simt(fhegpu_ctx *c, uint32_t *store, const OpRec *ops, uint32_t n_ops, uint32_t lanes) {
  const size_t smem = size_t(2) * c->p.words * sizeof(uint32_t);
  const uint64_t items = (uint64_t)n_ops * lanes;
  const uint64_t grid = std::min<uint64_t>(items, (uint64_t)c->num_sms * 8);
  if (c->p.k <= 4) {
    if (smem > 48 * 1024)
      CUDA_TRY(cudaFuncSetAttribute(level_simt_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    level_simt_kernel<4><<<(unsigned)grid, 256, smem, c->stream>>>(store, ops, n_ops, lanes, c->p);
  } else {
    if (smem > 48 * 1024)
      CUDA_TRY(cudaFuncSetAttribute(level_simt_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    level_simt_kernel<16><<<(unsigned)grid, 256, smem, c->stream>>>(store, ops, n_ops, lanes, c->p);
  }
  CUDA_TRY(cudaGetLastError());
  return FHEGPU_OK;
}

int effective_kernel(const fhegpu_ctx *c) {
  if (c->kernel_pref == FHEGPU_KERNEL_SIMT) return FHEGPU_KERNEL_SIMT;
  if (c->kernel_pref == FHEGPU_KERNEL_TCGEN05) return FHEGPU_KERNEL_TCGEN05;
  return c->tc_capable ? FHEGPU_KERNEL_TCGEN05 : FHEGPU_KERNEL_SIMT;
}

int launch_level(fhegpu_ctx *c, uint32_t *store, const OpRec *ops, uint32_t n_ops, uint32_t lanes) {
  if (n_ops == 0 || lanes == 0) return FHEGPU_OK;
  const int kern = effective_kernel(c);
  if (kern == FHEGPU_KERNEL_TCGEN05) {
    if (!c->tc_capable)
      return fail(FHEGPU_EUNSUP, "tcgen05 kernel requested but not available for this device/params");
    if (c->p.k == 9 && c->p.ell == 29) return launch_tc<9, 29>(c, store, ops, n_ops, lanes);
    if (c->p.k == 3 && c->p.ell == 17) return launch_tc<3, 17>(c, store, ops, n_ops, lanes);
    return fail(FHEGPU_EUNSUP, "no tcgen05 instantiation for these params");
  }
  return launch_simt(c, store, ops, n_ops, lanes);
}

// A whole program in one launch (dataflow over per-CTA progress counters); FHEGPU_EUNSUP when
// the parameter set / kernel choice has no warp-specialised tcgen05 kernel.
int launch_dataflow(fhegpu_ctx *c, uint32_t *store, const OpRec *ops, uint32_t n_ops, uint32_t lanes,
                    const int2 *deps, uint32_t *progress) {
  if (n_ops == 0 || lanes == 0) return FHEGPU_OK;
  if (effective_kernel(c) != FHEGPU_KERNEL_TCGEN05 || (c->p.dbg & 4u)) return FHEGPU_EUNSUP;
  if (!(c->p.k == 9 && c->p.ell == 29)) return FHEGPU_EUNSUP;
  if ((uint64_t)n_ops * lanes >= (1ull << 32) || c->num_sms > 256) return FHEGPU_EUNSUP;
  CUDA_TRY(cudaMemsetAsync(progress, 0, (size_t)c->num_sms * sizeof(uint32_t), c->stream));
  if (pm_ok(c->p.q, c->p.ell) && !(c->p.dbg & 2u))
    return launch_tc_ws_impl<9, 29, true>(c, store, ops, n_ops, lanes, deps, progress);
  return launch_tc_ws_impl<9, 29, false>(c, store, ops, n_ops, lanes, deps, progress);
}

unsigned grid_for(uint64_t work, int num_sms) {
  uint64_t g = (work + 255) / 256;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, (uint64_t)num_sms * 16));
}

// Ready-queue state before a run: every item's pending count from its op, the queue holding
// the root items (ops with no producer in the program) and EMPTY elsewhere, cursors reset.
__global__ void queue_init_kernel(uint32_t *counters, uint32_t *pending, uint32_t *queue, const uint32_t *pend0,
                                  const uint32_t *roots, uint32_t n_roots, uint32_t lanes, uint32_t n_items) {
  const uint32_t n_root_items = n_roots * lanes;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_items; i += gridDim.x * blockDim.x) {
    const uint32_t op = i / lanes, ln = i - op * lanes;
    pending[i] = pend0[op];
    queue[i] = i < n_root_items ? roots[op] * lanes + ln : tc::Q_EMPTY;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    counters[0] = 0u;
    counters[1] = n_root_items;
  }
}

#ifndef FHEGPU_ENC_QUEUE
#define FHEGPU_ENC_QUEUE 1     // A encoding of ready-queue launches (cfg2/cfg3: 1 is ~1% faster)
#endif

// A whole program in one launch over a ready queue (after queue_init_kernel).
int launch_queue(fhegpu_ctx *c, fhegpu_prog *pr, uint32_t lanes) {
  if (pr->n_ops == 0 || lanes == 0) return FHEGPU_OK;
  if (effective_kernel(c) != FHEGPU_KERNEL_TCGEN05 || (c->p.dbg & 4u)) return FHEGPU_EUNSUP;
  if (!(c->p.k == 9 && c->p.ell == 29)) return FHEGPU_EUNSUP;
  const uint64_t n_items = pr->n_ops * lanes;
  if (n_items >= (1ull << 31)) return FHEGPU_EUNSUP;
  if (int rc = ensure((void **)&pr->d_qrun, &pr->qrun_cap, (4 + 2 * n_items) * sizeof(uint32_t))) return rc;
  uint32_t *counters = pr->d_qrun, *pending = counters + 4, *queue = pending + n_items;
  const uint32_t *pend0 = pr->d_qmeta, *cons_off = pend0 + pr->n_ops, *cons = cons_off + pr->n_ops + 1;
  const uint32_t *roots = cons + pr->n_edges;
  queue_init_kernel<<<grid_for(n_items, c->num_sms), 256, 0, c->stream>>>(
      counters, pending, queue, pend0, roots, pr->n_roots, lanes, (uint32_t)n_items);
  CUDA_TRY(cudaGetLastError());
  const tc::QueueArgs qa{queue, counters, pending, cons_off, cons};
  if (pm_ok(c->p.q, c->p.ell) && !(c->p.dbg & 2u))
    return launch_tc_ws_enc<9, 29, true, FHEGPU_ENC_QUEUE, true>(c, c->store, pr->d_ops, (uint32_t)pr->n_ops,
                                                                 lanes, nullptr, nullptr, qa);
  return launch_tc_ws_enc<9, 29, false, FHEGPU_ENC_QUEUE, true>(c, c->store, pr->d_ops, (uint32_t)pr->n_ops,
                                                                lanes, nullptr, nullptr, qa);
}


// A whole single-lane program in one warp-dataflow launch (flow_nand.cuh).
int launch_flow(fhegpu_ctx *c, fhegpu_prog *pr, uint32_t lanes) {
  if (pr->n_ops == 0 || lanes == 0) return FHEGPU_OK;
  if (lanes != 1 || !(c->p.k == 3 && c->p.ell == 17) || (c->p.dbg & 4u)) return FHEGPU_EUNSUP;
  if (effective_kernel(c) != FHEGPU_KERNEL_TCGEN05) return FHEGPU_EUNSUP;   // 'simt': the cross-check kernel
  pr->flow_epoch = pr->flow_epoch % flow::TAG_MAX + 1u;
  const uint32_t q_magic = (uint32_t)((1ull << 32) / c->p.q);
  flow::flow_kernel<3, 17><<<pr->flow_ctas, 32 * flow::WARPS * flow::SPLIT, 0, c->stream>>>(
      c->store, pr->d_flow_scratch, pr->d_flow_ents, pr->d_flow_off, pr->flow_epoch, q_magic, c->p);
  CUDA_TRY(cudaGetLastError());
  return FHEGPU_OK;
}

#ifndef FHEGPU_ENC_RESIDENT
#define FHEGPU_ENC_RESIDENT 2     // {0,128} A operand: builders pace this pipeline (+4.5%, measured)
#endif

// A whole small per-lane program in one lane-resident launch (tc_nand_resident.cuh).
int launch_resident(fhegpu_ctx *c, fhegpu_prog *pr, uint32_t lanes) {
  if (lanes == 0 || pr->r_ops == 0) return FHEGPU_OK;
  if (effective_kernel(c) != FHEGPU_KERNEL_TCGEN05 || (c->p.dbg & 4u)) return FHEGPU_EUNSUP;
  if (!(c->p.k == 9 && c->p.ell == 29)) return FHEGPU_EUNSUP;
  using R = tc::GeoRes<9, 29>;
  const uint32_t smem = R::smem_bytes(pr->r_in, pr->r_local);
  if (smem > 227u * 1024u) return FHEGPU_EUNSUP;
  const uint32_t n_groups = (lanes + tc::RES_W - 1) / tc::RES_W;    // the last group may be partial
  const unsigned grid = (unsigned)std::min<uint64_t>(n_groups, (uint64_t)c->num_sms);
  DevParams p = c->p;
  const bool pm = pm_ok(c->p.q, c->p.ell) && !(c->p.dbg & 2u);
  // plans whose slot order has no operand produced < 5 slots back compile the RAW waits out
  // dbg bit 21 forces the instantiation with every RAW wait compiled in (parity tests)
  const bool deps = pr->r_deps || (c->p.dbg & (1u << 21));
  auto kern = pm ? (deps ? tc::resident_tc_kernel<9, 29, true, FHEGPU_ENC_RESIDENT, true>
                               : tc::resident_tc_kernel<9, 29, true, FHEGPU_ENC_RESIDENT, false>)
                 : (deps ? tc::resident_tc_kernel<9, 29, false, FHEGPU_ENC_RESIDENT, true>
                               : tc::resident_tc_kernel<9, 29, false, FHEGPU_ENC_RESIDENT, false>);
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, R::THREADS, smem, c->stream>>>(c->store, pr->d_rplan, pr->d_rin, pr->r_ops, pr->r_in, pr->r_local,
                                               pr->r_out, lanes, n_groups, p);
  CUDA_TRY(cudaGetLastError());
  return FHEGPU_OK;
}

// A whole deep per-lane program in one register-file launch (tc_nand_regfile.cuh).
int launch_regfile(fhegpu_ctx *c, fhegpu_prog *pr, uint32_t lanes, uint32_t *store, uint32_t *spill = nullptr) {
  if (lanes == 0 || pr->rf_ops == 0) return FHEGPU_OK;
  if (effective_kernel(c) != FHEGPU_KERNEL_TCGEN05 || (c->p.dbg & 4u)) return FHEGPU_EUNSUP;
  if (!(c->p.k == 9 && c->p.ell == 29)) return FHEGPU_EUNSUP;
  using F = tc::GeoRF<9, 29>;
  const uint32_t smem = F::smem_bytes(pr->rf_buf);
  if (smem > 227u * 1024u) return FHEGPU_EUNSUP;
  const unsigned grid = (unsigned)std::min<uint64_t>(lanes, (uint64_t)c->num_sms);
  if (spill == nullptr) {
    if (pr->rf_spill_base + (uint64_t)grid * pr->rf_spill > c->capacity)
      return fail(FHEGPU_EINVAL, "register-file spill region beyond store capacity");
    spill = c->store + pr->rf_spill_base * c->p.ct_words;
  }
  DevParams p = c->p;
  const bool pm = pm_ok(c->p.q, c->p.ell) && !(c->p.dbg & 2u);
  auto kern = pm ? tc::regfile_tc_kernel<9, 29, true, FHEGPU_ENC_RESIDENT>
                 : tc::regfile_tc_kernel<9, 29, false, FHEGPU_ENC_RESIDENT>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, F::THREADS, smem, c->stream>>>(store, pr->d_rfslots, pr->d_rffills, pr->rf_ops, pr->rf_fills,
                                               pr->rf_buf, lanes, spill, pr->rf_spill, p);
  CUDA_TRY(cudaGetLastError());
  return FHEGPU_OK;
}

}  // namespace

extern "C" {

const char *fhegpu_last_error(void) { return g_err.c_str(); }
const char *fhegpu_version(void) { return "fhegpu 0.1 (sm_100a)"; }

int fhegpu_ctx_create(const fhegpu_params *params, int device, fhegpu_ctx **out) {
  if (!params || !out) return fail(FHEGPU_EINVAL, "null argument");
  *out = nullptr;
  const uint32_t k = params->n + 1, ell = params->ell, q = params->q;
  if (params->n < 1 || k > 16) return fail(FHEGPU_EUNSUP, "library supports 1 <= n <= 15");
  if (q < 8 || (q & 1u) == 0 || q >= (1u << 31))
    return fail(FHEGPU_EUNSUP, "library supports odd 8 <= q < 2^31");
  if (ell != (uint32_t)(32 - __builtin_clz(q - 1)))
    return fail(FHEGPU_EINVAL, "ell must equal bitlen(q - 1)");
  CUDA_TRY(cudaSetDevice(device));
  auto *c = new fhegpu_ctx();
  c->device = device;
  c->n = params->n;
  c->m = params->m;
  c->p.k = k;
  c->p.ell = ell;
  c->p.q = q;
  c->p.rows = k * ell;
  c->p.words = k * ell * k;
  c->p.ct_words = (c->p.words + 3u) & ~3u;
  c->p.mu = ~0ull / q;  // floor((2^64 - 1) / q) == floor(2^64 / q) for odd q
  c->p.dbg = 0;
  c->p.pm_c = (uint32_t)((1ull << ell) - q);
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    delete c;
    return fail(FHEGPU_ECUDA, std::string("cudaGetDeviceProperties: ") + cudaGetErrorString(e));
  }
  c->num_sms = prop.multiProcessorCount;
  c->tc_capable = (prop.major == 10 && prop.minor == 0) && tc_instantiated(k, ell);
  e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(FHEGPU_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
  }
  c->stream = c->own_stream;
  *out = c;
  return FHEGPU_OK;
}

void fhegpu_ctx_destroy(fhegpu_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaFree(c->store);
  cudaFree(c->d_stage);
  cudaFree(c->d_idx);
  cudaFree(c->d_comp);
  cudaFree(c->d_copy);
  cudaFree(c->d_tmp_ops);
  cudaFree(c->d_jump);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  cudaFree(c->d_hstage);
  if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  for (int r = 0; r < kStreamRegions; ++r) {
    if (c->ev_in[r]) cudaEventDestroy(c->ev_in[r]);
    if (c->ev_done[r]) cudaEventDestroy(c->ev_done[r]);
    if (c->ev_free[r]) cudaEventDestroy(c->ev_free[r]);
  }
  delete c;
}

int fhegpu_ctx_set_stream(fhegpu_ctx *c, void *stream) {
  if (!c) return fail(FHEGPU_EINVAL, "null ctx");
  c->stream = (cudaStream_t)stream;  // NULL = the legacy default stream
  return FHEGPU_OK;
}

void *fhegpu_ctx_own_stream(const fhegpu_ctx *c) { return c ? (void *)c->own_stream : nullptr; }

int fhegpu_ctx_set_kernel(fhegpu_ctx *c, int kernel) {
  if (!c) return fail(FHEGPU_EINVAL, "null ctx");
  if (kernel < 0 || kernel > 2) return fail(FHEGPU_EINVAL, "unknown kernel id");
  if (kernel == FHEGPU_KERNEL_TCGEN05 && !c->tc_capable)
    return fail(FHEGPU_EUNSUP, "tcgen05 kernel unavailable for this device/params");
  c->kernel_pref = kernel;
  return FHEGPU_OK;
}

int fhegpu_ctx_kernel(const fhegpu_ctx *c) { return c ? effective_kernel(c) : -1; }

int fhegpu_ctx_num_sms(const fhegpu_ctx *c) { return c ? c->num_sms : 0; }

int fhegpu_ctx_set_debug(fhegpu_ctx *c, uint32_t dbg) {
  if (!c) return fail(FHEGPU_EINVAL, "null ctx");
  c->p.dbg = dbg;
  return FHEGPU_OK;
}

uint32_t fhegpu_ct_words(const fhegpu_ctx *c) { return c ? c->p.ct_words : 0; }

int fhegpu_sync(fhegpu_ctx *c) {
  if (!c) return fail(FHEGPU_EINVAL, "null ctx");
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FHEGPU_OK;
}

int fhegpu_store_reserve(fhegpu_ctx *c, uint64_t n_cts) {
  if (!c) return fail(FHEGPU_EINVAL, "null ctx");
  if (n_cts <= c->capacity) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  uint32_t *nw = nullptr;
  const size_t bytes = (size_t)n_cts * c->p.ct_words * sizeof(uint32_t);
  cudaError_t e = cudaMalloc(&nw, bytes);
  if (e != cudaSuccess)
    return fail(FHEGPU_ENOMEM, "store_reserve: cannot allocate " + std::to_string(bytes) + " bytes");
  if (c->store) {
    CUDA_TRY(cudaMemcpyAsync(nw, c->store, (size_t)c->capacity * c->p.ct_words * 4,
                             cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    cudaFree(c->store);
  }
  c->store = nw;
  c->capacity = n_cts;
  ++c->store_gen;
  return FHEGPU_OK;
}

uint64_t fhegpu_store_capacity(const fhegpu_ctx *c) { return c ? c->capacity : 0; }

uint64_t fhegpu_store_device_ptr(const fhegpu_ctx *c) { return c ? (uint64_t)(uintptr_t)c->store : 0; }

static int check_idx(fhegpu_ctx *c, const uint64_t *idx, uint64_t count) {
  for (uint64_t i = 0; i < count; ++i)
    if (idx[i] >= c->capacity)
      return fail(FHEGPU_EINVAL, "ciphertext index " + std::to_string(idx[i]) + " beyond capacity " +
                                     std::to_string(c->capacity));
  return FHEGPU_OK;
}

int fhegpu_store_write(fhegpu_ctx *c, const uint64_t *idx, uint64_t count, const uint32_t *host_v) {
  if (!c || (count && (!idx || !host_v))) return fail(FHEGPU_EINVAL, "null argument");
  if (int rc = check_idx(c, idx, count)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t per = (size_t)c->p.words * 4;
  const uint64_t chunk = std::max<uint64_t>(1, kStagingCap / per);
  for (uint64_t s = 0; s < count; s += chunk) {
    const uint64_t n = std::min(chunk, count - s);
    if (int rc = ensure((void **)&c->d_stage, &c->stage_bytes, n * per)) return rc;
    if (int rc = ensure((void **)&c->d_idx, &c->idx_cap, n * 8)) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->d_stage, host_v + s * c->p.words, n * per, cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_idx, idx + s, n * 8, cudaMemcpyHostToDevice, c->stream));
    scatter_kernel<<<grid_for(n * c->p.ct_words, c->num_sms), 256, 0, c->stream>>>(
        c->store, c->d_idx, c->d_stage, n, c->p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(c->stream));  // staging is reused by the next chunk
  }
  return FHEGPU_OK;
}

static int read_impl(fhegpu_ctx *c, const uint64_t *idx, const uint8_t *comp, uint64_t count, int row,
                     uint32_t *host) {
  if (!c || (count && (!idx || !host))) return fail(FHEGPU_EINVAL, "null argument");
  if (row >= (int)c->p.rows) return fail(FHEGPU_EINVAL, "row out of range");
  if (int rc = check_idx(c, idx, count)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  const uint32_t per_words = row < 0 ? c->p.words : c->p.k;
  const size_t per = (size_t)per_words * 4;
  const uint64_t chunk = std::max<uint64_t>(1, kStagingCap / per);
  for (uint64_t s = 0; s < count; s += chunk) {
    const uint64_t n = std::min(chunk, count - s);
    if (int rc = ensure((void **)&c->d_stage, &c->stage_bytes, n * per)) return rc;
    if (int rc = ensure((void **)&c->d_idx, &c->idx_cap, n * 8)) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->d_idx, idx + s, n * 8, cudaMemcpyHostToDevice, c->stream));
    const uint8_t *dcomp = nullptr;
    if (comp) {
      if (int rc = ensure((void **)&c->d_comp, &c->comp_cap, n)) return rc;
      CUDA_TRY(cudaMemcpyAsync(c->d_comp, comp + s, n, cudaMemcpyHostToDevice, c->stream));
      dcomp = c->d_comp;
    }
    gather_kernel<<<grid_for(n * per_words, c->num_sms), 256, 0, c->stream>>>(
        c->store, c->d_idx, dcomp, c->d_stage, n, row, c->p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(host + s * per_words, c->d_stage, n * per, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  return FHEGPU_OK;
}

int fhegpu_store_read(fhegpu_ctx *c, const uint64_t *idx, const uint8_t *comp, uint64_t count,
                      uint32_t *host_v) {
  return read_impl(c, idx, comp, count, -1, host_v);
}

int fhegpu_store_read_rows(fhegpu_ctx *c, const uint64_t *idx, const uint8_t *comp, uint64_t count,
                           uint32_t row, uint32_t *host_rows) {
  return read_impl(c, idx, comp, count, (int)row, host_rows);
}

int fhegpu_store_decrypt_rows(fhegpu_ctx *c, const uint64_t *idx, const uint8_t *comp, uint64_t count,
                              uint32_t row, const uint32_t *pw, int32_t *host_x) {
  if (!c || !pw || (count && (!idx || !host_x))) return fail(FHEGPU_EINVAL, "null argument");
  if (row >= c->p.rows) return fail(FHEGPU_EINVAL, "row out of range");
  if (c->p.k * c->p.ell > 16 * 32) return fail(FHEGPU_EUNSUP, "k * ell beyond 512");
  if (int rc = check_idx(c, idx, count)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t pw_bytes = (size_t)c->p.k * c->p.ell * 4;
  const uint64_t chunk = std::max<uint64_t>(1, (kStagingCap - pw_bytes) / 4);
  for (uint64_t s = 0; s < count; s += chunk) {
    const uint64_t n = std::min(chunk, count - s);
    if (int rc = ensure((void **)&c->d_stage, &c->stage_bytes, pw_bytes + n * 4)) return rc;
    if (int rc = ensure((void **)&c->d_idx, &c->idx_cap, n * 8)) return rc;
    uint32_t *d_pw = c->d_stage;
    int32_t *d_x = reinterpret_cast<int32_t *>(c->d_stage + c->p.k * c->p.ell);
    CUDA_TRY(cudaMemcpyAsync(d_pw, pw, pw_bytes, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_idx, idx + s, n * 8, cudaMemcpyHostToDevice, c->stream));
    const uint8_t *dcomp = nullptr;
    if (comp) {
      if (int rc = ensure((void **)&c->d_comp, &c->comp_cap, n)) return rc;
      CUDA_TRY(cudaMemcpyAsync(c->d_comp, comp + s, n, cudaMemcpyHostToDevice, c->stream));
      dcomp = c->d_comp;
    }
    decrypt_rows_kernel<<<grid_for(n, c->num_sms), 256, 0, c->stream>>>(c->store, c->d_idx, dcomp, d_pw, d_x, n,
                                                                        row, c->p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(host_x + s, d_x, n * 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  return FHEGPU_OK;
}

int fhegpu_store_copy_slots(fhegpu_ctx *c, const uint32_t *src_slots, const uint32_t *dst_slots, uint32_t n,
                            uint64_t lanes) {
  if (!c || (n && (!src_slots || !dst_slots))) return fail(FHEGPU_EINVAL, "null argument");
  if (n == 0 || lanes == 0) return FHEGPU_OK;
  std::vector<uint32_t> both(2 * (size_t)n);
  for (uint32_t i = 0; i < n; ++i) {
    if (((uint64_t)src_slots[i] + 1) * lanes > c->capacity || ((uint64_t)dst_slots[i] + 1) * lanes > c->capacity)
      return fail(FHEGPU_EINVAL, "slot " + std::to_string(std::max(src_slots[i], dst_slots[i])) + " x " +
                                     std::to_string(lanes) + " lanes beyond store capacity " +
                                     std::to_string(c->capacity));
    both[i] = src_slots[i];
    both[n + i] = dst_slots[i];
  }
  {  // no destination may be written twice or read by another pair
    std::vector<uint32_t> dsts(both.begin() + n, both.end());
    std::sort(dsts.begin(), dsts.end());
    for (uint32_t i = 1; i < n; ++i)
      if (dsts[i] == dsts[i - 1]) return fail(FHEGPU_EINVAL, "duplicate destination slot " + std::to_string(dsts[i]));
    for (uint32_t i = 0; i < n; ++i)
      if (both[i] != both[n + i] && std::binary_search(dsts.begin(), dsts.end(), both[i]))
        return fail(FHEGPU_EINVAL, "source slot " + std::to_string(both[i]) + " is another pair's destination");
  }
  CUDA_TRY(cudaSetDevice(c->device));
  // a dedicated buffer, written only by stream-ordered copies: the previous call's kernel has
  // read it before this upload lands, so the call stays asynchronous
  if (int rc = ensure((void **)&c->d_copy, &c->copy_cap, both.size() * 4)) return rc;
  uint32_t *d = c->d_copy;
  CUDA_TRY(cudaMemcpyAsync(d, both.data(), both.size() * 4, cudaMemcpyHostToDevice, c->stream));
  const uint64_t run_u4 = lanes * c->p.ct_words / 4;
  dim3 grid((unsigned)std::max<uint64_t>(1, std::min<uint64_t>((run_u4 + 255) / 256, 1024)),
            std::min<uint32_t>(n, 65535u));
  copy_slots_kernel<<<grid, 256, 0, c->stream>>>(c->store, d, d + n, n, run_u4);
  CUDA_TRY(cudaGetLastError());
  return FHEGPU_OK;
}

int fhegpu_store_write_range(fhegpu_ctx *c, uint64_t first, uint64_t count, const uint32_t *host_v,
                             int async) {
  if (!c || (count && !host_v)) return fail(FHEGPU_EINVAL, "null argument");
  if (first + count > c->capacity) return fail(FHEGPU_EINVAL, "range beyond store capacity");
  if (count == 0) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t dense = (size_t)c->p.words * 4, pitch = (size_t)c->p.ct_words * 4;
  CUDA_TRY(cudaMemcpy2DAsync(c->store + first * c->p.ct_words, pitch, host_v, dense, dense, count,
                             cudaMemcpyHostToDevice, c->stream));
  if (!async) CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FHEGPU_OK;
}

int fhegpu_store_read_range(fhegpu_ctx *c, uint64_t first, uint64_t count, uint32_t *host_v,
                            int async) {
  if (!c || (count && !host_v)) return fail(FHEGPU_EINVAL, "null argument");
  if (first + count > c->capacity) return fail(FHEGPU_EINVAL, "range beyond store capacity");
  if (count == 0) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t dense = (size_t)c->p.words * 4, pitch = (size_t)c->p.ct_words * 4;
  CUDA_TRY(cudaMemcpy2DAsync(host_v, dense, c->store + first * c->p.ct_words, pitch, dense, count,
                             cudaMemcpyDeviceToHost, c->stream));
  if (!async) CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FHEGPU_OK;
}

namespace {

size_t packed_row_bytes(const fhegpu_ctx *c) { return ((size_t)c->p.rows * c->p.rows + 7) / 8; }

int set_pack_smem(fhegpu_ctx *c) {
  const size_t smem = std::max((packed_row_bytes(c) + 3) / 4 * 4, (size_t)c->p.words * 4);
  if (smem > 48 * 1024) {
    CUDA_TRY(cudaFuncSetAttribute(packed_to_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_TRY(cudaFuncSetAttribute(store_to_packed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  return FHEGPU_OK;
}

}  // namespace

int fhegpu_store_write_packed(fhegpu_ctx *c, uint64_t first, uint64_t count, const uint8_t *host) {
  if (!c || (count && !host)) return fail(FHEGPU_EINVAL, "null argument");
  if (first + count > c->capacity) return fail(FHEGPU_EINVAL, "range beyond store capacity");
  if (count == 0) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  if (int rc = set_pack_smem(c)) return rc;
  const size_t per = packed_row_bytes(c);
  const uint64_t chunk = std::max<uint64_t>(1, kStagingCap / per);
  for (uint64_t s = 0; s < count; s += chunk) {
    const uint64_t n = std::min(chunk, count - s);
    if (int rc = ensure((void **)&c->d_stage, &c->stage_bytes, n * per)) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->d_stage, host + s * per, n * per, cudaMemcpyHostToDevice, c->stream));
    packed_to_store_kernel<<<(unsigned)std::min<uint64_t>(n, c->num_sms * 8), 256, (per + 3) / 4 * 4, c->stream>>>(
        c->store + (first + s) * c->p.ct_words, (const uint8_t *)c->d_stage, n, (uint32_t)per, c->p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(c->stream));  // staging is reused by the next chunk
  }
  return FHEGPU_OK;
}

int fhegpu_store_read_packed(fhegpu_ctx *c, uint64_t first, uint64_t count, uint8_t *host) {
  if (!c || (count && !host)) return fail(FHEGPU_EINVAL, "null argument");
  if (first + count > c->capacity) return fail(FHEGPU_EINVAL, "range beyond store capacity");
  if (count == 0) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  if (int rc = set_pack_smem(c)) return rc;
  const size_t per = packed_row_bytes(c);
  const uint64_t chunk = std::max<uint64_t>(1, kStagingCap / per);
  for (uint64_t s = 0; s < count; s += chunk) {
    const uint64_t n = std::min(chunk, count - s);
    if (int rc = ensure((void **)&c->d_stage, &c->stage_bytes, n * per)) return rc;
    store_to_packed_kernel<<<(unsigned)std::min<uint64_t>(n, c->num_sms * 8), 256, (size_t)c->p.words * 4,
                             c->stream>>>((uint8_t *)c->d_stage, c->store + (first + s) * c->p.ct_words, n,
                                          (uint32_t)per, c->p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(host + s * per, c->d_stage, n * per, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  return FHEGPU_OK;
}

int fhegpu_prog_create(fhegpu_ctx *c, const fhegpu_op *ops, uint64_t n_ops,
                       const uint64_t *level_offsets, uint32_t n_levels, fhegpu_prog **out) {
  if (!c || !out || (n_ops && !ops) || !level_offsets) return fail(FHEGPU_EINVAL, "null argument");
  *out = nullptr;
  if (level_offsets[0] != 0 || level_offsets[n_levels] != n_ops)
    return fail(FHEGPU_EINVAL, "level offsets must span [0, n_ops]");
  for (uint32_t l = 0; l < n_levels; ++l)
    if (level_offsets[l + 1] < level_offsets[l]) return fail(FHEGPU_EINVAL, "level offsets not sorted");
  uint64_t n_slots = 0;
  for (uint64_t i = 0; i < n_ops; ++i) {
    const uint32_t mx = std::max(ops[i].left, std::max(ops[i].right, ops[i].out));
    if (mx >= (1u << 31) || (ops[i].flags & ~(3u | FHEGPU_OP_STREAM_OUT | FHEGPU_OP_TEMP)))
      return fail(FHEGPU_EINVAL, "bad op record " + std::to_string(i));
    n_slots = std::max<uint64_t>(n_slots, uint64_t(mx) + 1);
  }
  CUDA_TRY(cudaSetDevice(c->device));
  auto *pr = new fhegpu_prog();
  pr->n_ops = n_ops;
  pr->n_slots = n_slots;
  pr->offsets.assign(level_offsets, level_offsets + n_levels + 1);
  if (n_ops) {
    cudaError_t e = cudaMalloc(&pr->d_ops, n_ops * sizeof(OpRec));
    if (e != cudaSuccess) {
      delete pr;
      return fail(FHEGPU_ENOMEM, "prog_create: cannot allocate op table");
    }
    e = cudaMemcpyAsync(pr->d_ops, ops, n_ops * sizeof(OpRec), cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      cudaFree(pr->d_ops);
      delete pr;
      return fail(FHEGPU_ECUDA, std::string("prog_create upload: ") + cudaGetErrorString(e));
    }
  }
  *out = pr;
  return FHEGPU_OK;
}

int fhegpu_prog_run_range(fhegpu_ctx *c, fhegpu_prog *pr, uint32_t lanes, uint32_t first,
                          uint32_t last) {
  if (!c || !pr) return fail(FHEGPU_EINVAL, "null argument");
  const uint32_t n_levels = (uint32_t)pr->offsets.size() - 1;
  last = std::min(last, n_levels);
  // every slot the program (or its resident plan) names, for every lane, must be in the store
  const uint64_t slots = std::max({pr->n_slots, pr->use_resident ? pr->r_slots : 0,
                                    pr->use_regfile ? pr->rf_slots : 0});
  if (lanes && slots && (slots > c->capacity / lanes || slots * lanes > c->capacity))
    return fail(FHEGPU_EINVAL, "program needs " + std::to_string(slots) + " slots x " + std::to_string(lanes) +
                                   " lanes; store holds " + std::to_string(c->capacity) + " ciphertexts");
  CUDA_TRY(cudaSetDevice(c->device));
  if (pr->use_regfile && first == 0 && last == n_levels && !(c->p.dbg & 32768u)) {
    const int rc = launch_regfile(c, pr, lanes, c->store);
    if (rc != FHEGPU_EUNSUP) return rc;
    // else: level by level (register-file programs keep their level structure)
  } else if (pr->use_resident && first == 0 && last == n_levels && !(c->p.dbg & 32768u)) {
    const int rc = launch_resident(c, pr, lanes);
    if (rc != FHEGPU_EUNSUP) return rc;
    // else: level by level (resident programs keep their level structure)
  } else if (pr->use_flow && first == 0 && last == n_levels && !(c->p.dbg & 32768u)) {
    const int rc = launch_flow(c, pr, lanes);
    if (rc != FHEGPU_EUNSUP) return rc;
    // else: level by level (flow programs keep their level structure)
  } else if (pr->use_queue && first == 0 && last == n_levels && !(c->p.dbg & 32768u)) {
    const int rc = launch_queue(c, pr, lanes);
    if (rc != FHEGPU_EUNSUP) return rc;
    // else: level by level (queue programs keep their level structure)
  } else if (pr->d_deps && first == 0 && last == n_levels && !(c->p.dbg & 32768u)) {
    const int rc = launch_dataflow(c, c->store, pr->d_ops, (uint32_t)pr->n_ops, lanes, pr->d_deps,
                                   pr->d_progress);
    if (rc != FHEGPU_EUNSUP) return rc;
    if (!pr->levels_valid)
      return fail(FHEGPU_EUNSUP, "program needs the dataflow kernel (tcgen05, k = 9, ell = 29, "
                                 "< 2^32 items), which does not apply here");
    // else: level by level (valid: no op depends on an op of its own level)
  } else if (pr->d_deps && !pr->levels_valid) {
    return fail(FHEGPU_EINVAL, "a program without level structure runs whole (dataflow) only");
  }
  for (uint32_t l = first; l < last; ++l) {
    const uint64_t a = pr->offsets[l], b = pr->offsets[l + 1];
    if (int rc = launch_level(c, c->store, pr->d_ops + a, (uint32_t)(b - a), lanes)) return rc;
  }
  return FHEGPU_OK;
}

int fhegpu_prog_run(fhegpu_ctx *c, fhegpu_prog *pr, uint32_t lanes) {
  if (!pr) return fail(FHEGPU_EINVAL, "null prog");
  const uint32_t n_levels = (uint32_t)pr->offsets.size() - 1;
  // graphs pay off for chains of level launches; whole-program launches (register-file,
  // lane-resident, ready-queue, dataflow) run directly
  if (!c || !c->use_graphs || n_levels < 4 || c->stream == nullptr || pr->use_regfile || pr->use_resident ||
      pr->use_queue || pr->d_deps)
    return fhegpu_prog_run_range(c, pr, lanes, 0, n_levels);
  CUDA_TRY(cudaSetDevice(c->device));
  const int kern = effective_kernel(c);
  if (!pr->graph || pr->graph_lanes != lanes || pr->graph_stream != c->stream ||
      pr->graph_kernel != kern || pr->graph_dbg != c->p.dbg || pr->graph_store_gen != c->store_gen) {
    if (pr->graph) {
      cudaGraphExecDestroy(pr->graph);
      pr->graph = nullptr;
    }
    // first use: run eagerly once (sets kernel attributes outside capture), then capture
    if (int rc = fhegpu_prog_run_range(c, pr, lanes, 0, n_levels)) return rc;
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = fhegpu_prog_run_range(c, pr, lanes, 0, n_levels);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return fail(FHEGPU_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&pr->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(FHEGPU_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    pr->graph_lanes = lanes;
    pr->graph_stream = c->stream;
    pr->graph_kernel = kern;
    pr->graph_dbg = c->p.dbg;
    pr->graph_store_gen = c->store_gen;
    return FHEGPU_OK;                  // this call already ran the program once
  }
  CUDA_TRY(cudaGraphLaunch(pr->graph, c->stream));
  return FHEGPU_OK;
}

namespace {

int ensure_streaming(fhegpu_ctx *c) {
  if (c->h2d_stream) return FHEGPU_OK;
  CUDA_TRY(cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
  for (int r = 0; r < kStreamRegions; ++r) {
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_in[r], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_done[r], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_free[r], cudaEventDisableTiming));
  }
  return FHEGPU_OK;
}

}  // namespace

int fhegpu_prog_run_host(fhegpu_ctx *c, fhegpu_prog *pr, uint64_t lanes, uint32_t chunk_lanes,
                         int host_format, uint32_t n_in, const uint32_t *in_slots,
                         const void *const *host_in, uint32_t n_out, const uint32_t *out_slots,
                         void *const *host_out) {
  if (!c || !pr || (n_in && (!in_slots || !host_in)) || (n_out && (!out_slots || !host_out)))
    return fail(FHEGPU_EINVAL, "null argument");
  if (lanes == 0) return FHEGPU_OK;
  if (chunk_lanes == 0) return fail(FHEGPU_EINVAL, "chunk_lanes must be positive");
  if (host_format != FHEGPU_HOST_COMPACT && host_format != FHEGPU_HOST_PACKED)
    return fail(FHEGPU_EINVAL, "unknown host format");
  uint64_t n_slots = pr->n_slots;
  for (uint32_t i = 0; i < n_in; ++i) {
    if (!host_in[i]) return fail(FHEGPU_EINVAL, "null host input");
    n_slots = std::max<uint64_t>(n_slots, uint64_t(in_slots[i]) + 1);
  }
  for (uint32_t i = 0; i < n_out; ++i) {
    if (!host_out[i]) return fail(FHEGPU_EINVAL, "null host output");
    n_slots = std::max<uint64_t>(n_slots, uint64_t(out_slots[i]) + 1);
  }
  const uint64_t chunk = std::min<uint64_t>(chunk_lanes, lanes);
  const uint64_t n_chunks = (lanes + chunk - 1) / chunk;
  const int regions = (int)std::min<uint64_t>(kStreamRegions, n_chunks);
  const uint64_t region_cts = n_slots * chunk;
  if (region_cts * regions > c->capacity)
    return fail(FHEGPU_EINVAL, "store holds " + std::to_string(c->capacity) + " ciphertexts; streaming needs " +
                                   std::to_string(region_cts * regions) + " (reserve more or use smaller chunks)");
  CUDA_TRY(cudaSetDevice(c->device));
  if (int rc = ensure_streaming(c)) return rc;
  const bool packed = host_format == FHEGPU_HOST_PACKED;
  const size_t row_bytes = packed ? ((size_t)c->p.rows * c->p.rows + 7) / 8 : (size_t)c->p.words * 4;
  // staging per region: n_in + n_out arrays of `chunk` host-format rows (contiguous PCIe
  // copies run ~10% faster than pitched ones; the repack to the store's padded rows is
  // HBM-cheap and, for the packed format, cuts PCIe bytes by 1 - N^2/8 / (4 N k))
  const uint64_t stage_rows = (uint64_t)(n_in + n_out) * chunk;
  if (int rc = ensure((void **)&c->d_hstage, &c->hstage_bytes, regions * stage_rows * row_bytes)) return rc;
  const uint32_t n_levels = (uint32_t)pr->offsets.size() - 1;
  const unsigned repack_grid = (unsigned)std::max(1, c->num_sms * 8);
  // register-file programs run each chunk as one launch, spilling right after the streaming
  // regions when the store has room for it (else level launches)
  const uint64_t rf_spill_cts = (uint64_t)c->num_sms * pr->rf_spill;
  const bool use_rf = pr->use_regfile && !(c->p.dbg & 32768u) && region_cts * regions + rf_spill_cts <= c->capacity;
  uint32_t *rf_spill_ptr = c->store + region_cts * regions * c->p.ct_words;
  if (packed)
    if (int rc = set_pack_smem(c)) return rc;
  // everything queued on the context stream so far happens before the first copy
  CUDA_TRY(cudaEventRecord(c->ev_start, c->stream));
  CUDA_TRY(cudaStreamWaitEvent(c->h2d_stream, c->ev_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(c->d2h_stream, c->ev_start, 0));
  for (uint64_t ch = 0; ch < n_chunks; ++ch) {
    const int r = (int)(ch % regions);
    const uint64_t lane0 = ch * chunk, cl = std::min(chunk, lanes - lane0);
    uint32_t *base = c->store + (uint64_t)r * region_cts * c->p.ct_words;
    uint8_t *stage = (uint8_t *)c->d_hstage + (uint64_t)r * stage_rows * row_bytes;
    uint8_t *stage_out = stage + (uint64_t)n_in * chunk * row_bytes;
    // copy-in: region r (store + staging) is free once chunk ch - regions was copied out
    if (ch >= (uint64_t)regions) CUDA_TRY(cudaStreamWaitEvent(c->h2d_stream, c->ev_free[r], 0));
    for (uint32_t i = 0; i < n_in; ++i)
      CUDA_TRY(cudaMemcpyAsync(stage + (uint64_t)i * chunk * row_bytes,
                               (const uint8_t *)host_in[i] + lane0 * row_bytes, cl * row_bytes,
                               cudaMemcpyHostToDevice, c->h2d_stream));
    CUDA_TRY(cudaEventRecord(c->ev_in[r], c->h2d_stream));
    // evaluate: repack inputs, every level over this chunk's lanes (store layout
    // slot * cl + lane inside region r), repack outputs
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_in[r], 0));
    const unsigned g = (unsigned)std::min<uint64_t>(cl, repack_grid);
    for (uint32_t i = 0; i < n_in; ++i) {
      uint32_t *dst = base + (uint64_t)in_slots[i] * cl * c->p.ct_words;
      const uint8_t *src = stage + (uint64_t)i * chunk * row_bytes;
      if (packed)
        packed_to_store_kernel<<<g, 256, (row_bytes + 3) / 4 * 4, c->stream>>>(dst, src, cl, (uint32_t)row_bytes, c->p);
      else
        dense_to_store_kernel<<<g, 256, 0, c->stream>>>(dst, (const uint32_t *)src, cl, c->p);
    }
    CUDA_TRY(cudaGetLastError());
    int rc = FHEGPU_EUNSUP;
    if (use_rf) rc = launch_regfile(c, pr, (uint32_t)cl, base, rf_spill_ptr);   // the whole chunk in one launch
    if (rc == FHEGPU_EUNSUP) {
      for (uint32_t l = 0; l < n_levels; ++l) {
        const uint64_t a = pr->offsets[l], b = pr->offsets[l + 1];
        if (int rc2 = launch_level(c, base, pr->d_ops + a, (uint32_t)(b - a), (uint32_t)cl)) return rc2;
      }
    } else if (rc) {
      return rc;
    }
    for (uint32_t i = 0; i < n_out; ++i) {
      uint8_t *dst = stage_out + (uint64_t)i * chunk * row_bytes;
      const uint32_t *src = base + (uint64_t)out_slots[i] * cl * c->p.ct_words;
      if (packed)
        store_to_packed_kernel<<<g, 256, (size_t)c->p.words * 4, c->stream>>>(dst, src, cl, (uint32_t)row_bytes, c->p);
      else
        store_to_dense_kernel<<<g, 256, 0, c->stream>>>((uint32_t *)dst, src, cl, c->p);
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(c->ev_done[r], c->stream));
    // copy-out
    CUDA_TRY(cudaStreamWaitEvent(c->d2h_stream, c->ev_done[r], 0));
    for (uint32_t i = 0; i < n_out; ++i)
      CUDA_TRY(cudaMemcpyAsync((uint8_t *)host_out[i] + lane0 * row_bytes, stage_out + (uint64_t)i * chunk * row_bytes,
                               cl * row_bytes, cudaMemcpyDeviceToHost, c->d2h_stream));
    CUDA_TRY(cudaEventRecord(c->ev_free[r], c->d2h_stream));
  }
  // the context stream observes completion of every copy-out
  for (int r = 0; r < regions; ++r) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_free[r], 0));
  return FHEGPU_OK;
}

int fhegpu_prog_set_deps(fhegpu_ctx *c, fhegpu_prog *pr, const int32_t *deps) {
  if (!c || !pr || (pr->n_ops && !deps)) return fail(FHEGPU_EINVAL, "null argument");
  if (pr->n_ops >= (1ull << 31)) return fail(FHEGPU_EINVAL, "program too large for dataflow");
  for (uint64_t i = 0; i < 2 * pr->n_ops; ++i)
    if (deps[i] < -1 || (int64_t)deps[i] >= (int64_t)(i / 2))
      return fail(FHEGPU_EINVAL, "dependency " + std::to_string(i) + " is not an earlier op");
  // level launches stay a valid fallback only if no op depends on an op of its own level
  pr->levels_valid = true;
  for (size_t l = 0; l + 1 < pr->offsets.size() && pr->levels_valid; ++l)
    for (uint64_t i = pr->offsets[l]; i < pr->offsets[l + 1]; ++i)
      if ((deps[2 * i] >= 0 && (uint64_t)deps[2 * i] >= pr->offsets[l]) ||
          (deps[2 * i + 1] >= 0 && (uint64_t)deps[2 * i + 1] >= pr->offsets[l])) {
        pr->levels_valid = false;
        break;
      }
  CUDA_TRY(cudaSetDevice(c->device));
  cudaFree(pr->d_deps);
  cudaFree(pr->d_progress);
  pr->d_deps = nullptr;
  pr->d_progress = nullptr;
  if (pr->n_ops == 0) return FHEGPU_OK;
  CUDA_TRY(cudaMalloc(&pr->d_deps, pr->n_ops * sizeof(int2)));
  CUDA_TRY(cudaMalloc(&pr->d_progress, (size_t)std::max(c->num_sms, 1) * sizeof(uint32_t)));
  CUDA_TRY(cudaMemcpyAsync(pr->d_deps, deps, pr->n_ops * sizeof(int2), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  pr->deps_host.assign(deps, deps + 2 * pr->n_ops);
  pr->use_queue = false;                 // (re)enable with fhegpu_prog_set_queue
  if (pr->graph) {                      // launch structure changed
    cudaGraphExecDestroy(pr->graph);
    pr->graph = nullptr;
  }
  return FHEGPU_OK;
}

int fhegpu_prog_set_queue(fhegpu_ctx *c, fhegpu_prog *pr, int enable) {
  if (!c || !pr) return fail(FHEGPU_EINVAL, "null argument");
  if (pr->graph) {                      // launch structure changes
    cudaGraphExecDestroy(pr->graph);
    pr->graph = nullptr;
  }
  if (!enable) {
    pr->use_queue = false;
    return FHEGPU_OK;
  }
  const uint64_t n = pr->n_ops;
  if (pr->deps_host.size() != 2 * n) return fail(FHEGPU_EINVAL, "set the program's dependencies first");
  if (!pr->levels_valid) return fail(FHEGPU_EINVAL, "ready-queue programs need a level structure");
  // pending count = distinct producing ops; consumer lists (CSR) per producing op
  std::vector<uint32_t> pend0(n), cons_off(n + 1, 0);
  for (uint64_t i = 0; i < n; ++i) {
    const int32_t a = pr->deps_host[2 * i], b = pr->deps_host[2 * i + 1];
    pend0[i] = (a >= 0) + (b >= 0 && b != a);
    if (a >= 0) ++cons_off[a + 1];
    if (b >= 0 && b != a) ++cons_off[b + 1];
  }
  for (uint64_t i = 0; i < n; ++i) cons_off[i + 1] += cons_off[i];
  std::vector<uint32_t> cons(cons_off[n]), fill(cons_off.begin(), cons_off.end() - 1), roots;
  for (uint64_t i = 0; i < n; ++i) {
    const int32_t a = pr->deps_host[2 * i], b = pr->deps_host[2 * i + 1];
    if (a >= 0) cons[fill[a]++] = (uint32_t)i;
    if (b >= 0 && b != a) cons[fill[b]++] = (uint32_t)i;
    if (pend0[i] == 0) roots.push_back((uint32_t)i);
  }
  std::vector<uint32_t> meta;
  meta.reserve(2 * n + 1 + cons.size() + roots.size());
  meta.insert(meta.end(), pend0.begin(), pend0.end());
  meta.insert(meta.end(), cons_off.begin(), cons_off.end());
  meta.insert(meta.end(), cons.begin(), cons.end());
  meta.insert(meta.end(), roots.begin(), roots.end());
  CUDA_TRY(cudaSetDevice(c->device));
  cudaFree(pr->d_qmeta);
  pr->d_qmeta = nullptr;
  CUDA_TRY(cudaMalloc(&pr->d_qmeta, meta.size() * sizeof(uint32_t)));
  CUDA_TRY(cudaMemcpy(pr->d_qmeta, meta.data(), meta.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  pr->n_edges = cons.size();
  pr->n_roots = (uint32_t)roots.size();
  pr->use_queue = true;
  return FHEGPU_OK;
}

int fhegpu_flow_plan(const fhegpu_op *ops, const int32_t *deps, uint64_t n_ops, const uint64_t *level_offsets,
                     uint32_t n_levels, uint32_t n_cta, uint32_t *entries, uint32_t *worker_off,
                     double *model_cycles) {
  if (!ops || !deps || !level_offsets || !entries || !worker_off || n_cta == 0)
    return fail(FHEGPU_EINVAL, "null argument");
  if (n_ops == 0 || n_ops >= flow::MAX_GATES || level_offsets[0] != 0 || level_offsets[n_levels] != n_ops)
    return fail(FHEGPU_EINVAL, "bad program");
  for (uint64_t i = 0; i < 2 * n_ops; ++i)
    if (deps[i] < -1 || (int64_t)deps[i] >= (int64_t)(i / 2))
      return fail(FHEGPU_EINVAL, "dependency " + std::to_string(i) + " is not an earlier op");
  static_assert(sizeof(fhegpu_op) == sizeof(OpRec), "op record layout");
  const flow::FlowPlan pl = flow::flow_plan(reinterpret_cast<const OpRec *>(ops), deps, n_ops, level_offsets,
                                            n_levels, n_cta);
  std::memcpy(entries, pl.ents.data(), n_ops * sizeof(flow::Entry));
  std::memcpy(worker_off, pl.worker_off.data(), pl.worker_off.size() * sizeof(uint32_t));
  if (model_cycles) *model_cycles = pl.makespan;
  return FHEGPU_OK;
}

int fhegpu_prog_set_flow(fhegpu_ctx *c, fhegpu_prog *pr, int enable, double *model_cycles, uint32_t *stats) {
  if (!c || !pr) return fail(FHEGPU_EINVAL, "null argument");
  pr->use_flow = false;
  if (!enable) return FHEGPU_OK;
  const uint64_t n = pr->n_ops;
  if (pr->deps_host.size() != 2 * n) return fail(FHEGPU_EINVAL, "set the program's dependencies first");
  if (!pr->levels_valid) return fail(FHEGPU_EINVAL, "warp-dataflow programs need a level structure");
  if (!(c->p.k == 3 && c->p.ell == 17) || c->p.q > (1u << flow::VBITS))
    return fail(FHEGPU_EUNSUP, "warp-dataflow launches serve k = 3, ell = 17, q <= 2^17");
  if (n == 0 || n >= flow::MAX_GATES) return fail(FHEGPU_EUNSUP, "program size outside the warp-dataflow range");
  CUDA_TRY(cudaSetDevice(c->device));
  std::vector<OpRec> ops(n);
  CUDA_TRY(cudaMemcpy(ops.data(), pr->d_ops, n * sizeof(OpRec), cudaMemcpyDeviceToHost));
  const uint32_t n_cta = (uint32_t)std::max(c->num_sms, 1);
  const flow::FlowPlan pl = flow::flow_plan(ops.data(), pr->deps_host.data(), n, pr->offsets.data(),
                                            (uint32_t)pr->offsets.size() - 1, n_cta);
  if (pl.max_gates_per_worker > flow::TAG_MAX)
    return fail(FHEGPU_EUNSUP, "too many gates per worker for the ring tags");
  cudaFree(pr->d_flow_ents);
  cudaFree(pr->d_flow_off);
  cudaFree(pr->d_flow_scratch);
  pr->d_flow_ents = nullptr, pr->d_flow_off = nullptr, pr->d_flow_scratch = nullptr;
  const size_t scratch_bytes = n * (size_t)(c->p.rows) * sizeof(uint4);
  CUDA_TRY(cudaMalloc(&pr->d_flow_ents, n * sizeof(flow::Entry)));
  CUDA_TRY(cudaMalloc(&pr->d_flow_off, pl.worker_off.size() * sizeof(uint32_t)));
  CUDA_TRY(cudaMalloc(&pr->d_flow_scratch, scratch_bytes));
  CUDA_TRY(cudaMemcpy(pr->d_flow_ents, pl.ents.data(), n * sizeof(flow::Entry), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(pr->d_flow_off, pl.worker_off.data(), pl.worker_off.size() * sizeof(uint32_t),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemset(pr->d_flow_scratch, 0, scratch_bytes));      // tag 0: never written
  pr->flow_ctas = n_cta;
  pr->flow_epoch = 0;
  pr->flow_makespan = pl.makespan;
  pr->flow_stats[0] = pl.ring_operands, pr->flow_stats[1] = pl.scratch_operands;
  pr->flow_stats[2] = pl.store_operands, pr->flow_stats[3] = pl.max_gates_per_worker;
  if (model_cycles) *model_cycles = pl.makespan;
  if (stats) std::copy(pr->flow_stats, pr->flow_stats + 4, stats);
  if (pr->graph) {                      // launch structure changes
    cudaGraphExecDestroy(pr->graph);
    pr->graph = nullptr;
  }
  pr->use_flow = true;
  return FHEGPU_OK;
}

int fhegpu_prog_set_resident(fhegpu_ctx *c, fhegpu_prog *pr, const fhegpu_res_op *plan, uint32_t n_ops,
                             const uint32_t *in_slots, uint32_t n_in, uint32_t n_local) {
  if (!c || !pr) return fail(FHEGPU_EINVAL, "null argument");
  if (pr->graph) {
    cudaGraphExecDestroy(pr->graph);
    pr->graph = nullptr;
  }
  if (n_ops == 0) {
    pr->use_resident = false;
    return FHEGPU_OK;
  }
  if (!plan || (n_in && !in_slots)) return fail(FHEGPU_EINVAL, "null argument");
  if (n_ops > (uint32_t)tc::RES_MAX_OPS || n_in > (uint32_t)tc::RES_MAX_IN || n_local > (uint32_t)tc::RES_MAX_LOCAL)
    return fail(FHEGPU_EINVAL, "resident program too large");
  static_assert(sizeof(fhegpu_res_op) == sizeof(tc::ResOp), "fhegpu_res_op layout");
  uint32_t n_out = 0;
  for (uint32_t i = 0; i < n_ops; ++i) {
    const fhegpu_res_op &o = plan[i];
    auto bad_src = [&](uint32_t kind, uint32_t idx, int32_t prod) {
      if (kind == 0) return idx >= n_in || prod != -1;
      return kind != 1 || idx >= n_local || prod < 0 || (uint32_t)prod >= i || plan[prod].dest != idx;
    };
    if (bad_src(o.lkind, o.lidx, o.lprod) || bad_src(o.rkind, o.ridx, o.rprod) || o.dest >= n_local ||
        o.is_out > 1 || (o.flags & ~3u))
      return fail(FHEGPU_EINVAL, "bad resident op " + std::to_string(i));
    n_out += o.is_out;
  }
  // buffer rules the kernel's store-hazard and reuse logic rely on (fhegpu.h): a buffer holds
  // outputs only or temporaries only, and no gate overwrites a buffer whose value still has a
  // reader later in the plan
  for (uint32_t i = 0; i < n_ops; ++i)
    for (uint32_t j = i + 1; j < n_ops; ++j) {
      if (plan[j].dest != plan[i].dest) continue;
      if (plan[j].is_out != plan[i].is_out)
        return fail(FHEGPU_EINVAL, "resident ops " + std::to_string(i) + " and " + std::to_string(j) +
                                       " share a buffer between an output and a temporary");
      for (uint32_t r = j + 1; r < n_ops; ++r)
        if ((plan[r].lkind && plan[r].lprod == (int32_t)i) || (plan[r].rkind && plan[r].rprod == (int32_t)i))
          return fail(FHEGPU_EINVAL, "resident op " + std::to_string(j) + " overwrites buffer " +
                                         std::to_string(plan[i].dest) + " before op " + std::to_string(r) +
                                         " reads op " + std::to_string(i) + "'s value");
    }
  uint64_t r_slots = 0;
  for (uint32_t i = 0; i < n_in; ++i) r_slots = std::max<uint64_t>(r_slots, uint64_t(in_slots[i]) + 1);
  for (uint32_t i = 0; i < n_ops; ++i)
    if (plan[i].is_out) r_slots = std::max<uint64_t>(r_slots, uint64_t(plan[i].out_slot) + 1);
  CUDA_TRY(cudaSetDevice(c->device));
  cudaFree(pr->d_rplan);
  cudaFree(pr->d_rin);
  pr->d_rplan = nullptr;
  pr->d_rin = nullptr;
  // the plan, then the group's slot order (operand reuse, RAW distances)
  std::vector<uint8_t> buf(n_ops * sizeof(tc::ResOp) + n_ops * tc::RES_W);
  std::memcpy(buf.data(), plan, n_ops * sizeof(tc::ResOp));
  tc::ResSlotOrder sched;
  const uint8_t *order = buf.data() + n_ops * sizeof(tc::ResOp);
  sched.run(reinterpret_cast<const tc::ResOp *>(plan), (int)n_ops, tc::RES_W, buf.data() + n_ops * sizeof(tc::ResOp));
  pr->r_deps = tc::ResSlotOrder::near_deps(reinterpret_cast<const tc::ResOp *>(plan), (int)n_ops, tc::RES_W, order);
  CUDA_TRY(cudaMalloc(&pr->d_rplan, buf.size()));
  CUDA_TRY(cudaMalloc(&pr->d_rin, std::max(n_in, 1u) * sizeof(uint32_t)));
  CUDA_TRY(cudaMemcpy(pr->d_rplan, buf.data(), buf.size(), cudaMemcpyHostToDevice));
  if (n_in) CUDA_TRY(cudaMemcpy(pr->d_rin, in_slots, n_in * sizeof(uint32_t), cudaMemcpyHostToDevice));
  pr->r_ops = n_ops;
  pr->r_in = n_in;
  pr->r_local = n_local;
  pr->r_out = n_out;
  pr->r_slots = r_slots;
  pr->use_resident = true;
  return FHEGPU_OK;
}

int fhegpu_rf_plan(const fhegpu_rf_gate *gates, uint32_t n_gates, const uint32_t *in_slots, uint32_t n_in,
                   uint32_t n_buf, uint32_t min_dist, uint32_t lookahead, uint32_t *order, fhegpu_rf_slot *slots,
                   fhegpu_rf_fill *fills, uint32_t fill_cap, uint32_t *n_fills, uint32_t *n_spill, uint32_t *stats) {
  if (!gates || (n_in && !in_slots) || !order || !slots || !fills || !n_fills || !n_spill)
    return fail(FHEGPU_EINVAL, "null argument");
  rf::Planner pl;
  pl.gates = gates, pl.n = n_gates, pl.n_in = n_in, pl.in_slots = in_slots;
  pl.n_buf = n_buf, pl.dist = std::max(1u, min_dist), pl.look = lookahead;
  pl.reuse = !getenv("FHEGPU_RF_NOREUSE");     // experiment knob: schedule without reuse preference
  if (!pl.run()) return fail(FHEGPU_EINVAL, pl.err);
  if (pl.fills.size() > fill_cap)
    return fail(FHEGPU_EINVAL, "fill_cap " + std::to_string(fill_cap) + " < " + std::to_string(pl.fills.size()));
  std::memcpy(order, pl.order.data(), n_gates * sizeof(uint32_t));
  std::memcpy(slots, pl.slots.data(), n_gates * sizeof(fhegpu_rf_slot));
  if (!pl.fills.empty()) std::memcpy(fills, pl.fills.data(), pl.fills.size() * sizeof(fhegpu_rf_fill));
  *n_fills = (uint32_t)pl.fills.size();
  *n_spill = pl.n_spill;
  if (stats)
    stats[0] = pl.stalls, stats[1] = pl.n_stores, stats[2] = (uint32_t)pl.fills.size(), stats[3] = pl.n_reuse_l,
    stats[4] = pl.n_reuse_r;
  return FHEGPU_OK;
}

int fhegpu_prog_set_regfile(fhegpu_ctx *c, fhegpu_prog *pr, const fhegpu_rf_slot *slots, uint32_t n_slots,
                            const fhegpu_rf_fill *fills, uint32_t n_fills, uint32_t n_buf, uint32_t n_spill,
                            uint64_t spill_base) {
  if (!c || !pr) return fail(FHEGPU_EINVAL, "null argument");
  if (pr->graph) {
    cudaGraphExecDestroy(pr->graph);
    pr->graph = nullptr;
  }
  if (n_slots == 0) {
    pr->use_regfile = false;
    return FHEGPU_OK;
  }
  if (!slots || (n_fills && !fills)) return fail(FHEGPU_EINVAL, "null argument");
  if (n_buf < 4 || tc::GeoRF<9, 29>::smem_bytes(n_buf) > 227u * 1024u)
    return fail(FHEGPU_EINVAL, "register file of " + std::to_string(n_buf) + " buffers does not fit shared memory");
  static_assert(sizeof(fhegpu_rf_slot) == 16 && sizeof(fhegpu_rf_fill) == 32, "plan record layout");
  uint64_t rf_slots = 0;
  auto loc = [&](uint32_t x) {
    if (x & rf::STORE_SPILL) return (x & ~rf::STORE_SPILL) < n_spill;
    rf_slots = std::max<uint64_t>(rf_slots, uint64_t(x) + 1);
    return true;
  };
  for (uint32_t t = 0; t < n_slots; ++t) {
    const fhegpu_rf_slot &s = slots[t];
    bool ok = s.lbuf < n_buf && s.rbuf < n_buf && s.dbuf < n_buf;
    for (uint32_t w : {s.lwait, s.rwait})
      if (w != rf::NONE) ok = ok && ((w & rf::WAIT_FILL) ? (w & ~rf::WAIT_FILL) < n_fills : w < t);
    if (s.bits & rf::SB_STORE) ok = ok && loc(s.store);
    if (!ok) return fail(FHEGPU_EINVAL, "bad register-file slot " + std::to_string(t));
  }
  for (uint32_t f = 0; f < n_fills; ++f) {
    const fhegpu_rf_fill &x = fills[f];
    // a fill's conditions look back only (else the producer would wait on its own consumers)
    if (x.buf >= n_buf || !loc(x.src) || x.consumer >= n_slots || x.w_built > x.consumer ||
        x.w_epi > x.consumer || x.w_st > x.consumer || (f && x.consumer < fills[f - 1].consumer))
      return fail(FHEGPU_EINVAL, "bad register-file fill " + std::to_string(f));
  }
  CUDA_TRY(cudaSetDevice(c->device));
  cudaFree(pr->d_rfslots);
  cudaFree(pr->d_rffills);
  pr->d_rfslots = nullptr;
  pr->d_rffills = nullptr;
  CUDA_TRY(cudaMalloc(&pr->d_rfslots, (size_t)n_slots * sizeof(fhegpu_rf_slot)));
  CUDA_TRY(cudaMalloc(&pr->d_rffills, std::max<size_t>(1, n_fills) * sizeof(fhegpu_rf_fill)));
  CUDA_TRY(cudaMemcpy(pr->d_rfslots, slots, (size_t)n_slots * sizeof(fhegpu_rf_slot), cudaMemcpyHostToDevice));
  if (n_fills) CUDA_TRY(cudaMemcpy(pr->d_rffills, fills, (size_t)n_fills * sizeof(fhegpu_rf_fill), cudaMemcpyHostToDevice));
  pr->rf_ops = n_slots;
  pr->rf_fills = n_fills;
  pr->rf_buf = n_buf;
  pr->rf_spill = n_spill;
  pr->rf_spill_base = spill_base;
  pr->rf_slots = rf_slots;
  pr->use_regfile = true;
  return FHEGPU_OK;
}

int fhegpu_res_slot_order(const fhegpu_res_op *plan, uint32_t n_ops, uint32_t lanes, uint8_t *order) {
  if (!plan || !order) return fail(FHEGPU_EINVAL, "null argument");
  if (lanes < 1 || lanes > 4 || n_ops > (uint32_t)tc::RES_MAX_OPS || lanes * n_ops > 32)
    return fail(FHEGPU_EINVAL, "slot order: lanes <= 4, n_ops <= 8");
  for (uint32_t i = 0; i < n_ops; ++i) {
    const fhegpu_res_op &o = plan[i];
    if ((o.lkind && (o.lprod < 0 || (uint32_t)o.lprod >= i)) || (o.rkind && (o.rprod < 0 || (uint32_t)o.rprod >= i)))
      return fail(FHEGPU_EINVAL, "bad resident op " + std::to_string(i));
  }
  tc::ResSlotOrder sched;
  sched.run(reinterpret_cast<const tc::ResOp *>(plan), (int)n_ops, (int)lanes, order);
  return FHEGPU_OK;
}

int fhegpu_ctx_set_graphs(fhegpu_ctx *c, int enable) {
  if (!c) return fail(FHEGPU_EINVAL, "null ctx");
  c->use_graphs = enable != 0;
  return FHEGPU_OK;
}

uint32_t fhegpu_prog_launches(const fhegpu_prog *pr) {
  if (!pr) return 0;
  if (pr->use_regfile || pr->use_resident || pr->use_flow) return 1;   // register-file / lane-resident /
                                                                       // warp-dataflow: one launch
  if (pr->use_queue) return 2;                  // ready queue: state reset + one launch
  if (pr->d_deps) return 1;                     // dataflow: one launch (tcgen05 parameter sets)
  uint32_t n = 0;
  for (size_t l = 0; l + 1 < pr->offsets.size(); ++l) n += pr->offsets[l + 1] > pr->offsets[l];
  return n;
}

void fhegpu_prog_destroy(fhegpu_prog *pr) {
  if (!pr) return;
  if (pr->graph) cudaGraphExecDestroy(pr->graph);
  cudaFree(pr->d_deps);
  cudaFree(pr->d_progress);
  cudaFree(pr->d_qmeta);
  cudaFree(pr->d_qrun);
  cudaFree(pr->d_rplan);
  cudaFree(pr->d_rin);
  cudaFree(pr->d_rfslots);
  cudaFree(pr->d_rffills);
  cudaFree(pr->d_flow_ents);
  cudaFree(pr->d_flow_off);
  cudaFree(pr->d_flow_scratch);
  cudaFree(pr->d_ops);
  delete pr;
}

namespace {

// One level of `count` products bits(V1) * V2 through the level kernels.  shared_left: v1 is
// ONE ciphertext used as every product's left operand.  ring: return C1 V2 mod q instead of
// NAND's (G - C1 V2) mod q, as the complement of the NAND result (fhe.py:366-379).
int product_batch(fhegpu_ctx *c, const uint32_t *v1, bool shared_left, const uint32_t *v2, uint32_t *out,
                  uint64_t count, bool ring, const char *what) {
  if (!c || (count && (!v1 || !v2 || !out))) return fail(FHEGPU_EINVAL, "null argument");
  if (count == 0) return FHEGPU_OK;
  if (count >= (1u << 29)) return fail(FHEGPU_EINVAL, "batch too large");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t ctb = (size_t)c->p.ct_words * 4, dense = (size_t)c->p.words * 4;
  const uint64_t n_left = shared_left ? 1 : count;
  const uint64_t right0 = n_left, out0 = n_left + count;
  uint32_t *buf = nullptr;
  CUDA_TRY(cudaMalloc(&buf, (out0 + count) * ctb));
  std::vector<OpRec> ops(count);
  for (uint64_t i = 0; i < count; ++i)
    ops[i] = OpRec{(uint32_t)(shared_left ? 0 : i), (uint32_t)(right0 + i), (uint32_t)(out0 + i), 0u};
  int rc = ensure((void **)&c->d_tmp_ops, &c->tmp_ops_cap, count * sizeof(OpRec));
  cudaError_t e = cudaSuccess;
  if (!rc) {
    // dense host rows -> padded device ciphertexts
    e = cudaMemset2DAsync(buf, ctb, 0, ctb, out0 + count, c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(buf, ctb, v1, dense, dense, n_left, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(buf + right0 * c->p.ct_words, ctb, v2, dense, dense, count,
                            cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(c->d_tmp_ops, ops.data(), count * sizeof(OpRec), cudaMemcpyHostToDevice,
                          c->stream);
    if (e == cudaSuccess) rc = launch_level(c, buf, c->d_tmp_ops, (uint32_t)count, 1);
    if (e == cudaSuccess && !rc && ring) {
      complement_rows_kernel<<<grid_for(count * c->p.words, c->num_sms), 256, 0, c->stream>>>(
          buf + out0 * c->p.ct_words, count, c->p);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess && !rc)
      e = cudaMemcpy2DAsync(out, dense, buf + out0 * c->p.ct_words, ctb, dense, count,
                            cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess && !rc) e = cudaStreamSynchronize(c->stream);
  }
  cudaFree(buf);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(FHEGPU_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return FHEGPU_OK;
}

}  // namespace

int fhegpu_nand_batch(fhegpu_ctx *c, const uint32_t *v1, const uint32_t *v2, uint32_t *out,
                      uint64_t count) {
  return product_batch(c, v1, false, v2, out, count, false, "nand_batch");
}

int fhegpu_mult_batch(fhegpu_ctx *c, const uint32_t *v1, const uint32_t *v2, uint32_t *out,
                      uint64_t count) {
  return product_batch(c, v1, false, v2, out, count, true, "mult_batch");
}

int fhegpu_const_mult_batch(fhegpu_ctx *c, uint32_t k, const uint32_t *v, uint32_t *out, uint64_t count) {
  if (!c) return fail(FHEGPU_EINVAL, "null ctx");
  // left operand V_k = (k G) mod q: (k 2^j mod q) at row i*ell+j, column i (fhe.py:200-208)
  const uint32_t q = c->p.q, kk = k % q;
  std::vector<uint32_t> vk((size_t)c->p.words, 0u);
  for (uint32_t r = 0; r < c->p.rows; ++r) {
    const uint32_t i = r / c->p.ell, j = r % c->p.ell;
    vk[(size_t)r * c->p.k + i] = (uint32_t)(((uint64_t)kk << j) % q);
  }
  return product_batch(c, vk.data(), true, v, out, count, true, "const_mult_batch");
}

int fhegpu_add_batch(fhegpu_ctx *c, const uint32_t *v1, const uint32_t *v2, uint32_t *out,
                     uint64_t count) {
  if (!c || (count && (!v1 || !v2 || !out))) return fail(FHEGPU_EINVAL, "null argument");
  if (count == 0) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t per = (size_t)c->p.words * 4;
  uint32_t *buf = nullptr;
  CUDA_TRY(cudaMalloc(&buf, 3 * count * per));
  cudaError_t e = cudaMemcpyAsync(buf, v1, count * per, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(buf + count * c->p.words, v2, count * per, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) {
    add_kernel<<<grid_for(count * c->p.words, c->num_sms), 256, 0, c->stream>>>(
        buf, buf + count * c->p.words, buf + 2 * count * c->p.words, count, c->p);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, buf + 2 * count * c->p.words, count * per, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(buf);
  if (e != cudaSuccess) return fail(FHEGPU_ECUDA, std::string("add_batch: ") + cudaGetErrorString(e));
  return FHEGPU_OK;
}

int fhegpu_not_batch(fhegpu_ctx *c, const uint32_t *v, uint32_t *out, uint64_t count) {
  if (!c || (count && (!v || !out))) return fail(FHEGPU_EINVAL, "null argument");
  if (count == 0) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t per = (size_t)c->p.words * 4;
  uint32_t *buf = nullptr;
  CUDA_TRY(cudaMalloc(&buf, 2 * count * per));
  cudaError_t e = cudaMemcpyAsync(buf, v, count * per, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) {
    complement_kernel<<<grid_for(count * c->p.words, c->num_sms), 256, 0, c->stream>>>(
        buf, buf + count * c->p.words, count, c->p);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, buf + count * c->p.words, count * per, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(buf);
  if (e != cudaSuccess) return fail(FHEGPU_ECUDA, std::string("not_batch: ") + cudaGetErrorString(e));
  return FHEGPU_OK;
}

int fhegpu_encrypt(fhegpu_ctx *c, const uint32_t *pk, const fhegpu_pcg64 *streams, uint32_t n_streams,
                   const uint32_t *stream_idx, const uint64_t *u32_offset, const uint32_t *mu,
                   const uint64_t *target, uint64_t count) {
  if (!c || (count && (!pk || !streams || !stream_idx || !u32_offset || !mu || !target)))
    return fail(FHEGPU_EINVAL, "null argument");
  if (count == 0) return FHEGPU_OK;
  if (c->m == 0 || c->m > 4096) return fail(FHEGPU_EINVAL, "bad m");
  for (uint64_t e = 0; e < count; ++e) {
    if (stream_idx[e] >= n_streams) return fail(FHEGPU_EINVAL, "stream index out of range");
    if (target[e] >= c->capacity) return fail(FHEGPU_EINVAL, "encrypt target beyond store capacity");
    if (mu[e] >= c->p.q) return fail(FHEGPU_EINVAL, "plaintext must be < q");
  }
  for (uint32_t i = 0; i < c->m * c->p.k; ++i)
    if (pk[i] >= c->p.q) return fail(FHEGPU_EINVAL, "public key entries must be < q");
  for (uint32_t i = 0; i < n_streams; ++i)
    if ((streams[i].inc_lo & 1u) == 0) return fail(FHEGPU_EINVAL, "PCG64 increment must be odd");
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->d_jump) {
    JumpTable h;
    const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    u128 a = mult, g = 1;
    for (int j = 0; j < 64; ++j) {
      h.a[j] = a;
      h.g[j] = g;
      g = g * (a + 1);
      a = a * a;
    }
    CUDA_TRY(cudaMalloc(&c->d_jump, sizeof(JumpTable)));
    CUDA_TRY(cudaMemcpy(c->d_jump, &h, sizeof(JumpTable), cudaMemcpyHostToDevice));
  }
  // one staging allocation: streams | stream_idx | offsets | mu | target | pk
  const size_t b_str = (size_t)n_streams * sizeof(StreamRec), b_idx = count * 4, b_off = count * 8,
               b_mu = count * 4, b_tgt = count * 8, b_pk = (size_t)c->m * c->p.k * 4;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t total = al(b_str) + al(b_idx) + al(b_off) + al(b_mu) + al(b_tgt) + al(b_pk);
  uint8_t *buf = nullptr;
  CUDA_TRY(cudaMalloc(&buf, total));
  uint8_t *q = buf;
  auto put = [&](const void *src, size_t n) {
    uint8_t *dst = q;
    cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, c->stream);
    q += al(n);
    return dst;
  };
  auto *d_str = (const StreamRec *)put(streams, b_str);
  auto *d_idx = (const uint32_t *)put(stream_idx, b_idx);
  auto *d_off = (const uint64_t *)put(u32_offset, b_off);
  auto *d_mu = (const uint32_t *)put(mu, b_mu);
  auto *d_tgt = (const uint64_t *)put(target, b_tgt);
  auto *d_pk = (const uint32_t *)put(pk, b_pk);
  const uint64_t work = count * c->p.rows;
  encrypt_kernel<<<grid_for(work, c->num_sms), 256, b_pk, c->stream>>>(
      c->store, c->d_jump, d_str, d_idx, d_off, d_mu, d_tgt, d_pk, count, c->m, c->p);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(buf);
  if (e != cudaSuccess) return fail(FHEGPU_ECUDA, std::string("encrypt: ") + cudaGetErrorString(e));
  return FHEGPU_OK;
}

// Debug: copy the warp-specialised kernel's timeline probe (64 x 16 clock64 values).
int fhegpu_debug_ws_trace(uint64_t *host) {
  if (!host) return fail(FHEGPU_EINVAL, "null argument");
  CUDA_TRY(cudaMemcpyFromSymbol(host, tc::g_ws_trace, sizeof(uint64_t) * 64 * 16));
  return FHEGPU_OK;
}

// Debug: copy the warp-dataflow kernel's per-gate probe (12 u32 per gate; -DFHEGPU_TRACE=1 builds).
int fhegpu_debug_flow_trace(uint32_t *host, uint32_t n_gates) {
  if (!host) return fail(FHEGPU_EINVAL, "null argument");
  if (n_gates > flow::FLOW_TRACE_GATES) return fail(FHEGPU_EUNSUP, "not a trace build");
  CUDA_TRY(cudaMemcpyFromSymbol(host, flow::g_flow_trace, sizeof(uint32_t) * flow::FLOW_TRACE_WORDS * n_gates));
  return FHEGPU_OK;
}

// -- bitsliced cleartext engine (CleartextEngine twin, engine.py:69-121) -----------------------

struct fhegpu_bits {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  uint64_t lanes = 0;
  uint32_t words = 0;        // u32 words per wire
  uint32_t tail_mask = 0;    // valid lane bits of the last word
  uint32_t *store = nullptr;
  uint64_t capacity = 0;     // wires
  OpRec *d_ops = nullptr;
  size_t ops_cap = 0;
  uint64_t *d_slots = nullptr;
  size_t slots_cap = 0;
  uint32_t *d_io = nullptr;
  size_t io_cap = 0;
  uint8_t *d_comp = nullptr;
  size_t comp_cap = 0;
};

int fhegpu_bits_create(int device, uint64_t lanes, fhegpu_bits **out) {
  if (!out) return fail(FHEGPU_EINVAL, "null argument");
  *out = nullptr;
  if (lanes == 0 || lanes > (uint64_t(1) << 36)) return fail(FHEGPU_EINVAL, "lanes must be in [1, 2^36]");
  CUDA_TRY(cudaSetDevice(device));
  auto *b = new fhegpu_bits();
  b->device = device;
  b->lanes = lanes;
  b->words = (uint32_t)((lanes + 31) / 32);
  b->tail_mask = (lanes % 32) ? ((1u << (lanes % 32)) - 1u) : 0xFFFFFFFFu;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete b;
    return fail(FHEGPU_ECUDA, std::string("bits_create: ") + cudaGetErrorString(e));
  }
  b->num_sms = prop.multiProcessorCount;
  *out = b;
  return FHEGPU_OK;
}

void fhegpu_bits_destroy(fhegpu_bits *b) {
  if (!b) return;
  cudaSetDevice(b->device);
  cudaStreamSynchronize(b->stream);
  cudaFree(b->store);
  cudaFree(b->d_ops);
  cudaFree(b->d_slots);
  cudaFree(b->d_io);
  cudaFree(b->d_comp);
  cudaStreamDestroy(b->stream);
  delete b;
}

uint32_t fhegpu_bits_words(const fhegpu_bits *b) { return b ? b->words : 0; }

int fhegpu_bits_reserve(fhegpu_bits *b, uint64_t wires) {
  if (!b) return fail(FHEGPU_EINVAL, "null handle");
  if (wires <= b->capacity) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(b->device));
  uint32_t *nw = nullptr;
  const size_t bytes = (size_t)wires * b->words * 4;
  if (cudaMalloc(&nw, bytes) != cudaSuccess) return fail(FHEGPU_ENOMEM, "bits_reserve: out of device memory");
  cudaError_t e = cudaMemsetAsync(nw, 0, bytes, b->stream);
  if (e == cudaSuccess && b->store)
    e = cudaMemcpyAsync(nw, b->store, b->capacity * b->words * 4, cudaMemcpyDeviceToDevice, b->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(b->stream);
  if (e != cudaSuccess) {
    cudaFree(nw);
    return fail(FHEGPU_ECUDA, std::string("bits_reserve: ") + cudaGetErrorString(e));
  }
  cudaFree(b->store);
  b->store = nw;
  b->capacity = wires;
  return FHEGPU_OK;
}

static int bits_check_slots(fhegpu_bits *b, const uint64_t *slots, uint64_t count) {
  for (uint64_t i = 0; i < count; ++i)
    if (slots[i] >= b->capacity) return fail(FHEGPU_EINVAL, "wire slot beyond capacity");
  return FHEGPU_OK;
}

int fhegpu_bits_write(fhegpu_bits *b, const uint64_t *slots, uint64_t count, const uint32_t *words) {
  if (!b || (count && (!slots || !words))) return fail(FHEGPU_EINVAL, "null argument");
  if (count == 0) return FHEGPU_OK;
  if (int rc = bits_check_slots(b, slots, count)) return rc;
  CUDA_TRY(cudaSetDevice(b->device));
  const size_t bytes = (size_t)count * b->words * 4;
  if (int rc = ensure((void **)&b->d_io, &b->io_cap, bytes)) return rc;
  if (int rc = ensure((void **)&b->d_slots, &b->slots_cap, count * 8)) return rc;
  CUDA_TRY(cudaMemcpyAsync(b->d_io, words, bytes, cudaMemcpyHostToDevice, b->stream));
  CUDA_TRY(cudaMemcpyAsync(b->d_slots, slots, count * 8, cudaMemcpyHostToDevice, b->stream));
  bits_scatter_kernel<<<grid_for(count * b->words, b->num_sms), 256, 0, b->stream>>>(b->store, b->d_slots,
                                                                                   b->d_io, count, b->words);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  return FHEGPU_OK;
}

int fhegpu_bits_run(fhegpu_bits *b, const fhegpu_op *ops, uint64_t n_ops, const uint64_t *level_offsets,
                    uint32_t n_levels) {
  if (!b || (n_ops && !ops) || !level_offsets) return fail(FHEGPU_EINVAL, "null argument");
  if (level_offsets[0] != 0 || level_offsets[n_levels] != n_ops)
    return fail(FHEGPU_EINVAL, "level offsets must span [0, n_ops]");
  for (uint64_t i = 0; i < n_ops; ++i) {
    const uint64_t mx = std::max(ops[i].left, std::max(ops[i].right, ops[i].out));
    if (mx >= b->capacity || (ops[i].flags & ~3u)) return fail(FHEGPU_EINVAL, "bad op record " + std::to_string(i));
  }
  if (n_ops == 0) return FHEGPU_OK;
  CUDA_TRY(cudaSetDevice(b->device));
  if (int rc = ensure((void **)&b->d_ops, &b->ops_cap, n_ops * sizeof(OpRec))) return rc;
  CUDA_TRY(cudaMemcpyAsync(b->d_ops, ops, n_ops * sizeof(OpRec), cudaMemcpyHostToDevice, b->stream));
  for (uint32_t l = 0; l < n_levels; ++l) {
    const uint64_t a = level_offsets[l], e = level_offsets[l + 1];
    if (e <= a) continue;
    const uint32_t n = (uint32_t)(e - a);
    bits_level_kernel<<<grid_for((uint64_t)n * b->words, b->num_sms), 256, 0, b->stream>>>(
        b->store, b->d_ops + a, n, b->words, b->tail_mask);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(b->stream));   // the op table is reused by the next call
  return FHEGPU_OK;
}

int fhegpu_bits_read(fhegpu_bits *b, const uint64_t *slots, const uint8_t *comp, uint64_t count,
                     uint32_t *words) {
  if (!b || (count && (!slots || !words))) return fail(FHEGPU_EINVAL, "null argument");
  if (count == 0) return FHEGPU_OK;
  if (int rc = bits_check_slots(b, slots, count)) return rc;
  CUDA_TRY(cudaSetDevice(b->device));
  const size_t bytes = (size_t)count * b->words * 4;
  if (int rc = ensure((void **)&b->d_io, &b->io_cap, bytes)) return rc;
  if (int rc = ensure((void **)&b->d_slots, &b->slots_cap, count * 8)) return rc;
  CUDA_TRY(cudaMemcpyAsync(b->d_slots, slots, count * 8, cudaMemcpyHostToDevice, b->stream));
  const uint8_t *dcomp = nullptr;
  if (comp) {
    if (int rc = ensure((void **)&b->d_comp, &b->comp_cap, count)) return rc;
    CUDA_TRY(cudaMemcpyAsync(b->d_comp, comp, count, cudaMemcpyHostToDevice, b->stream));
    dcomp = b->d_comp;
  }
  bits_gather_kernel<<<grid_for(count * b->words, b->num_sms), 256, 0, b->stream>>>(
      b->store, b->d_slots, dcomp, b->d_io, count, b->words, b->tail_mask);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(words, b->d_io, bytes, cudaMemcpyDeviceToHost, b->stream));
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  return FHEGPU_OK;
}

}  // extern "C"
