// tc_nand_resident.cuh -- lane-resident launches of small per-lane programs (the gate benchmark's
// XOR + AND, or any netlist of <= RES_MAX_OPS gates per lane whose outputs are its sinks).
//
// The level / dataflow launches move every operand through L2 (2 x 9.4 KB per gate) and every
// output back (9.4 KB): measured 1.55 uJ of the 4.6 uJ a gate costs above idle, at the board
// power limit that sets the throughput.  Here a CTA takes W lanes at a time and
// runs the whole per-lane program on them: the program's inputs are bulk-loaded once into an
// input set (released after the group's last input reader, so the next group's loads overlap
// the rest of this one), every gate's output is written by the epilogue straight into a
// shared-memory buffer of that lane (the operand of later gates), and only the program's
// outputs are stored.  cfg1: 2 loads + 2 stores per 6 gates instead of 11 + 6.  Four warps copy
// the B operands so the A builders, the pipeline's pacer, only build A.
//
// Pipeline roles, TMEM double buffers, MMA sequence, A/B operand construction and the fold are
// those of level_tc_ws_kernel (tc_nand_ws.cuh).  Slot t of a CTA is (group g, op o, lane w)
// with t = g * S + o * W + w, S = n_ops * W: gates of one op for the W lanes back to back, ops
// in the host's topological order, so a gate's producer is >= W slots earlier.  A builder
// reading a gate output waits on that gate's mbarrier (out_ready), which the epilogue arrives on
// once the output sits in its local buffer (one phase per lane group) -- unless the producer is
// >= 5 slots back, which the A-buffer handshake already implies (see the slot table setup).
// Timeline probes (trace_ev, -DFHEGPU_TRACE=1 builds only): tools/timeline_resident.py.
#pragma once

#include <climits>
#include <unordered_map>
#include <utility>

#include "tc_nand_ws.cuh"

namespace fhegpu {
namespace tc {

#ifndef FHEGPU_RES_W
#define FHEGPU_RES_W 3
#endif
#ifndef FHEGPU_RES_NSETS
#define FHEGPU_RES_NSETS 1
#endif
constexpr int RES_W = FHEGPU_RES_W;          // lanes per group
constexpr int RES_NSETS = FHEGPU_RES_NSETS;  // input sets (1: the next group's inputs load after
                                             // the group's last input reader)
constexpr int RES_MAX_OPS = 8;    // gates per lane program
constexpr int RES_MAX_IN = 4;     // program inputs
constexpr int RES_MAX_LOCAL = 8;  // per-lane shared-memory ciphertext buffers

// One gate of the per-lane program (16 bytes, same layout as fhegpu_res_op).
struct ResOp {
  uint8_t lkind, lidx, rkind, ridx;  // operand source: kind 0 = program input idx, 1 = local buffer idx
  uint8_t dest, is_out, flags, pad;  // local buffer written; 1: also stored to out_slot; complements
  int16_t lprod, rprod;              // plan index of the gate producing a local operand (-1: input)
  uint32_t out_slot;                 // store slot of a program output
};

#ifndef FHEGPU_RES_HINT
#define FHEGPU_RES_HINT 0    // 1: program inputs and outputs move with an L2 evict_first policy
#endif

__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Slot order of a group (host side, fhegpu_prog_set_resident): the W * n_ops slots (gate o of
// lane w) in the order the CTA runs them, one byte each: o | w << 3 | 32 (left operand reused) |
// 64 (right operand reused).  Slot t runs in TMEM / B buffer t & 1, so a gate placed two slots
// after its lane's previous gate finds that gate's A (TMEM) and B (shared memory) operands still
// in its buffers: an identical left operand (same source, same complement) rebuilds only the
// A columns the tail accumulator overwrote, an identical right operand skips the B copy.  A
// local operand produced fewer than 5 slots back costs a wait on its producer's epilogue, an
// output gate right after its lane's output gate into the same buffer an epilogue barrier.  The
// order maximises reuse (left 3, right 1) minus 4 per such wait (2 per barrier) over all orders
// that keep each lane's gates in plan order: exhaustive search over (per-lane progress, last 4
// slots), memoised (W * n_ops <= 24 slots).
struct ResSlotOrder {
  const ResOp *plan;
  int n, W;
  int same_l[RES_MAX_OPS], same_r[RES_MAX_OPS];
  std::unordered_map<uint64_t, std::pair<int, int>> memo;   // state -> (best score, lane taken)

  static bool same_src(const ResOp &a, const ResOp &b, bool left) {
    const uint8_t ka = left ? a.lkind : a.rkind, kb = left ? b.lkind : b.rkind;
    const uint32_t ia = ka ? (uint32_t)(left ? a.lprod : a.rprod) : (left ? a.lidx : a.ridx);
    const uint32_t ib = kb ? (uint32_t)(left ? b.lprod : b.rprod) : (left ? b.lidx : b.ridx);
    const uint32_t m = left ? 1u : 2u;
    return ka == kb && ia == ib && (a.flags & m) == (b.flags & m);
  }
  // state: progress of each lane (4 bits) | last 4 slots (6 bits each: 0 none, else 1 + o + 8 w)
  static uint64_t key(const int *prog, int W, const int *last) {
    uint64_t k = 0;
    for (int w = 0; w < W; ++w) k = (k << 4) | (uint64_t)prog[w];
    for (int i = 0; i < 4; ++i) k = (k << 6) | (uint64_t)last[i];
    return k;
  }
  int gain(int o, int w, const int *last, bool *ra, bool *rb) const {
    int s = 0;
    *ra = *rb = false;
    if (o > 0 && last[1] == 1 + (o - 1) + 8 * w) {
      *ra = same_l[o];
      *rb = same_r[o];
      s += 3 * same_l[o] + same_r[o];
    }
    const ResOp &op = plan[o];
    if (last[0] > 0) {                             // store hazard (an epilogue barrier): avoid
      const int po = (last[0] - 1) & 7, pw = (last[0] - 1) >> 3;
      if (pw == w && op.is_out && plan[po].is_out && plan[po].dest == op.dest) s -= 2;
    }
    for (int side = 0; side < 2; ++side) {
      const int kind = side ? op.rkind : op.lkind, prod = side ? op.rprod : op.lprod;
      if (!kind) continue;
      for (int i = 0; i < 4; ++i)
        if (last[i] == 1 + prod + 8 * w) s -= 4;
    }
    return s;
  }
  int best(int *prog, int *last, int left) {
    if (left == 0) return 0;
    const uint64_t k = key(prog, W, last);
    auto it = memo.find(k);
    if (it != memo.end()) return it->second.first;
    int bs = INT32_MIN, bw = -1;
    for (int w = 0; w < W; ++w) {
      const int o = prog[w];
      if (o >= n) continue;
      bool ra, rb;
      const int g = gain(o, w, last, &ra, &rb);
      int nl[4] = {1 + o + 8 * w, last[0], last[1], last[2]};
      ++prog[w];
      const int sc = g + best(prog, nl, left - 1);
      --prog[w];
      if (sc > bs) bs = sc, bw = w;
    }
    memo.emplace(k, std::make_pair(bs, bw));
    return bs;
  }
  // any local operand produced fewer than 5 slots back (else the kernel compiles its waits out)
  static bool near_deps(const ResOp *p, int n_ops, int lanes, const uint8_t *order) {
    int pos[RES_MAX_OPS][4];
    for (int t = 0; t < n_ops * lanes; ++t) pos[order[t] & 7][(order[t] >> 3) & 3] = t;
    for (int t = 0; t < n_ops * lanes; ++t) {
      const ResOp &op = p[order[t] & 7];
      const int w = (order[t] >> 3) & 3;
      if ((op.lkind && t - pos[op.lprod][w] < 5) || (op.rkind && t - pos[op.rprod][w] < 5)) return true;
    }
    return false;
  }
  void run(const ResOp *p, int n_ops, int lanes, uint8_t *order) {
    plan = p, n = n_ops, W = lanes;
    for (int o = 0; o < n; ++o) {
      same_l[o] = o > 0 && same_src(p[o], p[o - 1], true);
      same_r[o] = o > 0 && same_src(p[o], p[o - 1], false);
    }
    int prog[4] = {0, 0, 0, 0}, last[4] = {0, 0, 0, 0};
    best(prog, last, n * W);
    for (int t = 0; t < n * W; ++t) {
      const int w = memo.at(key(prog, W, last)).second, o = prog[w];
      bool ra, rb;
      gain(o, w, last, &ra, &rb);
      order[t] = (uint8_t)(o | (w << 3) | (ra ? 32 : 0) | (rb ? 64 : 0));
      ++prog[w];
      for (int i = 3; i > 0; --i) last[i] = last[i - 1];
      last[0] = 1 + o + 8 * w;
    }
  }
};

// A operand of one row, words [W0, W1): bits -> K slots, tcgen05.st into TMEM (4 words = one
// 32-column store, a remainder word = one 8-column store).
template <int K, int W0, int W1, int ENC>
__device__ __forceinline__ void build_a_words(const uint32_t *v1, int row, int row_blk, int row_bit, bool comp,
                                              uint32_t q, uint32_t a_addr) {
  uint32_t words[W1 - W0];
#pragma unroll
  for (int i = W0; i < W1; ++i) words[i - W0] = v1[row * K + i];
  if (comp) {
#pragma unroll
    for (int i = W0; i < W1; ++i) words[i - W0] = sub_mod(i == row_blk ? (1u << row_bit) : 0u, words[i - W0], q);
  }
#pragma unroll
  for (int w0 = W0; w0 < W1; w0 += 4) {
    if (w0 + 4 <= W1) {
      uint32_t sp[32];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t one[8];
        spread_word_sr<ENC>(words[w0 + j - W0], one);
#pragma unroll
        for (int x = 0; x < 8; ++x) sp[8 * j + x] = one[x];
      }
      tmem_st32(a_addr + 8 * w0, sp);
    } else {
#pragma unroll
      for (int w = w0; w < W1; ++w) {
        uint32_t sp[8];
        spread_word_sr<ENC>(words[w - W0], sp);
        tmem_st8(a_addr + 8 * w, sp);
      }
    }
  }
}

template <int K, int ELL>
struct GeoRes {
  using W = GeoWS<K, ELL, true, 1, false>;
  using B = Geo<K, ELL>;
  static constexpr int CT_BYTES = B::CT_BYTES, CT_WORDS = B::CT_WORDS;
  static constexpr int B_BYTES = B::B_BYTES;
  static constexpr int TA_BYTES = B::TA_BYTES;   // one 8-row tail group, aliased over M (SBO 0)
  static constexpr int N_OUT = 3;
#ifndef FHEGPU_RES_EPI_SPLIT
#define FHEGPU_RES_EPI_SPLIT 1   // 2: 16 epilogue warps (72 registers: slower, measured)
#endif
  // epilogue warps: 8 x SPLIT (SPLIT = 2: two threads per row, values 0-4 and 5-8)
#ifndef FHEGPU_RES_BSPLIT
#define FHEGPU_RES_BSPLIT 1    // 2: two builder threads per A row (words 0-3 / 4-8)
#endif
  static constexpr int EPI_SPLIT = FHEGPU_RES_EPI_SPLIT;
  static constexpr int BSPLIT = FHEGPU_RES_BSPLIT;
  static constexpr int NE_WARPS = 8 * EPI_SPLIT;
#ifndef FHEGPU_RES_BCOPY_WARPS
#define FHEGPU_RES_BCOPY_WARPS 4   // warps that copy the B operand (0: the A builders do it too)
#endif
  static constexpr int NB_WARPS = 4 * W::MT * BSPLIT;
  static constexpr int NBC_WARPS = FHEGPU_RES_BCOPY_WARPS;
  static constexpr int WARP_BC0 = 3 + NB_WARPS;
  static constexpr int WARP_EPI0 = WARP_BC0 + NBC_WARPS;
  static constexpr int THREADS = 32 * (3 + NB_WARPS + NBC_WARPS + NE_WARPS);
  static constexpr int OFF_BAR_SIZE = 64 * 8;
  // runtime layout (host computes the same): inputs | locals | B x 2 | TA x 2 | barriers | plan
  __host__ __device__ static uint32_t off_local(uint32_t n_in) { return RES_NSETS * RES_W * n_in * CT_BYTES; }
  __host__ __device__ static uint32_t off_b(uint32_t n_in, uint32_t n_local) {
    return ((off_local(n_in) + RES_W * n_local * CT_BYTES + 127u) / 128u) * 128u;
  }
  __host__ __device__ static uint32_t off_ta(uint32_t n_in, uint32_t n_local) {
    return off_b(n_in, n_local) + 2u * B_BYTES;
  }
  __host__ __device__ static uint32_t off_bar(uint32_t n_in, uint32_t n_local) {
    return ((off_ta(n_in, n_local) + 2u * TA_BYTES + 127u) / 128u) * 128u;
  }
  __host__ __device__ static uint32_t smem_bytes(uint32_t n_in, uint32_t n_local) {
    return off_bar(n_in, n_local) + OFF_BAR_SIZE + RES_MAX_OPS * sizeof(ResOp) +
           RES_MAX_OPS * RES_W * 16u + 32u;
  }
};

// Position of slot t in its group, advanced incrementally (no runtime divisions per slot).
struct SlotPos {
  uint32_t g = 0, r = 0, o = 0, w = 0, gS = 0;   // group, slot in group, gate, lane, group's first slot
  __device__ __forceinline__ void next(uint32_t S, uint32_t W) {
    if (++w == W) {
      w = 0;
      ++o;
    }
    if (++r == S) {
      r = 0;
      o = 0;
      ++g;
      gS += S;
    }
  }
};

// Per slot of a group (r = o * W + w), precomputed once per CTA: operand / destination buffer
// indices (ciphertext units; inputs relative to their set), flags, and the RAW dependency.
struct __align__(16) SlotInfo {
  uint32_t v1, v2;         // left / right operand buffer (ciphertext words offset)
  uint32_t dest;           // destination local buffer (ciphertext words offset)
  uint8_t dep_l, dep_r;    // out_ready index (o * W + w) of a local operand's producer (0xFF: input)
  uint8_t bits;            // 1, 2: complement left / right; 4: output gate; 8 / 16: left / right local;
                           // 32: the group's last input-reading slot; 64 / 128: left / right
                           // operand reused from slot t - 2 (ResSlotOrder)
  uint8_t ow;              // gate | lane << 3 | 32 (store hazard on the previous slot)
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t *v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}

__device__ __forceinline__ void bulk_wait_read_dyn(uint32_t n) {
  switch (n) {   // cp.async.bulk.wait_group.read takes an immediate
    case 0: bulk_wait_read_n<0>(); break;
    case 1: bulk_wait_read_n<1>(); break;
    case 2: bulk_wait_read_n<2>(); break;
    case 3: bulk_wait_read_n<3>(); break;
    case 4: bulk_wait_read_n<4>(); break;
    case 5: bulk_wait_read_n<5>(); break;
    case 6: bulk_wait_read_n<6>(); break;
    default: bulk_wait_read_n<7>(); break;
  }
}

template <int K, int ELL, bool PM, int ENC, bool DEPS>
__global__ void __launch_bounds__(GeoRes<K, ELL>::THREADS, 1)
resident_tc_kernel(uint32_t *__restrict__ store, const ResOp *__restrict__ plan, const uint32_t *__restrict__ in_slots,
                   uint32_t n_ops, uint32_t n_in, uint32_t n_local, uint32_t n_out, uint32_t lanes,
                   uint32_t n_groups, DevParams p) {
  using R = GeoRes<K, ELL>;
  using G = GeoWS<K, ELL, PM, ENC, false>;       // roles, TMEM columns, MMA descriptors
  constexpr int W = RES_W;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t *s_inb = reinterpret_cast<uint32_t *>(smem);
  uint32_t *s_loc = reinterpret_cast<uint32_t *>(smem + R::off_local(n_in));
  uint8_t *s_b = smem + R::off_b(n_in, n_local);
  uint8_t *s_ta = smem + R::off_ta(n_in, n_local);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + R::off_bar(n_in, n_local));
  uint64_t *in_full = bar;                  // [2] input set loaded
  uint64_t *in_empty = bar + 2;             // [2] input set read by every gate of its group
  uint64_t *op_full = bar + 4;              // [2]
  uint64_t *main_done = bar + 6;            // [2]
  uint64_t *a_free = bar + 8;               // [2]
  uint64_t *d_free = bar + 10;              // [2]
  uint64_t *out_free = bar + 12;            // [N_OUT] tail rows of slot t may be written
  uint64_t *tail_ready = bar + 12 + R::N_OUT;
  uint64_t *out_ready = bar + 12 + 2 * R::N_OUT;           // [RES_MAX_OPS * W] gate output in its buffer
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(out_ready + RES_MAX_OPS * RES_W);
  ResOp *s_plan = reinterpret_cast<ResOp *>(smem + R::off_bar(n_in, n_local) + R::OFF_BAR_SIZE);
  SlotInfo *s_slot = reinterpret_cast<SlotInfo *>(s_plan + RES_MAX_OPS);   // 16-byte aligned

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t S = n_ops * W;                                     // slots per group
  const uint32_t my_groups = blockIdx.x < n_groups ? (n_groups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t n_slots = my_groups * S;
  auto lane_of_group = [&](uint32_t g, uint32_t w) { return (g * gridDim.x + blockIdx.x) * W + w; };
  auto in_ptr = [&](uint32_t set, uint32_t w, uint32_t i) {
    return s_inb + ((set * W + w) * n_in + i) * R::CT_WORDS;
  };

  if (warp == G::WARP_MMA) tmem_alloc<512>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&in_full[i], 1);
      mbar_init(&in_empty[i], R::NB_WARPS + R::NBC_WARPS);
      mbar_init(&op_full[i], R::NB_WARPS + R::NBC_WARPS);
      mbar_init(&main_done[i], 1);
      mbar_init(&a_free[i], 1);
      mbar_init(&d_free[i], R::NE_WARPS);
    }
    for (int i = 0; i < R::N_OUT; ++i) {
      mbar_init(&out_free[i], 1);
      mbar_init(&tail_ready[i], 1);
    }
    for (int i = 0; i < RES_MAX_OPS * W; ++i) mbar_init(&out_ready[i], 1);
    fence_mbar_init();
  }
  for (uint32_t i = tid; i < n_ops * (sizeof(ResOp) / 4); i += R::THREADS)
    reinterpret_cast<uint32_t *>(s_plan)[i] = reinterpret_cast<const uint32_t *>(plan)[i];
  // slot order (ResSlotOrder), stored after the plan
  const uint8_t *order = reinterpret_cast<const uint8_t *>(plan + n_ops);
  if (tid < S) {
    const uint32_t code = order[tid];
    const uint32_t o = code & 7u, w = (code >> 3) & 3u;
    const ResOp op = plan[o];
    SlotInfo si;
    si.v1 = (op.lkind ? w * n_local + op.lidx : w * n_in + op.lidx) * R::CT_WORDS;
    si.v2 = (op.rkind ? w * n_local + op.ridx : w * n_in + op.ridx) * R::CT_WORDS;
    si.dest = (w * n_local + op.dest) * R::CT_WORDS;
    uint32_t in_last = 0, slot_l = 0, slot_r = 0;  // last input-reading slot; producers' slots
    for (uint32_t r = 0; r < S; ++r) {
      const uint32_t c = order[r] & 31u;
      if (plan[c & 7u].lkind == 0 || plan[c & 7u].rkind == 0) in_last = r;
      if (op.lkind && c == ((uint32_t)op.lprod | w << 3)) slot_l = r;
      if (op.rkind && c == ((uint32_t)op.rprod | w << 3)) slot_r = r;
    }
    const bool reuse = !(p.dbg & (1u << 20));       // dbg bit 20: no operand reuse
    si.bits = (op.flags & 3u) | (op.is_out ? 4u : 0u) | (op.lkind ? 8u : 0u) | (op.rkind ? 16u : 0u) |
              (tid == in_last ? 32u : 0u) | (reuse && (code & 32u) ? 64u : 0u) |
              (reuse && (code & 64u) ? 128u : 0u);
    // store hazard: the previous slot is an output gate of the same lane writing the same buffer,
    // so this gate's writes must wait for that slot's store to have read it (epilogue, below)
    const uint32_t prev = order[(tid + S - 1) % S];
    const bool hazard = op.is_out && plan[prev & 7u].is_out && ((prev >> 3) & 3u) == w &&
                        plan[prev & 7u].dest == op.dest;
    si.ow = (uint8_t)((code & 31u) | (hazard ? 32u : 0u));
    // A producer >= 5 slots back needs no wait: the builder's a_free wait for slot t implies
    // main_done(t-2), hence the MMA of t-2 was issued after d_free(t-4), which every epilogue
    // warp arrives on only after finishing slot t-5 (outputs written, out_ready published).
    // (dbg bit 21, with the DEPS instantiation: wait on every local producer -- parity tests of
    // the rule above)
    const uint32_t near = (p.dbg & (1u << 21)) ? S : 5u;
    si.dep_l = op.lkind && tid - slot_l < near ? (uint8_t)slot_l : (uint8_t)0xFF;
    si.dep_r = op.rkind && tid - slot_r < near ? (uint8_t)slot_r : (uint8_t)0xFF;
    s_slot[tid] = si;
  }
  for (uint32_t w = tid; w < 2 * R::B_BYTES / 4; w += R::THREADS) reinterpret_cast<uint32_t *>(s_b)[w] = 0u;
  for (uint32_t w = tid; w < 2 * R::TA_BYTES / 4; w += R::THREADS) reinterpret_cast<uint32_t *>(s_ta)[w] = 0u;
  // ciphertext padding words of every local buffer stay zero (the epilogue writes N * K words)
  for (uint32_t w = tid; w < W * n_local * R::CT_WORDS; w += R::THREADS) s_loc[w] = 0u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == G::WARP_PROD) {
    // ------------------------------ producer: program inputs, one group ahead ------------------------------
    if (lane == 0) {
      for (uint32_t g = 0; g < my_groups; ++g) {
        const uint32_t set = RES_NSETS == 2 ? g & 1u : 0u, ph = RES_NSETS == 2 ? g >> 1 : g;
        mbar_wait(&in_empty[set], (ph & 1u) ^ 1u);
        const uint32_t ln0 = lane_of_group(g, 0);
        const uint32_t valid = min((uint32_t)W, lanes - ln0);      // the last group may be partial
        mbar_expect_tx(&in_full[set], valid * n_in * R::CT_BYTES);
        for (uint32_t w = 0; w < valid; ++w) {
          const uint32_t ln = ln0 + w;
          for (uint32_t i = 0; i < n_in; ++i)
            if (FHEGPU_RES_HINT)
              bulk_g2s_hint(in_ptr(set, w, i), store + ((uint64_t)in_slots[i] * lanes + ln) * R::CT_WORDS,
                            R::CT_BYTES, &in_full[set], policy_evict_first());
            else
              bulk_g2s(in_ptr(set, w, i), store + ((uint64_t)in_slots[i] * lanes + ln) * R::CT_WORDS, R::CT_BYTES,
                       &in_full[set]);
        }
      }
    }
  } else if (warp == G::WARP_MMA) {
    // ------------------------------ MMA issuer (as level_tc_ws_kernel) ------------------------------
    const uint64_t bdesc0 = smem_desc(smem_u32(s_b), G::LBO, G::SBO);
    const uint64_t tdesc0 = smem_desc(smem_u32(s_ta), G::TA_LBO, 0u);
    for (uint32_t t = 0; t < n_slots; ++t) {
      const uint32_t b = t & 1u, u = t >> 1;
      mbar_wait(&op_full[b], u & 1u);
      if (lane == 0) trace_ev(p, t, 2);
      mbar_wait(&d_free[b], (u & 1u) ^ 1u);
      if (lane == 0) trace_ev(p, t, 3);
      tc_fence_after();
      const uint32_t tb = tmem_base + b * G::BUF_COLS;
      const uint64_t bd_b = bdesc0 + ((b * R::B_BYTES) >> 4);
      const uint64_t td_b = tdesc0 + ((b * R::TA_BYTES) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int mt = 0; mt < G::MT; ++mt) {
#pragma unroll
          for (int s = 0; s < K; ++s)
            mma_i8_ts(tb + mt * G::NPAD, tb + G::D_COLS + mt * 8 * K + 8 * s, bd_b + ((s * 4 * G::LBO) >> 4),
                      G::IDESC, s > 0 ? 1u : 0u);
        }
        if constexpr (G::TAIL > 0) {
#pragma unroll
          for (int s = 0; s < K; ++s)
            mma_i8_ss(tb + G::D_COLS, td_b + ((s * 2 * G::TA_LBO) >> 4), bd_b + ((s * 4 * G::LBO) >> 4),
                      G::IDESC_TAIL, s > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
      if (elect_one()) mma_commit(&main_done[b]);
      __syncwarp();
      if (lane == 0) trace_ev(p, t, 4);
    }
  } else if (warp == G::WARP_TAIL) {
    // ------------------------------ tail rows, into the gate's local buffer ------------------------------
    if constexpr (G::TAIL > 0) {
      SlotPos pos;
      for (uint32_t t = 0; t < n_slots; ++t, pos.next(S, W)) {
        const uint32_t b = t & 1u, u = t >> 1;
        mbar_wait(&main_done[b], u & 1u);
        if (lane == 0) trace_ev(p, t, 12);
        tc_fence_after();
        uint32_t d[36];
        load_acc36(tmem_base + b * G::BUF_COLS + G::D_COLS, d, false);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_free[b]);
        const uint32_t ob = t % R::N_OUT, ou = t / R::N_OUT;
        mbar_wait(&out_free[ob], ou & 1u);
        if (lane == 0) trace_ev(p, t, 13);
        uint32_t *out_st = s_loc + s_slot[pos.r].dest;
        if (lane < G::TAIL) {
          const int row = G::MMA_ROWS + lane;
          const int rb = row / ELL, rbit = row - rb * ELL;
#pragma unroll
          for (int i = 0; i < K; ++i) out_st[row * K + i] = finish_neg<ELL, PM, ENC>(&d[i * 4], i == rb ? (1u << rbit) : 0u, p);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tail_ready[ob]);
        if (lane == 0) trace_ev(p, t, 14);
      }
    }
  } else if (warp >= R::WARP_BC0 && warp < R::WARP_EPI0) {
    // ------------------------------ B operand copiers ------------------------------
    // V2 rows into the MN-major canonical layout (digits = the value's bytes), off the A
    // builders' critical path (measured: the builders pace the resident pipeline)
    const int bc = tid - 32 * R::WARP_BC0;
    constexpr int NBT = 32 * (R::NBC_WARPS > 0 ? R::NBC_WARPS : 1);
    constexpr int B_ROWS = (G::KB + NBT - 1) / NBT;
    int b_src[B_ROWS], b_dst[B_ROWS], b_w[B_ROWS], b_j[B_ROWS];
#pragma unroll
    for (int x = 0; x < B_ROWS; ++x) {
      const int kr = bc + x * NBT;
      const int ww = kr >> 5, kk = kr & 31;
      const int j = 8 * (kk & 3) + (kk >> 2);
      b_src[x] = kr < G::KB && j < ELL ? (ww * ELL + j) * K : -1;
      b_dst[x] = (kr >> 3) * G::LBO + (kr & 7) * 16;
      b_w[x] = ww;
      b_j[x] = j;
    }
    SlotPos pos;
    const uint32_t in_set_words = W * n_in * R::CT_WORDS;
    for (uint32_t t = 0; t < n_slots; ++t, pos.next(S, W)) {
      const uint32_t g = pos.g, r = pos.r;
      const uint32_t set = RES_NSETS == 2 ? g & 1u : 0u, ph = RES_NSETS == 2 ? g >> 1 : g;
      const uint32_t b = t & 1u, u = t >> 1;
      if (r == 0) mbar_wait(&in_full[set], ph & 1u);
      const SlotInfo si = s_slot[r];
      mbar_wait(&a_free[b], (u & 1u) ^ 1u);        // B(b) was last read by the MMAs of slot t - 2
      if (DEPS && si.dep_r != 0xFF) mbar_wait(&out_ready[si.dep_r], g & 1u);
      const uint32_t *v2 = ((si.bits & 16u) ? s_loc : s_inb + set * in_set_words) + si.v2;
      const bool comp2 = si.bits & 2u;
      uint8_t *bb = s_b + b * R::B_BYTES;
#pragma unroll
      for (int x = 0; x < ((si.bits & 128u) ? 0 : B_ROWS); ++x) {   // reuse: B(b) holds this B
        if (b_src[x] < 0) continue;
        uint32_t vals[K];
#pragma unroll
        for (int i = 0; i < K; ++i) vals[i] = v2[b_src[x] + i];
        if (comp2) {
#pragma unroll
          for (int i = 0; i < K; ++i) vals[i] = sub_mod(i == b_w[x] ? (1u << b_j[x]) : 0u, vals[i], p.q);
        }
        uint8_t *dst = bb + b_dst[x];
#pragma unroll
        for (int ch = 0; ch < G::NCH; ++ch) {
          uint4 val;
          val.x = 4 * ch + 0 < K ? vals[4 * ch + 0] : 0u;
          val.y = 4 * ch + 1 < K ? vals[4 * ch + 1] : 0u;
          val.z = 4 * ch + 2 < K ? vals[4 * ch + 2] : 0u;
          val.w = 4 * ch + 3 < K ? vals[4 * ch + 3] : 0u;
          *reinterpret_cast<uint4 *>(dst + ch * G::SBO) = val;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&op_full[b]);
        if (si.bits & 32u) mbar_arrive(&in_empty[set]);
      }
    }
  } else if (warp < R::WARP_EPI0) {
    // ------------------------------ operand builders ------------------------------
    const int bt = tid - 32 * G::WARP_BUILD0;
    const int bw = bt >> 5;
    const int quad = warp & 3;
    const int tile = (bw >> 2) % G::MT;
    const int part = (bw >> 2) / G::MT;          // BSPLIT = 2: words 0-3 (part 0) or 4-8 (part 1)
    const int row = 128 * tile + 32 * quad + lane;
    const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
    const int row_blk = row / ELL, row_bit = row - row_blk * ELL;
    constexpr int NBT = 128 * G::MT * R::BSPLIT;
    const int tb = R::BSPLIT == 1 ? bt : bt - 128 * G::MT;   // tail-A thread index (part 1)
    constexpr int B_ROWS = (G::KB + NBT - 1) / NBT;
    int b_src[B_ROWS], b_dst[B_ROWS], b_w[B_ROWS], b_j[B_ROWS];
#pragma unroll
    for (int x = 0; x < B_ROWS; ++x) {
      const int kr = bt + x * NBT;
      const int ww = kr >> 5, kk = kr & 31;
      const int j = 8 * (kk & 3) + (kk >> 2);
      const bool ok = kr < G::KB && j < ELL;
      b_src[x] = ok ? (ww * ELL + j) * K : -1;
      b_dst[x] = (kr >> 3) * G::LBO + (kr & 7) * 16;
      b_w[x] = ww;
      b_j[x] = j;
    }
    SlotPos pos;
    const uint32_t in_set_words = W * n_in * R::CT_WORDS;
    for (uint32_t t = 0; t < n_slots; ++t, pos.next(S, W)) {
      const uint32_t g = pos.g, r = pos.r;
      const uint32_t set = RES_NSETS == 2 ? g & 1u : 0u, ph = RES_NSETS == 2 ? g >> 1 : g;
      const uint32_t b = t & 1u, u = t >> 1;
      if (r == 0) mbar_wait(&in_full[set], ph & 1u);
      if (bt == 0) trace_ev(p, t, 5);
      const SlotInfo si = s_slot[r];
      if (bt == 0) trace_ev(p, t, 6);
      mbar_wait(&a_free[b], (u & 1u) ^ 1u);
      // operands produced in this group: wait until the epilogue has put them in their buffers
      // (one mbarrier phase per lane group; the producer's next group runs after this slot)
      if (DEPS && !FHEGPU_ABL(p, 1u << 19)) {         // dbg bit 19: no waits (timing only)
        if (si.dep_l != 0xFF) mbar_wait(&out_ready[si.dep_l], g & 1u);
        if (si.dep_r != 0xFF) mbar_wait(&out_ready[si.dep_r], g & 1u);
      }
      if (bt == 0) trace_ev(p, t, 7);
      tc_fence_after();
      const uint32_t *in_b = s_inb + set * in_set_words;
      const uint32_t *v1 = ((si.bits & 8u) ? s_loc : in_b) + si.v1;
      const uint32_t *v2 = ((si.bits & 16u) ? s_loc : in_b) + si.v2;
      const bool comp1 = si.bits & 1u, comp2 = si.bits & 2u;
      uint8_t *bb = s_b + b * R::B_BYTES;
      {
        const uint32_t a_addr = tmem_base + b * G::BUF_COLS + lane_off + G::D_COLS + tile * 8 * K;
        if (si.bits & 64u) {                       // reuse: only the columns the tail MMA overwrote
          if (tile == 0) build_a_words<K, 0, 6, ENC>(v1, row, row_blk, row_bit, comp1, p.q, a_addr);
        } else if constexpr (R::BSPLIT == 1) {
          build_a_words<K, 0, K, ENC>(v1, row, row_blk, row_bit, comp1, p.q, a_addr);
        } else {
          if (part == 0) build_a_words<K, 0, 4, ENC>(v1, row, row_blk, row_bit, comp1, p.q, a_addr);
          else build_a_words<K, 4, K, ENC>(v1, row, row_blk, row_bit, comp1, p.q, a_addr);
        }
      }
      if constexpr (G::TAIL > 0) {
        if (tb >= 0 && tb < G::TAIL * K && !(si.bits & 64u)) {   // reuse: TA(b) holds this tail A
          const int m = tb / K, ww = tb - m * K;
          const int rr = G::MMA_ROWS + m;
          uint32_t v = v1[rr * K + ww];
          if (comp1) v = sub_mod(ww == rr / ELL ? (1u << (rr % ELL)) : 0u, v, p.q);
          uint32_t sp[8];
          spread_word_sr<ENC>(v, sp);
          uint8_t *dst = s_ta + b * R::TA_BYTES + (2 * ww) * G::TA_LBO + m * 16;
          *reinterpret_cast<uint4 *>(dst) = make_uint4(sp[0], sp[1], sp[2], sp[3]);
          *reinterpret_cast<uint4 *>(dst + G::TA_LBO) = make_uint4(sp[4], sp[5], sp[6], sp[7]);
        }
      }
#pragma unroll
      for (int x = 0; x < (R::NBC_WARPS > 0 ? 0 : B_ROWS); ++x) {   // else the B copiers do it
        if (b_src[x] < 0) continue;
        uint32_t vals[K];
#pragma unroll
        for (int i = 0; i < K; ++i) vals[i] = v2[b_src[x] + i];
        if (comp2) {
#pragma unroll
          for (int i = 0; i < K; ++i) vals[i] = sub_mod(i == b_w[x] ? (1u << b_j[x]) : 0u, vals[i], p.q);
        }
        uint8_t *dst = bb + b_dst[x];
#pragma unroll
        for (int ch = 0; ch < G::NCH; ++ch) {
          uint4 val;
          val.x = 4 * ch + 0 < K ? vals[4 * ch + 0] : 0u;
          val.y = 4 * ch + 1 < K ? vals[4 * ch + 1] : 0u;
          val.z = 4 * ch + 2 < K ? vals[4 * ch + 2] : 0u;
          val.w = 4 * ch + 3 < K ? vals[4 * ch + 3] : 0u;
          *reinterpret_cast<uint4 *>(dst + ch * G::SBO) = val;
        }
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&op_full[b]);
        if (si.bits & 32u) mbar_arrive(&in_empty[set]);   // every input reader of the group is built
      }
      if (bt == 0) trace_ev(p, t, 8);
    }
  } else {
    // ------------------------------ epilogue, into the gate's local buffer ------------------------------
    const int et = tid - 32 * R::WARP_EPI0;
    const int ew = et >> 5;
    const int quad = warp & 3;
    const int tile = (ew >> 2) & 1;
    const int part = ew >> 3;                      // value range of this thread (EPI_SPLIT = 2)
    const int row = 128 * tile + 32 * quad + lane;
    const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
    const int row_blk = row / ELL, row_bit = row - row_blk * ELL;
    constexpr uint32_t NE_THREADS = 32 * R::NE_WARPS;
    if (et == 0) mbar_arrive(&out_free[0]);
    SlotPos pos;
    for (uint32_t t = 0; t < n_slots; ++t, pos.next(S, W)) {
      const uint32_t b = t & 1u, u = t >> 1;
      const uint32_t g = pos.g, r = pos.r;
      const SlotInfo si = s_slot[r];
      const uint32_t o = si.ow & 7u, w = (si.ow >> 3) & 3u;
      uint32_t *out_st = s_loc + si.dest;
      mbar_wait(&main_done[b], u & 1u);
      if (si.ow & 32u) named_bar(2, NE_THREADS);   // store hazard: slot t-1's store has read the buffer
      if (et == 0) trace_ev(p, t, 9);
      tc_fence_after();
      const uint32_t dcol = tmem_base + b * G::BUF_COLS + lane_off + tile * G::NPAD;
      if constexpr (R::EPI_SPLIT == 1) {
        uint32_t d[36];
        load_acc36(dcol, d, false);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_free[b]);
#pragma unroll
        for (int i = 0; i < K; ++i)
          out_st[row * K + i] = finish_neg<ELL, PM, ENC>(&d[i * 4], i == row_blk ? (1u << row_bit) : 0u, p);
      } else {
        static_assert(K == 9, "split epilogue: values 0-4 and 5-8");
        uint32_t d[20];
        if (part == 0) {                           // values 0-4: columns 0-19
          tmem_ld16(dcol, d);
          tmem_ld4(dcol + 16, d + 16);
        } else {                                   // values 5-8: columns 20-35 (naturally aligned pieces)
          tmem_ld4(dcol + 20, d);
          tmem_ld8(dcol + 24, d + 4);
          tmem_ld4(dcol + 32, d + 12);
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_free[b]);
        if (part == 0) {
#pragma unroll
          for (int i = 0; i < 5; ++i)
            out_st[row * K + i] = finish_neg<ELL, PM, ENC>(&d[i * 4], i == row_blk ? (1u << row_bit) : 0u, p);
        } else {
#pragma unroll
          for (int i = 5; i < 9; ++i)
            out_st[row * K + i] =
                finish_neg<ELL, PM, ENC>(&d[(i - 5) * 4], i == row_blk ? (1u << row_bit) : 0u, p);
        }
      }
      fence_proxy_async_smem();
      const SlotInfo sn = s_slot[r + 1 == S ? 0u : r + 1];
      const bool next_hazard = (sn.ow & 32u) && t + 1 < n_slots;
      if (et == 0 && t + 1 < n_slots) {
        // the next gate writes an output buffer: every earlier store (outputs of one group may
        // share a buffer) must have read its source
        if (sn.bits & 4u) bulk_wait_read_n<0>();
        if (!next_hazard) mbar_arrive(&out_free[(t + 1) % R::N_OUT]);
      }
      named_bar(1, NE_THREADS);
      if (et == 0) trace_ev(p, t, 10);
      if (et == 0) {
        const uint32_t ob = t % R::N_OUT, ou = t / R::N_OUT;
        mbar_wait(&tail_ready[ob], ou & 1u);
        const uint32_t ln = lane_of_group(g, w);
        if ((si.bits & 4u) && ln < lanes) {               // partial last group: no store
          uint32_t *dst = store + ((uint64_t)s_plan[o].out_slot * lanes + ln) * R::CT_WORDS;
          if (FHEGPU_RES_HINT) bulk_s2g_hint(dst, out_st, R::CT_BYTES, policy_evict_first());
          else bulk_s2g(dst, out_st, R::CT_BYTES);
        }
        if (next_hazard) {                         // the next gate rewrites this buffer
          bulk_wait_read_n<0>();
          mbar_arrive(&out_free[(t + 1) % R::N_OUT]);
        }
      } else if (et == 32) {
        // the gate's output is readable in its buffer: published by a thread without bulk
        // stores in flight (a release on the storing thread would wait for its stores)
        const uint32_t ob = t % R::N_OUT, ou = t / R::N_OUT;
        mbar_wait(&tail_ready[ob], ou & 1u);
        mbar_arrive(&out_ready[r]);
        trace_ev(p, t, 11);
      }
    }
    if (et == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == G::WARP_MMA) tmem_dealloc<512>(tmem_base);
}

}  // namespace tc
}  // namespace fhegpu
