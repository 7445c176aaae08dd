// tc_nand_ws.cuh -- warp-specialised, pipelined tcgen05 level kernel (the production kernel).
//
// Same math as tc_nand.cuh (compact NAND: out = (G - bits(V1) V2) mod q, the product on
// the tensor cores as a u8 GEMM), restructured so the phases of different gates overlap
// inside one persistent CTA per SM (608 threads):
//
//   warp 0        tail     : A of the 5 rows past the 2 MMA tiles (smem), their accumulator
//                            read-out (TMEM lanes 0..4, hence a quadrant-0 warp) and the
//                            st.global of those rows; frees the A buffer right after the read
//   warp 1        producer : cp.async.bulk of both operands into an S_IN-stage ring
//   warp 2        MMA      : one thread issues 2 x 9 TMEM-A tile MMAs + 9 smem-A tail MMAs
//   warps 3..10   builders : B operand (smem, MN-major) + A operand (bits -> s8 {0,-1},
//                            tcgen05.st into TMEM) of gate t while the MMAs of gate t-1 run
//   warps 11..18  epilogue : tcgen05.ld of gate t-1's tile accumulators, mod-q fold,
//                            one bulk store of rows 0..255
//
// TMEM (512 columns): two buffers of {D tile0, D tile1, A tile0, A tile1} (240 columns);
// the tail accumulates into the tile-0 A columns of its buffer, issued after the tile MMAs
// (tcgen05.mma executes in issue order; the 9 tile-1 MMAs separate tile 0's last read of
// those columns from the tail's writes).
//
// mbarriers: in_full/in_empty per input stage; per TMEM buffer b: op_full (builders + tail
// -> MMA), main_done (tcgen05.commit -> epilogue, tail), a_free (tail read-out -> builders
// of gate t+2), d_free (epilogue tile read-out -> MMA of gate t+2).
//
// A operand: word w of row r spreads into 8 u32 (32 K slots); output o holds in byte q
// the bit 8q + o of w replicated to 0x00/0xFF by a sign-replicating PRMT of (w << (7 - o)),
// i.e. the s8 value 0 or -1, so D = -(digit sums) and the epilogue negates.  K slot 4o + q
// of word w pairs with V2 row w * ELL + 8q + o in B.
#pragma once

#include "tc_nand.cuh"

namespace fhegpu {
namespace tc {

// Pipeline timeline probe (dbg bit 14, builds with -DFHEGPU_TRACE=1 only -- tools/timeline.py):
// CTA 0 records clock64 per (gate, event).  Compiled out by default: even predicated off, the
// probes cost the issue-bound roles a few instructions per gate.
#ifndef FHEGPU_TRACE
#define FHEGPU_TRACE 0
#endif
// Stage-ablation knobs (debug bits that skip loads, operand builds, MMAs, epilogue math or
// stores; results invalid -- tools/probes/ablate.py): compiled in only with -DFHEGPU_ABLATE=1,
// so release kernels carry none of their branches.
#ifndef FHEGPU_ABLATE
#define FHEGPU_ABLATE 0
#endif
#define FHEGPU_ABL(p, mask) (FHEGPU_ABLATE && ((p).dbg & (mask)))
__device__ uint64_t g_ws_trace[64 * 16];
__device__ __forceinline__ void trace_ev(const DevParams &p, uint32_t t, int ev) {
#if FHEGPU_TRACE
  // window of 64 gates starting at gate 64 * (dbg >> 20) of CTA 0
  const uint32_t t0 = 64u * (p.dbg >> 20);
  if ((p.dbg & 16384u) && blockIdx.x == 0 && t >= t0 && t < t0 + 64) g_ws_trace[(t - t0) * 16 + ev] = clock64();
#endif
}

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read_n() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_n() {                 // writes complete, not just read
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// -- dataflow scheduling (one launch for a whole program) --------------------------------
// Item i (ops in topological order, lanes inner) runs on CTA i % G as that CTA's local item
// i / G; progress[c] = number of CTA c's local items whose output ciphertext is globally
// written.  A consumer waits for progress[producer CTA] > producer's local index.
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Block until the item that produced an operand (op index `dep`, same lane) is written.
// `seen` caches the last progress value read (acquire) per CTA: counters only grow, so a
// cached value that already covers the dependency needs no global round trip.
__device__ __forceinline__ void wait_dep(const uint32_t *progress, uint32_t *seen, int dep, uint32_t lanes,
                                         uint32_t ln) {
  if (dep < 0) return;
  const uint32_t i = (uint32_t)dep * lanes + ln;
  const uint32_t c = i % gridDim.x, k = i / gridDim.x;
  if (seen[c] > k) return;
  uint32_t v;
  while ((v = ld_acquire_gpu(progress + c)) <= k) __nanosleep(32);
  seen[c] = v;
}

// Counters only grow: max-reduction with release semantics, so the two publishers (the
// epilogue store thread when it is about to block, the tail warp otherwise) never regress.
__device__ __forceinline__ void red_max_release_gpu(uint32_t *p, uint32_t v) {
  asm volatile("red.release.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release_cta_smem(uint32_t *p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_cta_smem(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// Make local items [0, n) visible to other CTAs (their bulk stores have completed).  A
// release on the thread that issued the bulk stores waits for ALL its outstanding stores,
// so the steady state posts n to shared memory instead (post_local) and the tail warp,
// which has no global stores in flight, performs the release (relay).
__device__ __forceinline__ void publish(uint32_t *progress, uint32_t n) {
  fence_proxy_async_global();
  red_max_release_gpu(progress + blockIdx.x, n);
}

__device__ __forceinline__ void post_local(uint32_t *s_pub, uint32_t n) {
  // the stores being posted have COMPLETED (cp.async.bulk.wait_group returned: their writes
  // are acknowledged at L2, where consumers' bulk loads read); the proxy fence orders them
  // before this thread's later generic operations and the shared-memory post only has to
  // be observed after that point -- a CTA-scope release here would wait for the stores
  // still in flight, which is the cost this relay exists to avoid
  fence_proxy_async_global();
  asm volatile("st.volatile.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(s_pub)), "r"(n) : "memory");
}

// L2 evict-first policy for stores of streamed outputs (op flag FHEGPU_OP_STREAM_OUT)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_s2g_hint(void *dst, const void *src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint32_t prmt_sign(uint32_t x) {
  uint32_t r;  // default-mode prmt: selector nibble bit 3 replicates the selected byte's msb
  asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(x));
  return r;
}

#ifndef FHEGPU_PUBLISH_LAG
#define FHEGPU_PUBLISH_LAG 1   // dataflow: publish outputs this many gates behind the epilogue
#endif

// A operand encoding (kernel template parameter ENC), both toggling one bit per byte in the
// MMA datapath ({0, -1} bytes, all eight bits, cost 2.6% under the power cap):
//   1: s8 {0, +1} = (w >> o) & 0x01010101 -- two ALU-pipe ops per output register;
//      D = digit sums.  Used by dataflow (tiled) launches.
//   2: u8 {0, 128} = (w << (7 - o)) & 0x80808080 -- ptxas issues the left shift on the FMA
//      pipe (IMAD.SHL), halving the ALU work of the spread, which saturates that pipe
//      (tools/micro/tmem_st_bench.cu); D = 128 x digit sums.  Level launches: +1.7%
//      (load-bound there, the builders finish early); in dataflow launches the larger
//      accumulators and the epilogue's extra shift cost more than the builders gain (-6%).
#ifndef FHEGPU_ENC_LEVELS
#define FHEGPU_ENC_LEVELS 2
#endif
#ifndef FHEGPU_ENC_FLOW
#define FHEGPU_ENC_FLOW 1
#endif

template <int ENC>
struct AEnc {
  static_assert(ENC == 1 || ENC == 2, "A operand encoding");
  static constexpr int SHIFT = ENC == 2 ? 7 : 0;        // log2 of the accumulator scale
  static constexpr uint32_t A_FMT = ENC == 2 ? 0u : 1u;  // idesc a_format: u8 / s8
};

// 32 bits of w -> 32 K slots: out[o] byte q = bit (8q + o) (scaled per encoding).
template <int ENC>
__device__ __forceinline__ void spread_word_sr(uint32_t w, uint32_t (&out)[8]) {
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    if constexpr (ENC == 2) out[o] = (w * (1u << (7 - o))) & 0x80808080u;
    else out[o] = (w >> o) & 0x01010101u;
  }
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t *v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t *v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
}

// 36 accumulator columns (9 values x 4 digits) of this warp's 32 TMEM lanes.
__device__ __forceinline__ void load_acc36(uint32_t taddr, uint32_t (&d)[36], bool skip) {
  if (skip) {
#pragma unroll
    for (int i = 0; i < 36; ++i) d[i] = 0u;
    return;
  }
  tmem_ld32(taddr, d);
  tmem_ld4(taddr + 32, d + 32);
}

// tail MMA (5 live rows): M = FHEGPU_TAIL_M; FHEGPU_TAIL_ZERO backs the rows past the live
// 8-row group with zeros (see GeoWS::TA_GROUPS)
#ifndef FHEGPU_TAIL_M
#define FHEGPU_TAIL_M 64
#endif
#ifndef FHEGPU_TAIL_ZERO
#define FHEGPU_TAIL_ZERO 1
#endif

template <int K, int ELL, bool PM, int ENC, bool Q = false>
struct GeoWS {
  using B = Geo<K, ELL>;
  static constexpr int ROWS = B::ROWS;
  static constexpr int MT = B::MT;
  static constexpr int TAIL = B::TAIL;
  static constexpr int MMA_ROWS = B::MMA_ROWS;
  static constexpr int NPAD = B::NPAD, NCH = B::NCH, KB = B::KB, NDIG = B::NDIG;
  static constexpr uint32_t SBO = B::SBO, LBO = B::LBO, TA_LBO = B::TA_LBO;
  static constexpr int B_BYTES = B::B_BYTES;
  // tail A: the live 8-row core-matrix group (rows MMA_ROWS.., K-major) followed by
  // TAIL_M/8 - 1 all-zero groups, so the M = TAIL_M tail MMA multiplies B by zero rows
  // (no datapath toggles) instead of by copies of the live rows (SBO = 0 aliasing)
  static constexpr int TA_GROUPS = FHEGPU_TAIL_ZERO ? FHEGPU_TAIL_M / 8 : 1;
  static constexpr uint32_t TA_SBO = FHEGPU_TAIL_ZERO ? (uint32_t)B::TA_BYTES : 0u;
  static constexpr int TA_BYTES = B::TA_BYTES * TA_GROUPS;
  static constexpr int WORDS = B::WORDS;
  static constexpr int CT_WORDS = B::CT_WORDS, CT_BYTES = B::CT_BYTES;
  static constexpr int MAIN_BYTES = MMA_ROWS * K * 4;       // rows stored by the bulk copy
  static constexpr int D_COLS = B::D_COLS;                 // per buffer
  static constexpr int BUF_COLS = 256;                      // buffer stride in TMEM columns
#ifndef FHEGPU_WS_BCOPY
#define FHEGPU_WS_BCOPY 4      // ready-queue launches: warps dedicated to the B copy (cfg2/cfg3
#endif                         // +4%; level and tiled launches keep the builders' copy: -6% / -1%)
  static constexpr int NB_WARPS = 4 * MT, NE_WARPS = 4 * MT, NBC_WARPS = Q ? FHEGPU_WS_BCOPY : 0;
  static constexpr int WARP_TAIL = 0, WARP_PROD = 1, WARP_MMA = 2;
  static constexpr int WARP_BUILD0 = 3, WARP_BC0 = 3 + NB_WARPS, WARP_EPI0 = WARP_BC0 + NBC_WARPS;
  // ready-queue launches (Q): a fetcher warp (pops ready items) and a signaler warp (retires
  // completed items to their consumers) after the epilogue warps
  static constexpr int WARP_FETCH = WARP_EPI0 + NE_WARPS, WARP_SIG = WARP_FETCH + 1;
  static constexpr int THREADS = 32 * (3 + NB_WARPS + NBC_WARPS + NE_WARPS + (Q ? 2 : 0));
// ready-queue launches: operand stages, fetch-ring entries, queue pops per fetch batch
// (swept on cfg2/cfg3: 5/4/2; one pop per batch leaves the fetcher latency-bound, deeper
// rings put more items ahead of each dependency hop)
#ifndef FHEGPU_STAGES
#define FHEGPU_STAGES 7        // operand stages of level / dataflow launches
#endif
#ifndef FHEGPU_Q_STAGES
#define FHEGPU_Q_STAGES 5
#endif
#ifndef FHEGPU_Q_FQ
#define FHEGPU_Q_FQ 4
#endif
#ifndef FHEGPU_Q_FD
#define FHEGPU_Q_FD 2
#endif
  // operand stages: ~2.5 us load latency x bandwidth (ready-queue launches: every stage is
  // also latency on the dependency chain; their operands are mostly L2 hits)
  static constexpr int S_IN = Q ? FHEGPU_Q_STAGES : FHEGPU_STAGES;
  static constexpr int N_OUT = 3;                           // output staging buffers
  static constexpr uint32_t OP_ARRIVALS = NB_WARPS + NBC_WARPS;
  // idesc: S32 accumulator, A s8 (bits 7-9 = 1) or u8 (encoding 2), B u8, A K-major,
  // B MN-major, N>>3, M>>4
  static constexpr uint32_t IDESC = (2u << 4) | (AEnc<ENC>::A_FMT << 7) | (1u << 16) |
                                    ((uint32_t)(NPAD >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  // tail MMA (5 live rows): M = 64 has the issue cost of M = 128 (the floor is max(M, 128))
  // and half the datapath work
  static constexpr uint32_t IDESC_TAIL = (IDESC & ~(0x1fu << 24)) | ((uint32_t)(FHEGPU_TAIL_M >> 4) << 24);
  static constexpr int OFF_IN = 0;
  static constexpr int OFF_B = OFF_IN + S_IN * 2 * CT_BYTES;
  static constexpr int OFF_TA = ((OFF_B + 2 * B_BYTES + 127) / 128) * 128;
  static constexpr int OFF_OUT = ((OFF_TA + (TAIL ? 2 * TA_BYTES : 0) + 127) / 128) * 128;
  static constexpr int OFF_BAR = ((OFF_OUT + N_OUT * CT_BYTES + 127) / 128) * 128;
  static constexpr int OFF_SEEN = OFF_BAR + 256;          // dataflow: progress cache, <= 256 CTAs
  static constexpr int MAX_CTAS = 256;
  static constexpr int OFF_PUB = OFF_SEEN + 4 * MAX_CTAS;  // dataflow: epilogue -> tail relay
  static constexpr int OFF_FLAGS = OFF_PUB + 16;            // op flags of each input stage
  // ready queue (Q): fetched-entry ring, per-slot item / output rings, counters
  static constexpr int FQ = FHEGPU_Q_FQ, FD = FHEGPU_Q_FD;  // fetch ring entries, pops per batch
  static constexpr int QR = 64;                             // slot ring (item, output ciphertext)
  static constexpr int OFF_Q = OFF_FLAGS + 4 * ((S_IN + 3) / 4 * 4);
  static constexpr int OFF_FQ = OFF_Q;                      // FQ x uint4 {left, right, out, flags}
  static constexpr int OFF_FQI = OFF_FQ + 16 * FQ;          // FQ x {item, seq}
  static constexpr int OFF_QITEM = OFF_FQI + 8 * FQ;        // QR items
  static constexpr int OFF_QOUT = OFF_QITEM + 4 * QR;       // QR output ciphertext indices
  static constexpr int OFF_QCNT = OFF_QOUT + 4 * QR;        // fq_used, signaled, epi_end, pad
  static constexpr int SMEM = Q ? OFF_QCNT + 16 : OFF_Q;
  static_assert(NDIG == 4 && B::NCOL <= 36, "warp-specialised kernel: 4 digits, <= 36 columns");
  static_assert(MT >= 1 && TAIL <= 8, "two-tile geometry");
  static_assert((uint64_t)ROWS * 255u * 257u << AEnc<ENC>::SHIFT < (1ull << 32), "scaled digit sums fit u32");
  static_assert(B::D_COLS + B::A_COLS <= BUF_COLS, "two TMEM buffers must fit 512 columns");
  static_assert(MAIN_BYTES % 16 == 0, "bulk store size");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

// Digit-sum epilogue: d[] are the digit sums S_d scaled by 2^SHIFT.
template <int ELL, bool PM, int ENC>
__device__ __forceinline__ uint32_t finish_neg(const uint32_t *d, uint32_t g, const DevParams &p) {
  uint32_t r;
  if constexpr (PM) {
    // S = a + b 2^16 with a = S0 + S1 2^8, b = S2 + S3 2^8 (both < 2^26).  Folding b's bits
    // above 2^(ELL-16) with 2^ELL = c (mod q) gives t = a + bl 2^16 + c bh < 2q (host-checked,
    // pm_ok) -- and t = a + b 2^16 - q bh exactly, so t can be formed modulo 2^32 from the
    // wrapped S32 = S0 + S1 2^8 + S2 2^16 + S3 2^24.  Encoding 2 carries every digit sum
    // scaled by 2^7: a' = 2^7 a < 2^32 and b' = 2^7 b < 2^29 (top digits < 2^(ELL-24)) stay
    // exact, a = a' >> 7 and b 2^16 = b' << 9 (mod 2^32).
    constexpr int SH = AEnc<ENC>::SHIFT;
    const uint32_t b = d[2] + (d[3] << 8);
    const uint32_t a = d[0] + (d[1] << 8);
    const uint32_t s32 = (a >> SH) + (b << (16 - SH));
    const uint32_t t = s32 - p.q * (b >> (ELL - 16 + SH));
    r = min(t, t - p.q);                            // t < 2q
  } else {
    const int64_t sum = (int64_t)(int32_t)d[0] + ((int64_t)(int32_t)d[1] << 8) +
                        ((int64_t)(int32_t)d[2] << 16) + ((int64_t)(int32_t)d[3] << 24);
    const int64_t s = sum >> AEnc<ENC>::SHIFT;
    r = mod_u64((uint64_t)s, p.q, p.mu);
  }
  const uint32_t x = g - r;
  return min(x, x + p.q);                           // (g - r) mod q for g, r < q
}

// Ready-queue state of one run (fhegpu.cu launch_queue resets it before every launch).
struct QueueArgs {
  uint32_t *queue;            // n_items entries: ready items in push order, EMPTY until pushed
  uint32_t *counters;         // [0] pop cursor, [1] push cursor
  uint32_t *pending;          // per item: producing items not yet retired
  const uint32_t *cons_off;   // per op: consumer list offsets (n_ops + 1)
  const uint32_t *cons;       // consumer ops (distinct per producer)
};
constexpr uint32_t Q_EMPTY = 0xFFFFFFFFu, Q_END = 0xFFFFFFFEu;

__device__ __forceinline__ uint32_t ld_volatile_smem(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_smem(uint32_t *p, uint32_t v) {
  asm volatile("st.volatile.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_dec_acq_rel_gpu(uint32_t *p) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(0xFFFFFFFFu) : "memory");
  return old;
}
// bounded spin (a protocol error traps instead of hanging the GPU)
#define FHEGPU_SPIN_LIMIT (1u << 26)

// Op record of gate item `item` (or a dummy past the end): issued one gate ahead so the
// global-load latency never sits on a role's critical loop.
__device__ __forceinline__ OpRec fetch_op(const OpRec *ops, uint32_t item, uint32_t n_items,
                                          uint32_t lanes, uint32_t magic) {
  if (item >= n_items) return OpRec{0u, 0u, 0u, 0u};
  uint32_t q, r;
  div_lanes(item, lanes, magic, q, r);
  return ops[q];
}

__device__ __forceinline__ uint32_t lane_of(uint32_t item, uint32_t lanes, uint32_t magic) {
  uint32_t q, r;
  div_lanes(item, lanes, magic, q, r);
  return r;
}

template <int K, int ELL, bool PM, int ENC, bool Q>
__global__ void __launch_bounds__(GeoWS<K, ELL, PM, ENC, Q>::THREADS, 1)
level_tc_ws_kernel(uint32_t *__restrict__ store, const OpRec *__restrict__ ops, uint32_t n_ops,
                   uint32_t lanes, DevParams p, const int2 *__restrict__ deps, uint32_t *__restrict__ progress,
                   QueueArgs qa) {
  // deps == nullptr: one netlist level (the previous level completed before launch).
  // deps != nullptr: a whole program in dataflow order (ops topologically sorted, SSA slots:
  // no slot is written twice or overwritten while a reader may still need it); each operand
  // load waits for its producing item via `progress` (gridDim.x entries, zeroed per run).
  // Q: a whole program over a ready queue (SSA slots): CTAs pop items whose producers have
  // retired (fetcher warp), and retire their own completed items to the consumers' pending
  // counters, pushing each consumer whose count reaches zero (signaler warp).  Every role
  // then runs slot by slot until the END slot; the per-slot item lives in a smem ring.
  using G = GeoWS<K, ELL, PM, ENC, Q>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t *s_in = reinterpret_cast<uint32_t *>(smem + G::OFF_IN);
  uint8_t *s_b = smem + G::OFF_B;
  uint8_t *s_ta = smem + G::OFF_TA;
  uint32_t *s_out = reinterpret_cast<uint32_t *>(smem + G::OFF_OUT);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + G::OFF_BAR);
  uint64_t *in_full = bar;                    // [S_IN]
  uint64_t *in_empty = bar + G::S_IN;         // [S_IN]
  uint64_t *op_full = bar + 2 * G::S_IN;      // [2]
  uint64_t *main_done = op_full + 2;          // [2]
  uint64_t *a_free = main_done + 2;           // [2]
  uint64_t *d_free = a_free + 2;              // [2]
  uint64_t *out_free = d_free + 2;            // [N_OUT] staging o may take gate t's rows
  uint64_t *tail_ready = out_free + G::N_OUT; // [N_OUT] tail rows of gate t are in staging o
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tail_ready + G::N_OUT);
  uint32_t *s_seen = reinterpret_cast<uint32_t *>(smem + G::OFF_SEEN);
  uint32_t *s_pub = reinterpret_cast<uint32_t *>(smem + G::OFF_PUB);
  uint32_t *s_flags = reinterpret_cast<uint32_t *>(smem + G::OFF_FLAGS);  // written by the producer
  uint4 *s_fq = reinterpret_cast<uint4 *>(smem + G::OFF_FQ);               // Q: fetched ops
  uint32_t *s_fqi = reinterpret_cast<uint32_t *>(smem + G::OFF_FQI);       // Q: {item, seq}
  uint32_t *s_qitem = reinterpret_cast<uint32_t *>(smem + G::OFF_QITEM);   // Q: item of slot t
  uint32_t *s_qout = reinterpret_cast<uint32_t *>(smem + G::OFF_QOUT);     // Q: output ct of slot t
  uint32_t *s_qcnt = reinterpret_cast<uint32_t *>(smem + G::OFF_QCNT);     // Q: fq_used, signaled, epi_end

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t n_items = n_ops * lanes;     // host guarantees < 2^32

  // Programmatic dependent launch: the next level's grid may be scheduled now; its CTAs
  // take each SM as this grid's CTA leaves it and overlap their prologue with our tail.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == G::WARP_MMA) tmem_alloc<512>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < G::S_IN; ++i) {
      mbar_init(&in_full[i], 1);
      mbar_init(&in_empty[i], G::OP_ARRIVALS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&op_full[i], G::OP_ARRIVALS);
      mbar_init(&main_done[i], 1);
      mbar_init(&a_free[i], 1);
      mbar_init(&d_free[i], G::NE_WARPS);
    }
    for (int i = 0; i < G::N_OUT; ++i) {
      mbar_init(&out_free[i], 1);
      mbar_init(&tail_ready[i], 1);
    }
    fence_mbar_init();
  }
  for (int w = tid; w < 2 * G::B_BYTES / 4; w += G::THREADS) reinterpret_cast<uint32_t *>(s_b)[w] = 0u;
  if constexpr (G::TAIL > 0)
    for (int w = tid; w < 2 * G::TA_BYTES / 4; w += G::THREADS) reinterpret_cast<uint32_t *>(s_ta)[w] = 0u;
  for (int w = tid; w < G::N_OUT * G::CT_WORDS; w += G::THREADS) s_out[w] = 0u;   // padding stays 0
  for (int w = tid; w < G::MAX_CTAS; w += G::THREADS) s_seen[w] = 0u;
  if (tid == 0) *s_pub = 0u;
  if constexpr (Q) {
    for (int w = tid; w < 2 * G::FQ; w += G::THREADS) s_fqi[w] = 0u;
    if (tid < 4) s_qcnt[tid] = 0u;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // every global read/write of ciphertexts comes after the previous level has completed
  // (its outputs are our operands; slots it read may be our outputs); no-op without PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == G::WARP_PROD) {
    // ------------------------------ producer ------------------------------
    if (Q && lane == 0) {
      // ready-queue launch: slot t takes fetched entry t (its operands are already written)
      for (uint32_t t = 0;; ++t) {
        const uint32_t s = t % G::S_IN, k = t / G::S_IN, e = t % G::FQ;
        uint32_t spins = 0;
        while (ld_acquire_cta_smem(&s_fqi[2 * e + 1]) != t + 1)
          if (++spins > FHEGPU_SPIN_LIMIT) __trap();
        const uint4 ent = s_fq[e];
        const uint32_t item = s_fqi[2 * e];
        st_release_cta_smem(&s_qcnt[0], t + 1);     // entry consumed: the fetcher may refill it
        // slot-ring entry t % QR is reused once the signaler has retired slot t - QR
        spins = 0;
        while (t >= (uint32_t)G::QR && ld_volatile_smem(&s_qcnt[1]) + G::QR <= t) {
          __nanosleep(32);
          if (++spins > FHEGPU_SPIN_LIMIT) __trap();
        }
        mbar_wait(&in_empty[s], (k & 1u) ^ 1u);
        s_qitem[t % G::QR] = item;
        s_qout[t % G::QR] = ent.z;
        if (item == Q_END) {                       // every role leaves at this slot
          s_flags[s] = 0u;
          mbar_arrive(&in_full[s]);
          break;
        }
        fence_proxy_async_global();                 // acquired ready item -> async-proxy loads
        const bool same = ent.x == ent.y;
        s_flags[s] = ent.w | (same ? 4u : 0u);
        uint32_t *dst = s_in + s * 2 * G::CT_WORDS;
        mbar_expect_tx(&in_full[s], (same ? 1 : 2) * G::CT_BYTES);
        bulk_g2s(dst, store + (uint64_t)ent.x * G::CT_WORDS, G::CT_BYTES, &in_full[s]);
        if (!same) bulk_g2s(dst + G::CT_WORDS, store + (uint64_t)ent.y * G::CT_WORDS, G::CT_BYTES, &in_full[s]);
      }
    } else if (!Q && lane == 0) {
      uint32_t t = 0;
      OpRec op_next = fetch_op(ops, blockIdx.x, n_items, lanes, p.lanes_magic);
      int2 dep_next = make_int2(-1, -1);
      if (deps != nullptr && blockIdx.x < n_items) {
        uint32_t q0, r0;
        div_lanes(blockIdx.x, lanes, p.lanes_magic, q0, r0);
        dep_next = deps[q0];
      }
      for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
        const uint32_t s = t % G::S_IN, k = t / G::S_IN;
        const OpRec op = op_next;
        const int2 dep = dep_next;
        op_next = fetch_op(ops, item + gridDim.x, n_items, lanes, p.lanes_magic);
        if (deps != nullptr && item + gridDim.x < n_items) {     // prefetched one item ahead
          uint32_t q1, r1;
          div_lanes(item + gridDim.x, lanes, p.lanes_magic, q1, r1);
          dep_next = deps[q1];
        }
        mbar_wait(&in_empty[s], (k & 1u) ^ 1u);
        trace_ev(p, t, 0);
        const uint32_t ln = lane_of(item, lanes, p.lanes_magic);
        if (deps != nullptr) {
          wait_dep(progress, s_seen, dep.x, lanes, ln);
          wait_dep(progress, s_seen, dep.y, lanes, ln);
          fence_proxy_async_global();             // acquired generic flag -> async-proxy loads
        }
        uint32_t *dst = s_in + s * 2 * G::CT_WORDS;
        // NAND(x, x) (NOT by NAND, 3-17% of the reference netlists' gates): one load, the
        // builders read the second operand from the first buffer (flag bit 2)
        const bool same = op.left == op.right;
        s_flags[s] = op.flags | (same ? 4u : 0u); // published to the builders by in_full's arrive
        if (FHEGPU_ABL(p, 256u)) {                       // timing experiment: no operand loads
          mbar_arrive(&in_full[s]);
          continue;
        }
        mbar_expect_tx(&in_full[s], (same ? 1 : 2) * G::CT_BYTES);
        bulk_g2s(dst, store + ((uint64_t)op.left * lanes + ln) * G::CT_WORDS, G::CT_BYTES, &in_full[s]);
        if (!same)
          bulk_g2s(dst + G::CT_WORDS, store + ((uint64_t)op.right * lanes + ln) * G::CT_WORDS,
                   G::CT_BYTES, &in_full[s]);
      }
    }
  } else if (warp == G::WARP_MMA) {
    // ------------------------------ MMA issuer ------------------------------
    // The whole warp runs the loop (descriptors stay warp-uniform, in uniform registers);
    // one elected lane issues each tcgen05.mma / commit.
    uint32_t t = 0;
    const uint32_t idesc = G::IDESC;
    const uint64_t bdesc0 = smem_desc(smem_u32(s_b), G::LBO, G::SBO);
    const uint64_t tdesc0 = smem_desc(smem_u32(s_ta), G::TA_LBO, G::TA_SBO);
    for (uint32_t item = blockIdx.x; Q || item < n_items; item += gridDim.x, ++t) {
      const uint32_t b = t & 1u, u = t >> 1;
      mbar_wait(&op_full[b], u & 1u);
      if (Q && s_qitem[t % G::QR] == Q_END) {       // release the tail / epilogue and leave
        if (elect_one()) mma_commit(&main_done[b]);
        __syncwarp();
        break;
      }
      if (lane == 0) trace_ev(p, t, 2);
      mbar_wait(&d_free[b], (u & 1u) ^ 1u);       // epilogue of gate t-2 has read D(b)
      if (lane == 0) trace_ev(p, t, 3);
      tc_fence_after();
      const uint32_t tb = tmem_base + b * G::BUF_COLS;
      // descriptor address field is (addr >> 4): advance by adding byte offsets >> 4
      const uint64_t bd_b = bdesc0 + ((b * G::B_BYTES) >> 4);
      const uint64_t td_b = tdesc0 + ((b * G::TA_BYTES) >> 4);
      if (!FHEGPU_ABL(p, 128u)) {
        if (elect_one()) {
#pragma unroll
          for (int mt = 0; mt < G::MT; ++mt) {
            if (FHEGPU_ABL(p, 1u << 18)) break;             // ablation: no tile MMAs (results invalid)
#pragma unroll
            for (int s = 0; s < K; ++s)
              mma_i8_ts(tb + mt * G::NPAD, tb + G::D_COLS + mt * 8 * K + 8 * s,
                        bd_b + ((s * 4 * G::LBO) >> 4), idesc, s > 0 ? 1u : 0u);
          }
          if (G::TAIL > 0 && !FHEGPU_ABL(p, 1u << 17)) {  // ablation bit 17: no tail MMAs
#pragma unroll
            for (int s = 0; s < K; ++s)
              mma_i8_ss(tb + G::D_COLS, td_b + ((s * 2 * G::TA_LBO) >> 4),
                        bd_b + ((s * 4 * G::LBO) >> 4), G::IDESC_TAIL, s > 0 ? 1u : 0u);
          }
        }
        __syncwarp();
      }
      if (elect_one()) {
        mma_commit(&main_done[b]);
        if constexpr (G::TAIL == 0) mma_commit(&a_free[b]);
      }
      __syncwarp();
      if (lane == 0) trace_ev(p, t, 4);
    }
  } else if (warp == G::WARP_TAIL) {
    // ------------------------------ tail rows ------------------------------
    // Reads the tail accumulator of gate t right after its MMAs, frees the A buffer, then
    // folds the 5 rows into the epilogue's staging buffer (the builders build the tail A).
    if constexpr (G::TAIL > 0) {
      uint32_t t = 0;
      uint32_t relayed = 0;
      for (uint32_t item = blockIdx.x; Q || item < n_items; item += gridDim.x, ++t) {
        const uint32_t b = t & 1u, u = t >> 1;
        if (lane == 0) trace_ev(p, t, 12);
        if (progress != nullptr && lane == 0) {     // dataflow: relay the epilogue's count
          uint32_t v;
          asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(s_pub)) : "memory");
          if (v > relayed) {                        // covers completed stores only: relaxed
            asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(progress + blockIdx.x), "r"(v)
                         : "memory");
            relayed = v;
          }
        }
        mbar_wait(&main_done[b], u & 1u);
        if (Q && s_qitem[t % G::QR] == Q_END) break;
        if (lane == 0) trace_ev(p, t, 13);
        tc_fence_after();
        uint32_t d[36];
        load_acc36(tmem_base + b * G::BUF_COLS + G::D_COLS, d, false);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&a_free[b]);
          trace_ev(p, t, 10);
        }
        const uint32_t o = t % G::N_OUT, ou = t / G::N_OUT;
        mbar_wait(&out_free[o], ou & 1u);            // gate t-N_OUT's store has read staging o
        if (lane == 0) trace_ev(p, t, 14);
        uint32_t *out_st = s_out + o * G::CT_WORDS;
        if (lane < G::TAIL && !FHEGPU_ABL(p, 1024u)) {
          const int r = G::MMA_ROWS + lane;
          const int rb = r / ELL, rbit = r - rb * ELL;
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const uint32_t g = (i == rb) ? (1u << rbit) : 0u;
            out_st[r * K + i] = finish_neg<ELL, PM, ENC>(&d[i * 4], g, p);
          }
        }
        if (lane == 0) trace_ev(p, t, 1);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&tail_ready[o]);
          trace_ev(p, t, 15);
        }
      }
    }
  } else if (warp == G::WARP_FETCH || warp == G::WARP_SIG) {
    if constexpr (Q) {
      if (warp == G::WARP_FETCH) {
        // ------------------------------ fetcher (Q) ------------------------------
        // Pops FD queue positions at a time; lane j waits until position base + j holds a
        // pushed (ready) item, resolves its op to ciphertext indices and publishes the entry
        // on its own (a later position may depend on an earlier one: no batch-wide wait)
        uint32_t next = 0;
        for (;;) {
          if (lane == 0) {
            uint32_t spins = 0;
            while (next + G::FD - ld_acquire_cta_smem(&s_qcnt[0]) > (uint32_t)G::FQ) {
              __nanosleep(20);
              if (++spins > FHEGPU_SPIN_LIMIT) __trap();
            }
          }
          __syncwarp();
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(qa.counters, (uint32_t)G::FD);
          base = __shfl_sync(0xffffffffu, base, 0);
          if (lane < G::FD) {
            const uint32_t pos = base + lane, e = (next + lane) % G::FQ;
            uint32_t item = Q_END;
            uint4 ent = make_uint4(0u, 0u, 0u, 0u);
            if (pos < n_items) {
              uint32_t spins = 0;
              while ((item = ld_acquire_gpu(qa.queue + pos)) == Q_EMPTY) {
                __nanosleep(64);
                if (++spins > FHEGPU_SPIN_LIMIT) __trap();
              }
              uint32_t q, ln;
              div_lanes(item, lanes, p.lanes_magic, q, ln);
              const OpRec op = ops[q];
              ent = make_uint4(op.left * lanes + ln, op.right * lanes + ln, op.out * lanes + ln, op.flags);
            }
            s_fq[e] = ent;
            s_fqi[2 * e] = item;
            st_release_cta_smem(&s_fqi[2 * e + 1], next + lane + 1);
          }
          __syncwarp();
          next += G::FD;
          if (base + G::FD > n_items) break;      // an END entry has been published
        }
      } else {
        // ------------------------------ signaler (Q) ------------------------------
        // Retires slots whose output stores completed (posted by the epilogue): decrements
        // each consumer's pending count; consumers reaching zero are pushed (release) onto
        // the queue.  (slot, consumer) pairs of a batch of slots are spread over the lanes.
        const uint32_t FULL = 0xffffffffu;
        uint32_t done = 0;
        for (;;) {
          const uint32_t fin = ld_volatile_smem(&s_qcnt[2]);
          __threadfence_block();
          const uint32_t pub = ld_volatile_smem(s_pub);
          if (pub <= done) {
            if (fin != 0u && done + 1u >= fin) break;
            __nanosleep(64);
            continue;
          }
          const uint32_t n = min(pub - done, 32u);
          uint32_t c0 = 0, cnt = 0, ln = 0;
          if (lane < n) {
            const uint32_t item = s_qitem[(done + lane) % G::QR];
            uint32_t q;
            div_lanes(item, lanes, p.lanes_magic, q, ln);
            c0 = qa.cons_off[q];
            cnt = qa.cons_off[q + 1] - c0;
          }
          uint32_t incl = cnt;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const uint32_t v = __shfl_up_sync(FULL, incl, off);
            if (lane >= off) incl += v;
          }
          const uint32_t total = __shfl_sync(FULL, incl, 31), excl = incl - cnt;
          for (uint32_t base = 0; base < total; base += 32) {
            const uint32_t idx = base + lane;
            uint32_t owner = 0;
            for (uint32_t jj = 0; jj < n; ++jj) {
              const uint32_t ej = __shfl_sync(FULL, excl, jj), cj = __shfl_sync(FULL, cnt, jj);
              if (idx >= ej && idx < ej + cj) owner = jj;
            }
            const uint32_t oc0 = __shfl_sync(FULL, c0, owner), oex = __shfl_sync(FULL, excl, owner);
            const uint32_t oln = __shfl_sync(FULL, ln, owner);
            uint32_t ci = 0;
            bool ready = false;
            if (idx < total) {
              ci = qa.cons[oc0 + idx - oex] * lanes + oln;
              ready = atom_dec_acq_rel_gpu(qa.pending + ci) == 1u;
            }
            const uint32_t m = __ballot_sync(FULL, ready);
            if (m) {
              const int leader = __ffs(m) - 1;
              uint32_t tb = 0;
              if (lane == leader) tb = atomicAdd(qa.counters + 1, (uint32_t)__popc(m));
              tb = __shfl_sync(FULL, tb, leader);
              if (ready) st_release_gpu(qa.queue + tb + __popc(m & ((1u << lane) - 1u)), ci);
            }
          }
          done += n;
          st_volatile_smem(&s_qcnt[1], done);     // producer flow control (slot ring)
        }
      }
    }
  } else if (warp >= G::WARP_BC0 && warp < G::WARP_EPI0) {
    // ------------------------------ B operand copiers (FHEGPU_WS_BCOPY) ------------------------------
    const int bc = tid - 32 * G::WARP_BC0;
    constexpr int NBT = 32 * (G::NBC_WARPS > 0 ? G::NBC_WARPS : 1);
    constexpr int B_ROWS = (G::KB + NBT - 1) / NBT;
    int b_src[B_ROWS], b_dst[B_ROWS], b_w[B_ROWS], b_j[B_ROWS];
#pragma unroll
    for (int x = 0; x < B_ROWS; ++x) {
      const int kr = bc + x * NBT;
      const int w = kr >> 5, kk = kr & 31;
      const int j = 8 * (kk & 3) + (kk >> 2);
      b_src[x] = kr < G::KB && j < ELL ? (w * ELL + j) * K : -1;
      b_dst[x] = (kr >> 3) * G::LBO + (kr & 7) * 16;
      b_w[x] = w;
      b_j[x] = j;
    }
    uint32_t t = 0;
    for (uint32_t item = blockIdx.x; Q || item < n_items; item += gridDim.x, ++t) {
      const uint32_t s = t % G::S_IN, k = t / G::S_IN, b = t & 1u, u = t >> 1;
      mbar_wait(&in_full[s], k & 1u);
      if (Q && s_qitem[t % G::QR] == Q_END) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&op_full[b]);
        break;
      }
      const uint32_t flags = s_flags[s];
      mbar_wait(&a_free[b], (u & 1u) ^ 1u);            // B(b) was last read by the MMAs of t - 2
      const uint32_t *v1 = s_in + s * 2 * G::CT_WORDS;
      const uint32_t *v2 = (flags & 4u) ? v1 : v1 + G::CT_WORDS;
      uint8_t *bb = s_b + b * G::B_BYTES;
#pragma unroll
      for (int x = 0; x < B_ROWS; ++x) {
        if (b_src[x] < 0) continue;
        uint32_t vals[K];
#pragma unroll
        for (int i = 0; i < K; ++i) vals[i] = v2[b_src[x] + i];
        if (flags & 2u) {
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
        mbar_arrive(&in_empty[s]);
      }
    }
  } else if (warp < G::WARP_EPI0) {
    // ------------------------------ operand builders ------------------------------
    const int bt = tid - 32 * G::WARP_BUILD0;           // 0 .. 128*MT-1
    const int bw = bt >> 5;
    const int quad = warp & 3;
    const int tile = bw >> 2;
    const int row = 128 * tile + 32 * quad + lane;
    const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
    const int row_blk = row / ELL, row_bit = row - row_blk * ELL;
    // B copy addressing is the same every gate: K row kr <-> bit j = 8q + o of word w with
    // kk = 4o + q (matches spread_word_sr); this thread copies rows bt and bt + 128*MT
    constexpr int B_ROWS = (G::KB + 128 * G::MT - 1) / (128 * G::MT);
    int b_src[B_ROWS], b_dst[B_ROWS], b_w[B_ROWS], b_j[B_ROWS];
#pragma unroll
    for (int x = 0; x < B_ROWS; ++x) {
      const int kr = bt + x * 128 * G::MT;
      const int w = kr >> 5, kk = kr & 31;
      const int j = 8 * (kk & 3) + (kk >> 2);
      const bool ok = kr < G::KB && j < ELL && !FHEGPU_ABL(p, 32u);   // padding rows stay zero
      b_src[x] = ok ? (w * ELL + j) * K : -1;
      b_dst[x] = (kr >> 3) * G::LBO + (kr & 7) * 16;
      b_w[x] = w;
      b_j[x] = j;
    }
    uint32_t t = 0;
    for (uint32_t item = blockIdx.x; Q || item < n_items; item += gridDim.x, ++t) {
      const uint32_t s = t % G::S_IN, k = t / G::S_IN, b = t & 1u, u = t >> 1;
      mbar_wait(&in_full[s], k & 1u);
      if (Q && s_qitem[t % G::QR] == Q_END) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&op_full[b]);
        break;
      }
      const uint32_t flags = s_flags[s];
      const bool comp1 = flags & 1u, comp2 = flags & 2u;
      if (bt == 0) trace_ev(p, t, 5);
      mbar_wait(&a_free[b], (u & 1u) ^ 1u);            // gate t-2: MMAs done, tail read out
      if (bt == 0) trace_ev(p, t, 6);
      tc_fence_after();
      const uint32_t *v1 = s_in + s * 2 * G::CT_WORDS;
      const uint32_t *v2 = (flags & 4u) ? v1 : v1 + G::CT_WORDS;   // NAND(x, x): one buffer
      uint8_t *bb = s_b + b * G::B_BYTES;
      // A (TMEM tiles): this thread's row
      if (!FHEGPU_ABL(p, 16u)) {
        uint32_t words[K];
#pragma unroll
        for (int i = 0; i < K; ++i) words[i] = v1[row * K + i];
        if (comp1) {
#pragma unroll
          for (int i = 0; i < K; ++i) words[i] = sub_mod(i == row_blk ? (1u << row_bit) : 0u, words[i], p.q);
        }
        const uint32_t a_addr = tmem_base + b * G::BUF_COLS + lane_off + G::D_COLS + tile * 8 * K;
#pragma unroll
        for (int w0 = 0; w0 < K; w0 += 4) {
          if (w0 + 4 <= K) {                     // 4 words -> one 32-column store
            uint32_t sp[32];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t one[8];
              spread_word_sr<ENC>(words[w0 + j], one);
#pragma unroll
              for (int x = 0; x < 8; ++x) sp[8 * j + x] = one[x];
            }
            tmem_st32(a_addr + 8 * w0, sp);
          } else {
#pragma unroll
            for (int w = w0; w < K; ++w) {
              uint32_t sp[8];
              spread_word_sr<ENC>(words[w], sp);
              tmem_st8(a_addr + 8 * w, sp);
            }
          }
        }
      }
      // A of the smem tail tile (TA[b] was last read by the MMAs of gate t-2: a_free above)
      if constexpr (G::TAIL > 0) {
        if (bt < G::TAIL * K && !FHEGPU_ABL(p, 16u)) {
          const int m = bt / K, w = bt - m * K;
          const int r = G::MMA_ROWS + m;
          uint32_t v = v1[r * K + w];
          if (comp1) v = sub_mod(w == r / ELL ? (1u << (r % ELL)) : 0u, v, p.q);
          uint32_t sp[8];
          spread_word_sr<ENC>(v, sp);
          uint8_t *dst = s_ta + b * G::TA_BYTES + (2 * w) * G::TA_LBO + m * 16;
          *reinterpret_cast<uint4 *>(dst) = make_uint4(sp[0], sp[1], sp[2], sp[3]);
          *reinterpret_cast<uint4 *>(dst + G::TA_LBO) = make_uint4(sp[4], sp[5], sp[6], sp[7]);
        }
      }
      // B: V2 rows copied into the MN-major canonical layout (digits = the value's bytes)
#pragma unroll
      for (int x = 0; x < (G::NBC_WARPS > 0 ? 0 : B_ROWS); ++x) {   // FHEGPU_WS_BCOPY: the copy warps do it
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
        mbar_arrive(&in_empty[s]);
      }
      if (bt == 0) trace_ev(p, t, 7);
    }
  } else {
    // ------------------------------ epilogue ------------------------------
    const int et = tid - 32 * G::WARP_EPI0;
    const int ew = et >> 5;
    const int quad = warp & 3;
    const int tile = ew >> 2;
    const int row = 128 * tile + 32 * quad + lane;
    const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
    const int row_blk = row / ELL, row_bit = row - row_blk * ELL;
    constexpr uint32_t NE_THREADS = 32 * G::NE_WARPS;
    if constexpr (G::TAIL > 0) {
      if (et == 0) mbar_arrive(&out_free[0]);          // staging 0 is free for gate 0
    }
    uint32_t t = 0;
    OpRec op_next = Q ? OpRec{} : fetch_op(ops, blockIdx.x, n_items, lanes, p.lanes_magic);
    const uint64_t pol_stream = policy_evict_first();
    for (uint32_t item = blockIdx.x; Q || item < n_items; item += gridDim.x, ++t) {
      const uint32_t b = t & 1u, u = t >> 1;
      const OpRec op_cur = op_next;
      if (!Q && et == 0) op_next = fetch_op(ops, item + gridDim.x, n_items, lanes, p.lanes_magic);
      const uint32_t o = t % G::N_OUT, ou = t / G::N_OUT;
      uint32_t *out_st = s_out + o * G::CT_WORDS;
      // staging o was released by et 0 before the previous gate's barrier (or is fresh)
      if (et == 0) trace_ev(p, t, 8);
      if (Q && et == 0 && t > 0) {
        // ready queue: post completed stores for the signaler -- all of them before this
        // thread can block (a popped item elsewhere may wait for one), else all but the newest
        if (!mbar_test(&main_done[b], u & 1u)) {
          bulk_wait_n<0>();
          post_local(s_pub, t);
        } else if (t >= FHEGPU_PUBLISH_LAG) {
          bulk_wait_n<FHEGPU_PUBLISH_LAG>();
          post_local(s_pub, t - FHEGPU_PUBLISH_LAG);
        }
      }
      if (progress != nullptr && et == 0 && t > 0) {
        // dataflow: publish finished outputs -- all of them before this thread can block
        // (a later item of this CTA may be waiting for one), else all but the newest
        if (!mbar_test(&main_done[b], u & 1u)) {
          bulk_wait_n<0>();
          publish(progress, t);
        } else if (t >= FHEGPU_PUBLISH_LAG && !FHEGPU_ABL(p, 65536u)) {
          bulk_wait_n<FHEGPU_PUBLISH_LAG>();        // stores older than LAG gates are complete
          post_local(s_pub, t - FHEGPU_PUBLISH_LAG);  // the tail warp relays it
        }
      }
      mbar_wait(&main_done[b], u & 1u);
      if (Q && s_qitem[t % G::QR] == Q_END) break;
      if (et == 0) trace_ev(p, t, 9);
      tc_fence_after();
      uint32_t d[36];
      load_acc36(tmem_base + b * G::BUF_COLS + lane_off + tile * G::NPAD, d, FHEGPU_ABL(p, 4096u));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d_free[b]);
      if (!FHEGPU_ABL(p, 64u)) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const uint32_t g = (i == row_blk) ? (1u << row_bit) : 0u;
          out_st[row * K + i] = finish_neg<ELL, PM, ENC>(&d[i * 4], g, p);
        }
      }
      fence_proxy_async_smem();
      if (et == 0) {
        // release the staging buffer gate t+1 will use (last written by gate t+1-N_OUT):
        // at most N_OUT-2 older stores may still be reading; the barrier below orders this
        // wait before any epilogue thread's writes of gate t+1
        bulk_wait_read_n<G::N_OUT - 2>();
        if constexpr (G::TAIL > 0) mbar_arrive(&out_free[(t + 1) % G::N_OUT]);
      }
      named_bar(1, NE_THREADS);
      if (et == 0) trace_ev(p, t, 11);
      if (et == 0) {
        if constexpr (G::TAIL > 0) mbar_wait(&tail_ready[o], ou & 1u);
      }
      if (Q && et == 0) {
        bulk_s2g(store + (uint64_t)s_qout[t % G::QR] * G::CT_WORDS, out_st, G::CT_BYTES);
      } else if (et == 0 && !FHEGPU_ABL(p, 512u)) {
        const uint32_t ln = lane_of(item, lanes, p.lanes_magic);
        uint32_t *dst = store + ((uint64_t)op_cur.out * lanes + ln) * G::CT_WORDS;
        if (op_cur.flags & 8u) bulk_s2g_hint(dst, out_st, G::CT_BYTES, pol_stream);
        else bulk_s2g(dst, out_st, G::CT_BYTES);
      }
    }
    if (et == 0) {
      bulk_wait_all();
      if (progress != nullptr) publish(progress, t);
      if constexpr (Q) {                  // t = slots stored; the signaler retires them and leaves
        post_local(s_pub, t);
        __threadfence_block();
        st_volatile_smem(&s_qcnt[2], t + 1);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == G::WARP_MMA) tmem_dealloc<512>(tmem_base);
}

}  // namespace tc
}  // namespace fhegpu
