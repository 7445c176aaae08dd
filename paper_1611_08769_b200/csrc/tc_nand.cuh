// tc_nand.cuh -- sm_100a tensor-core level kernel for the homomorphic NAND.
//
// Math (compact identity; reference fhe.py:325-341):
//     out[r][i] = (G[r][i] - P[r][i]) mod q,   P = C1 V2,   C1 = bits(V1)  (N x N, 0/1)
// P is a dense integer contraction (N x N binary times N x k Z_q), so it runs on
// the 5th-gen tensor cores as a u8 x u8 -> s32 GEMM:
//   * A (M = rows r, K = bit slots) : the bits of V1 spread to bytes {0, 128},
//     built in registers and written straight into TMEM (tcgen05.st) -- A never
//     touches shared memory.  K slot 32*w + 8*g + p of row r holds bit
//     j = 8g + 7 - p of word w (the multiply-spread order below); one K step of
//     the i8 MMA (32 bytes) is exactly one compact word, so K steps = k.
//   * B (K x N, MN-major in smem) : row (K slot) of bit j of word w is the byte
//     vector of V2[w*ell + j][.], digit d of value i at column n = i*NDIG + d; for
//     NDIG = 4 that is the little-endian byte image of the compact row.
//   * D (TMEM, s32) : D[r][i*NDIG + d] = 128 * sum_c bit * digit_d(V2[c][i]) <= 128*255*N.
// Epilogue per row (one thread = one TMEM lane = one row): S = (sum_d D_d << 8d) >> 7,
// Barrett mod q, out = (G - S) mod q, staged in smem and bulk-stored to HBM.
//
// Structure: persistent CTAs (2 per SM: TMEM 256 columns each), grid-striding over
// the level's (gate, lane) items; operands of item t+1 are bulk-copied (TMA
// engine, cp.async.bulk + mbarrier) while item t computes; rows beyond the last
// full 128-row tile (5 of 261 at DEFAULT) are finished on CUDA cores while the
// MMAs run.
#pragma once

#include "common.cuh"

#ifndef FHEGPU_WAIT_NS
#define FHEGPU_WAIT_NS 0   // try_wait suspend-time hint (ns); 0 = no hint
#endif
#define FHEGPU_STR2(x) #x
#define FHEGPU_STR(x) FHEGPU_STR2(x)
#if FHEGPU_WAIT_NS > 0
#define FHEGPU_WAIT_HINT ", " FHEGPU_STR(FHEGPU_WAIT_NS)
#else
#define FHEGPU_WAIT_HINT ""
#endif

namespace fhegpu {
namespace tc {

// ---- PTX wrappers -----------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
#if FHEGPU_WAIT_BACKOFF > 0
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1" FHEGPU_WAIT_HINT ";\n\t"
      "@p bra DONE_%=;\n\t"
      "nanosleep.u32 " FHEGPU_STR(FHEGPU_WAIT_BACKOFF) ";\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1" FHEGPU_WAIT_HINT ";\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
#endif
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_read_le1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(NCOLS)
               : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}

__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// D[tmem] (+)= A[tmem] * B[smem desc], kind::i8, cta_group::1.
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[smem desc] * B[smem desc], kind::i8, cta_group::1.
__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_NONE (tcgen05 format: version 1 at bits 46-47).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // descriptor version (Blackwell)
  return d;                 // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// ---- compile-time geometry ---------------------------------------------------------

template <int K, int ELL>
struct Geo {
  static constexpr int ROWS = K * ELL;
  static constexpr int FULL = ROWS / 128;
  static constexpr int REM = ROWS % 128;
  // rows past the last full 128-row tile: a third MMA with A from an 8-row smem block
  static constexpr bool SMEM_TAIL = (FULL >= 1) && (REM > 0) && (REM <= 8);
  static constexpr int MT = SMEM_TAIL ? FULL : (FULL + (REM > 0 ? 1 : 0));  // TMEM-A tiles
  static constexpr int TAIL = SMEM_TAIL ? REM : 0;
  static constexpr int MMA_ROWS = MT * 128;
  static constexpr int THREADS = 128 * MT;
  static constexpr int NDIG = (ELL + 7) / 8;               // byte digits per value
  static constexpr int NCOL = K * NDIG;
  static constexpr int NPAD = ((NCOL + 15) / 16) * 16 < 16 ? 16 : ((NCOL + 15) / 16) * 16;
  static constexpr int NCH = NPAD / 16;                    // 16-byte MN chunks of B
  static constexpr int KB = 32 * K;                        // K extent in bytes
  static constexpr uint32_t SBO = 128;                     // B: MN-chunk stride (bytes)
  static constexpr uint32_t LBO = NCH * 128;               // B: 8-row K-group stride (bytes)
  static constexpr int B_BYTES = KB * NPAD;
  static constexpr uint32_t TA_LBO = 128;                  // tail A: 16-byte K-chunk stride
  static constexpr int TA_BYTES = (KB / 16) * 128;         // 8 rows x KB, K-major core matrices
  static constexpr int WORDS = ROWS * K;
  static constexpr int CT_WORDS = (WORDS + 3) & ~3;
  static constexpr int CT_BYTES = CT_WORDS * 4;
  static constexpr int D_COLS = MT * NPAD;
  static constexpr int A_COLS = MT * 8 * K;
  static constexpr int TMEM_NEED = D_COLS + A_COLS;
  static constexpr uint32_t TMEM_COLS = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64
                                      : TMEM_NEED <= 128 ? 128 : TMEM_NEED <= 256 ? 256 : 512;
  // idesc: c_format S32 (bits 4-5 = 2), a/b u8, A K-major, B MN-major (bit 16), N>>3, M>>4.
  static constexpr uint32_t IDESC =
      (2u << 4) | (1u << 16) | ((uint32_t)(NPAD >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  // smem carve-up (bytes, 128-aligned)
  static constexpr int OFF_IN = 0;                                   // [2 stages][2 operands]
  static constexpr int OFF_B = OFF_IN + 4 * CT_BYTES;
  static constexpr int OFF_TA = ((OFF_B + B_BYTES + 127) / 128) * 128;
  static constexpr int OFF_OUT = ((OFF_TA + (TAIL ? TA_BYTES : 0) + 127) / 128) * 128;  // [2]
  static constexpr int OFF_BAR = ((OFF_OUT + 2 * CT_BYTES + 127) / 128) * 128;
  static constexpr int SMEM = OFF_BAR + 128;
  static_assert(K <= 16 && ELL <= 31 && ELL >= 17, "geometry out of range");
  static_assert(NPAD <= 256, "N too large for one MMA");
  static_assert(TMEM_NEED <= 256, "TMEM budget is 256 columns per CTA (2 CTAs/SM)");
  static_assert(!TAIL || 8 * K >= NPAD, "tail accumulator reuses tile-0 A columns");
  static_assert(CT_BYTES % 16 == 0, "bulk copies need 16-byte multiples");
};

// byte n of the B row built from effective values vals[0..K-1]
template <int K, int NDIG>
__device__ __forceinline__ uint32_t b_word(const uint32_t *vals, int wi) {
  if constexpr (NDIG == 4) {
    return wi < K ? vals[wi] : 0u;
  } else {
    uint32_t out = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int n = 4 * wi + b;
      const int i = n / NDIG, d = n % NDIG;
      const uint32_t byte = (i < K) ? ((vals[i] >> (8 * d)) & 0xFFu) : 0u;
      out |= byte << (8 * b);
    }
    return out;
  }
}

// The 32 bits of one compact word spread to 32 u8 in {0, 128}: byte slot 8g + p holds
// bit 8g + 7 - p (multiply-spread: copies at stride 9 never overlap, so no carries).
__device__ __forceinline__ void spread_word(uint32_t w, uint32_t (&out)[8]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const uint32_t x = __byte_perm(w, 0u, 0x4440u + g);
    out[2 * g] = (x * 0x08040201u) & 0x80808080u;      // bits 7,6,5,4
    out[2 * g + 1] = (x * 0x80402010u) & 0x80808080u;  // bits 3,2,1,0
  }
}

// Reduce one output value.  d[] holds the NDIG s32 accumulators of column i
// (each 128 * digit sum).  Returns (G - S) mod q.
template <int ELL, int NDIG, bool PM>
__device__ __forceinline__ uint32_t finish_value(const uint32_t *d, uint32_t g, const DevParams &p) {
  uint32_t r;
  if constexpr (PM && NDIG == 4) {
    // S = A + B 2^16, A = S0 + S1 2^8, B = S2 + S3 2^8 (both < 2^26);
    // 2^ELL = c (mod q):  S = A + Bl 2^16 + c Bh  with B = Bh 2^(ELL-16) + Bl.  (< 2q, host-checked)
    const uint32_t a = (d[0] >> 7) + (d[1] << 1);
    const uint32_t b = (d[2] >> 7) + (d[3] << 1);
    const uint32_t bl = b & ((1u << (ELL - 16)) - 1u);
    const uint32_t bh = b >> (ELL - 16);
    const uint32_t t = a + (bl << 16) + p.pm_c * bh;
    r = t >= p.q ? t - p.q : t;
  } else {
    uint64_t s = 0;
#pragma unroll
    for (int dg = 0; dg < NDIG; ++dg) s += (uint64_t)d[dg] << (8 * dg);
    r = mod_u64(s >> 7, p.q, p.mu);
  }
  return sub_mod(g, r, p.q);
}

template <int K, int ELL, bool PM>
__global__ void __launch_bounds__(Geo<K, ELL>::THREADS, 2)
level_tc_kernel(uint32_t *__restrict__ store, const OpRec *__restrict__ ops, uint32_t n_ops,
                uint32_t lanes, DevParams p) {
  using G = Geo<K, ELL>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t *s_in = reinterpret_cast<uint32_t *>(smem + G::OFF_IN);
  uint8_t *s_b = smem + G::OFF_B;
  uint8_t *s_ta = smem + G::OFF_TA;
  uint32_t *s_out = reinterpret_cast<uint32_t *>(smem + G::OFF_OUT);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + G::OFF_BAR);  // 0,1 loads; 2 main; 3 tail
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + G::OFF_BAR + 64);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const uint64_t n_items = (uint64_t)n_ops * lanes;

  // programmatic dependent launch: the next level's CTAs may take SMs as ours leave and
  // run their prologue (TMEM alloc, barrier init, smem zeroing) under our tail
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 0) tmem_alloc<G::TMEM_COLS>(tmem_slot);
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  // zero once: B (its K-padding rows stay zero), tail A (rows TAIL..7), output padding
  for (int w = tid; w < G::B_BYTES / 4; w += G::THREADS) reinterpret_cast<uint32_t *>(s_b)[w] = 0u;
  if constexpr (G::TAIL > 0)
    for (int w = tid; w < G::TA_BYTES / 4; w += G::THREADS) reinterpret_cast<uint32_t *>(s_ta)[w] = 0u;
  for (int w = tid; w < 2 * G::CT_WORDS; w += G::THREADS) s_out[w] = 0u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t lane_off = ((uint32_t)(warp & 3) * 32u) << 16;  // this warp's TMEM lanes
  const int tile = warp >> 2;                                      // MMA tile of this thread's row
  const int row = tid;                                             // ciphertext row of this thread
  const int row_blk = row / ELL, row_bit = row - row_blk * ELL;
  // every ciphertext access comes after the previous level completed (no-op without PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");

  auto item_ptrs = [&](uint64_t item, const uint32_t *&a, const uint32_t *&b, uint32_t *&o,
                       uint32_t &flags) {
    const uint32_t op_i = (uint32_t)(item / lanes);
    const uint32_t lane = (uint32_t)(item - (uint64_t)op_i * lanes);
    const OpRec op = ops[op_i];
    a = store + ((uint64_t)op.left * lanes + lane) * G::CT_WORDS;
    b = store + ((uint64_t)op.right * lanes + lane) * G::CT_WORDS;
    o = store + ((uint64_t)op.out * lanes + lane) * G::CT_WORDS;
    flags = op.flags;
  };

  if (tid == 0 && blockIdx.x < n_items) {
    const uint32_t *a, *b;
    uint32_t *o, f;
    item_ptrs(blockIdx.x, a, b, o, f);
    mbar_expect_tx(&bar[0], 2 * G::CT_BYTES);
    bulk_g2s(s_in, a, G::CT_BYTES, &bar[0]);
    bulk_g2s(s_in + G::CT_WORDS, b, G::CT_BYTES, &bar[0]);
  }

  uint32_t t = 0;
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
    const uint32_t stage = t & 1u;
    const uint32_t *gA, *gB;
    uint32_t *gO, flags;
    item_ptrs(item, gA, gB, gO, flags);
    if (tid == 0) {
      const uint64_t nxt = item + gridDim.x;
      if (nxt < n_items) {
        const uint32_t *a, *b;
        uint32_t *o, f;
        item_ptrs(nxt, a, b, o, f);
        uint32_t *dst = s_in + (stage ^ 1u) * 2 * G::CT_WORDS;
        mbar_expect_tx(&bar[stage ^ 1u], 2 * G::CT_BYTES);
        bulk_g2s(dst, a, G::CT_BYTES, &bar[stage ^ 1u]);
        bulk_g2s(dst + G::CT_WORDS, b, G::CT_BYTES, &bar[stage ^ 1u]);
      }
      bulk_wait_read_le1();  // output staging of item t-2 has been read out
    }
    mbar_wait(&bar[stage], (t >> 1) & 1u);
    const uint32_t *v1 = s_in + stage * 2 * G::CT_WORDS;
    const uint32_t *v2 = v1 + G::CT_WORDS;
    const bool comp1 = flags & 1u, comp2 = flags & 2u;
    uint32_t *out_st = s_out + stage * G::CT_WORDS;

    // ---- phase 1a: B operand: one K row (= one compact row of V2) per thread ----
    for (int kr = tid; kr < G::KB; kr += G::THREADS) {
      const int w = kr >> 5, kk = kr & 31;
      const int j = (kk & ~7) + 7 - (kk & 7);
      if (j >= ELL) continue;                 // K padding rows: zero since init
      const int c = w * ELL + j;
      uint32_t vals[K];
#pragma unroll
      for (int i = 0; i < K; ++i) vals[i] = v2[c * K + i];
      if (comp2) {                            // (G - V) mod q, G[c][i] = 2^j iff i == w
#pragma unroll
        for (int i = 0; i < K; ++i) vals[i] = sub_mod(i == w ? (1u << j) : 0u, vals[i], p.q);
      }
      uint8_t *dst = s_b + (kr >> 3) * G::LBO + (kr & 7) * 16;
#pragma unroll
      for (int ch = 0; ch < G::NCH; ++ch) {
        uint4 val;
        val.x = b_word<K, G::NDIG>(vals, 4 * ch + 0);
        val.y = b_word<K, G::NDIG>(vals, 4 * ch + 1);
        val.z = b_word<K, G::NDIG>(vals, 4 * ch + 2);
        val.w = b_word<K, G::NDIG>(vals, 4 * ch + 3);
        *reinterpret_cast<uint4 *>(dst + ch * G::SBO) = val;
      }
    }

    // ---- phase 1b: A operand of the TMEM tiles: this thread's row, spread, into TMEM ----
    {
      uint32_t words[K];
#pragma unroll
      for (int i = 0; i < K; ++i) words[i] = (row < G::ROWS) ? v1[row * K + i] : 0u;
      if (comp1 && row < G::ROWS) {
#pragma unroll
        for (int i = 0; i < K; ++i)
          words[i] = sub_mod(i == row_blk ? (1u << row_bit) : 0u, words[i], p.q);
      }
      const uint32_t a_addr = tmem_base + lane_off + G::D_COLS + tile * 8 * K;
#pragma unroll
      for (int w = 0; w < K; ++w) {
        uint32_t sp[8];
        spread_word(words[w], sp);
        tmem_st8(a_addr + 8 * w, sp);
      }
    }
    // ---- phase 1c: A operand of the smem tail tile (rows MMA_ROWS .. ROWS-1) ----
    if constexpr (G::TAIL > 0) {
      if (tid < G::TAIL * K) {
        const int m = tid / K, w = tid - m * K;
        const int r = G::MMA_ROWS + m;
        uint32_t v = v1[r * K + w];
        if (comp1) v = sub_mod(w == r / ELL ? (1u << (r % ELL)) : 0u, v, p.q);
        uint32_t sp[8];
        spread_word(v, sp);
        uint8_t *dst = s_ta + (2 * w) * G::TA_LBO + m * 16;
        *reinterpret_cast<uint4 *>(dst) = make_uint4(sp[0], sp[1], sp[2], sp[3]);
        *reinterpret_cast<uint4 *>(dst + G::TA_LBO) = make_uint4(sp[4], sp[5], sp[6], sp[7]);
      }
    }
    tmem_wait_st();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();

    // ---- phase 2: MMA issue (one thread) ----
    if (tid == 0) {
      tc_fence_after();
      const uint32_t b_base = smem_u32(s_b);
#pragma unroll
      for (int mt = 0; mt < G::MT; ++mt) {
        const uint32_t d_t = tmem_base + mt * G::NPAD;
        const uint32_t a_t = tmem_base + G::D_COLS + mt * 8 * K;
#pragma unroll
        for (int s = 0; s < K; ++s) {
          const uint64_t bd = (p.dbg & 1u)
                                  ? smem_desc(b_base + s * 4 * G::LBO, G::SBO, G::LBO)
                                  : smem_desc(b_base + s * 4 * G::LBO, G::LBO, G::SBO);
          mma_i8_ts(d_t, a_t + 8 * s, bd, G::IDESC, s > 0 ? 1u : 0u);
        }
      }
      mma_commit(&bar[2]);
      if constexpr (G::TAIL > 0) {
        // tail accumulator lives in tile 0's A columns: wait until those MMAs are done
        mbar_wait(&bar[2], t & 1u);
        tc_fence_after();
        const uint32_t ta_base = smem_u32(s_ta);
        const uint32_t d_tail = tmem_base + G::D_COLS;
#pragma unroll
        for (int s = 0; s < K; ++s) {
          const uint64_t ad = smem_desc(ta_base + s * 2 * G::TA_LBO, G::TA_LBO, 0u);
          const uint64_t bd = smem_desc(b_base + s * 4 * G::LBO, G::LBO, G::SBO);
          mma_i8_ss(d_tail, ad, bd, G::IDESC, s > 0 ? 1u : 0u);
        }
        mma_commit(&bar[3]);
      }
    }

    // ---- phase 3: epilogue, TMEM -> registers -> (G - S) mod q -> smem ----
    mbar_wait(&bar[2], t & 1u);
    tc_fence_after();
    {
      uint32_t d[G::NPAD];
#pragma unroll
      for (int c = 0; c < G::NCH; ++c) {
        uint32_t chunk[16];
        tmem_ld16(tmem_base + lane_off + tile * G::NPAD + 16 * c, chunk);
#pragma unroll
        for (int x = 0; x < 16; ++x) d[16 * c + x] = chunk[x];
      }
      tmem_wait_ld();
      if (row < G::ROWS) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const uint32_t g = (i == row_blk) ? (1u << row_bit) : 0u;
          out_st[row * K + i] = finish_value<ELL, G::NDIG, PM>(&d[i * G::NDIG], g, p);
        }
      }
    }
    if constexpr (G::TAIL > 0) {
      if (warp == 0) {
        mbar_wait(&bar[3], t & 1u);
        tc_fence_after();
        uint32_t d[G::NPAD];
#pragma unroll
        for (int c = 0; c < G::NCH; ++c) {
          uint32_t chunk[16];
          tmem_ld16(tmem_base + G::D_COLS + 16 * c, chunk);
#pragma unroll
          for (int x = 0; x < 16; ++x) d[16 * c + x] = chunk[x];
        }
        tmem_wait_ld();
        if (tid < G::TAIL) {
          const int r = G::MMA_ROWS + tid;
          const int rb = r / ELL, rbit = r - rb * ELL;
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const uint32_t g = (i == rb) ? (1u << rbit) : 0u;
            out_st[r * K + i] = finish_value<ELL, G::NDIG, PM>(&d[i * G::NDIG], g, p);
          }
        }
      }
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) bulk_s2g(gO, out_st, G::CT_BYTES);
  }

  if (tid == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<G::TMEM_COLS>(tmem_base);
}

}  // namespace tc
}  // namespace fhegpu
