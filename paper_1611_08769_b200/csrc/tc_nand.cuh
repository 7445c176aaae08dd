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
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
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
  static constexpr bool CORE_TAIL = (FULL >= 1) && (REM > 0) && (REM <= 16);
  static constexpr int MT = CORE_TAIL ? FULL : (FULL + (REM > 0 ? 1 : 0));  // MMA tiles
  static constexpr int TAIL = CORE_TAIL ? REM : 0;        // rows done on CUDA cores
  static constexpr int MMA_ROWS = MT * 128;
  static constexpr int THREADS = 128 * MT;
  static constexpr int NDIG = (ELL + 7) / 8;               // byte digits per value
  static constexpr int NCOL = K * NDIG;
  static constexpr int NPAD = ((NCOL + 15) / 16) * 16 < 16 ? 16 : ((NCOL + 15) / 16) * 16;
  static constexpr int NCH = NPAD / 16;                    // 16-byte MN chunks of B
  static constexpr int KB = 32 * K;                        // K extent in bytes
  static constexpr uint32_t SBO = 128;                     // MN-chunk stride (bytes)
  static constexpr uint32_t LBO = NCH * 128;               // 8-row K-group stride (bytes)
  static constexpr int B_BYTES = KB * NPAD;
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
  // tail split: each (tail row, column) sum is shared by TSPLIT threads
  static constexpr int TSPLIT = 4;
  // smem carve-up (bytes, all 128-aligned)
  static constexpr int OFF_IN = 0;                                   // [2 stages][2 operands]
  static constexpr int OFF_B = OFF_IN + 4 * CT_BYTES;
  static constexpr int OFF_OUT = ((OFF_B + B_BYTES + 127) / 128) * 128;  // [2]
  static constexpr int OFF_BAR = ((OFF_OUT + 2 * CT_BYTES + 127) / 128) * 128;
  static constexpr int SMEM = OFF_BAR + 128;
  static_assert(K <= 16 && ELL <= 31 && ELL >= 4, "geometry out of range");
  static_assert(NPAD <= 256, "N too large for one MMA");
  static_assert(TMEM_NEED <= 256, "TMEM budget is 256 columns per CTA (2 CTAs/SM)");
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

template <int K, int ELL>
__global__ void __launch_bounds__(Geo<K, ELL>::THREADS, 2)
level_tc_kernel(uint32_t *__restrict__ store, const OpRec *__restrict__ ops, uint32_t n_ops,
                uint32_t lanes, DevParams p) {
  using G = Geo<K, ELL>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t *s_in = reinterpret_cast<uint32_t *>(smem + G::OFF_IN);
  uint8_t *s_b = smem + G::OFF_B;
  uint32_t *s_out = reinterpret_cast<uint32_t *>(smem + G::OFF_OUT);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + G::OFF_BAR);  // [0,1] loads, [2] mma
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + G::OFF_BAR + 64);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const uint64_t n_items = (uint64_t)n_ops * lanes;

  if (warp == 0) tmem_alloc<G::TMEM_COLS>(tmem_slot);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  // zero output staging once (its padding words are stored with every ciphertext)
  for (int w = tid; w < 2 * G::CT_WORDS; w += G::THREADS) s_out[w] = 0u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t lane_quad = (uint32_t)(warp & 3) * 32u;
  const uint32_t t_row_addr = tmem_base + (lane_quad << 16);  // this warp's TMEM lanes
  const int tile = warp >> 2;                                  // MMA tile of this thread's row
  const int row = tid;                                         // row within the ciphertext

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

    // ---- phase 1a: B operand (MN-major canonical layout, K slots permuted) ----
    for (int e = tid; e < G::KB * G::NCH; e += G::THREADS) {
      const int kr = e / G::NCH, ch = e - kr * G::NCH;
      const int w = kr >> 5, kk = kr & 31;
      const int j = (kk & ~7) + 7 - (kk & 7);
      uint4 val = make_uint4(0u, 0u, 0u, 0u);
      if (j < ELL) {
        const int c = w * ELL + j;
        if constexpr (G::NDIG == 4) {
          uint32_t q4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int wi = 4 * ch + u;
            uint32_t v = 0u;
            if (wi < K) {
              v = v2[c * K + wi];
              if (comp2) v = sub_mod(gadget_ct<ELL>(c, wi), v, p.q);
            }
            q4[u] = v;
          }
          val = make_uint4(q4[0], q4[1], q4[2], q4[3]);
        } else {
          uint32_t vals[K];
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const uint32_t v = v2[c * K + i];
            vals[i] = comp2 ? sub_mod(gadget_ct<ELL>(c, i), v, p.q) : v;
          }
          val.x = b_word<K, G::NDIG>(vals, 4 * ch + 0);
          val.y = b_word<K, G::NDIG>(vals, 4 * ch + 1);
          val.z = b_word<K, G::NDIG>(vals, 4 * ch + 2);
          val.w = b_word<K, G::NDIG>(vals, 4 * ch + 3);
        }
      }
      uint8_t *dst = s_b + (kr >> 3) * G::LBO + ch * G::SBO + (kr & 7) * 16;
      *reinterpret_cast<uint4 *>(dst) = val;
    }

    // ---- phase 1b: A operand, bits of row `row` spread to bytes, into TMEM ----
    {
      uint32_t words[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        uint32_t v = 0u;
        if (row < G::ROWS) {
          v = v1[row * K + i];
          if (comp1) v = sub_mod(gadget_ct<ELL>(row, i), v, p.q);
        }
        words[i] = v;
      }
      const uint32_t a_col = tmem_base + G::D_COLS + tile * 8 * K;
#pragma unroll
      for (int w = 0; w < K; ++w) {
        uint32_t spread[8];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint32_t x = (words[w] >> (8 * g)) & 0xFFu;
          spread[2 * g] = (x * 0x08040201u) & 0x80808080u;      // bits 7,6,5,4 -> bytes 0..3
          spread[2 * g + 1] = (x * 0x80402010u) & 0x80808080u;  // bits 3,2,1,0 -> bytes 0..3
        }
        tmem_st8((t_row_addr & 0xFFFF0000u) | ((a_col + 8 * w) & 0xFFFFu), spread);
      }
    }
    tmem_wait_st();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();

    // ---- phase 2: MMA issue (one thread) || CUDA-core tail rows ----
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
    }
    if constexpr (G::TAIL > 0) {
      constexpr int UNITS = G::TAIL * K;
      const int unit = tid / G::TSPLIT, sub = tid % G::TSPLIT;
      const bool active = unit < UNITS;
      const int tr = G::MMA_ROWS + (active ? unit / K : 0), i = active ? unit % K : 0;
      uint64_t acc = 0;
      if (active) {
        for (int blk = 0; blk < K; ++blk) {
          uint32_t wv = v1[tr * K + blk];
          if (comp1) wv = sub_mod(gadget_ct<ELL>(tr, blk), wv, p.q);
          for (int j = sub; j < ELL; j += G::TSPLIT) {
            const int c = blk * ELL + j;
            uint32_t v = v2[c * K + i];
            if (comp2) v = sub_mod(gadget_ct<ELL>(c, i), v, p.q);
            acc += ((wv >> j) & 1u) ? v : 0u;
          }
        }
      }
#pragma unroll
      for (int o = 1; o < G::TSPLIT; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (active && sub == 0)
        out_st[tr * K + i] = sub_mod(gadget_ct<ELL>(tr, i), mod_u64(acc, p.q, p.mu), p.q);
    }

    // ---- phase 3: epilogue, TMEM -> registers -> (G - S) mod q -> smem ----
    mbar_wait(&bar[2], t & 1u);
    tc_fence_after();
    {
      uint32_t d[G::NPAD];
#pragma unroll
      for (int c = 0; c < G::NCH; ++c) {
        uint32_t chunk[16];
        tmem_ld16((t_row_addr & 0xFFFF0000u) | ((tmem_base + tile * G::NPAD + 16 * c) & 0xFFFFu),
                  chunk);
#pragma unroll
        for (int x = 0; x < 16; ++x) d[16 * c + x] = chunk[x];
      }
      tmem_wait_ld();
      if (row < G::ROWS) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          uint64_t s = 0;
#pragma unroll
          for (int dg = 0; dg < G::NDIG; ++dg) s += (uint64_t)d[i * G::NDIG + dg] << (8 * dg);
          s >>= 7;  // A bytes are 128
          out_st[row * K + i] = sub_mod(gadget_ct<ELL>(row, i), mod_u64(s, p.q, p.mu), p.q);
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
