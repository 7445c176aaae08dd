// tc_nand_ws.cuh -- warp-specialised, pipelined tcgen05 level kernel (v3).
//
// Same math as tc_nand.cuh (compact NAND: out = (G - bits(V1) V2) mod q, the
// product on the tensor cores as a u8 GEMM), restructured so the phases of
// different gates overlap inside one persistent CTA per SM:
//
//   warp 0        producer : cp.async.bulk of both operands into an S_IN-stage ring
//   warp 1        MMA      : one thread issues tcgen05.mma (2 TMEM-A tiles + smem-A tail)
//   warps 2..9    builders : B operand (smem, MN-major) + A operand (bits -> s8 {0,-1},
//                            tcgen05.st into TMEM) for gate t while the MMA runs gate t-1
//   warps 10..17  epilogue : tcgen05.ld of gate t-1's accumulators, mod-q fold,
//                            bulk store -- while gate t builds
//
// TMEM (512 columns): two buffers of {D tile0, D tile1, A tile0, A tile1} (240 columns each);
// the 5-row tail accumulates into the tile-0 A columns of its own buffer once the tile
// MMAs are done.  Barriers (mbarrier): in_full/in_empty per input stage, op_full per
// buffer (builders -> MMA), main_done/tail_done per buffer (tcgen05.commit -> epilogue
// and MMA), epi_done per buffer (epilogue -> builders of gate t+2).
//
// A operand: word w of row r spreads into 8 u32 (32 K slots).  Output o holds, in byte q,
// bit 8q + o of w replicated to 0x00 / 0xFF by a sign-replicating PRMT of (w << (7 - o)),
// i.e. the s8 value 0 or -1; D = -(sum of digits) and the epilogue negates.  K slot
// 4o + q of word w therefore pairs with V2 row w * ELL + 8q + o in B.
#pragma once

#include "tc_nand.cuh"

namespace fhegpu {
namespace tc {

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 32 bits of w -> 32 s8 K slots {0, -1}: out[o] byte q = -(bit 8q + o).
__device__ __forceinline__ uint32_t prmt_sign(uint32_t x) {
  uint32_t r;  // default-mode prmt: selector nibble bit 3 replicates the selected byte's msb
  asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(x));
  return r;
}

__device__ __forceinline__ void spread_word_sr(uint32_t w, uint32_t (&out)[8]) {
#pragma unroll
  for (int o = 0; o < 8; ++o) out[o] = prmt_sign(w << (7 - o));
}

template <int K, int ELL, bool PM>
struct GeoWS {
  using B = Geo<K, ELL>;
  static constexpr int ROWS = B::ROWS;
  static constexpr int MT = B::MT;
  static constexpr int TAIL = B::TAIL;
  static constexpr int MMA_ROWS = B::MMA_ROWS;
  static constexpr int NPAD = B::NPAD, NCH = B::NCH, KB = B::KB, NDIG = B::NDIG;
  static constexpr uint32_t SBO = B::SBO, LBO = B::LBO, TA_LBO = B::TA_LBO;
  static constexpr int B_BYTES = B::B_BYTES, TA_BYTES = B::TA_BYTES;
  static constexpr int CT_WORDS = B::CT_WORDS, CT_BYTES = B::CT_BYTES;
  static constexpr int D_COLS = B::D_COLS;                 // per buffer
  static constexpr int BUF_COLS = 256;                      // buffer stride in TMEM columns
  static constexpr int NB_WARPS = 4 * MT, NE_WARPS = 4 * MT;
  static constexpr int WARP_BUILD0 = 2, WARP_EPI0 = 2 + NB_WARPS;
  static constexpr int THREADS = 32 * (2 + NB_WARPS + NE_WARPS);
  static constexpr int S_IN = 3;
  // idesc: S32 accumulator, A s8 (bits 7-9 = 1), B u8, A K-major, B MN-major, N>>3, M>>4
  static constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 16) |
                                    ((uint32_t)(NPAD >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  static constexpr int OFF_IN = 0;
  static constexpr int OFF_B = OFF_IN + S_IN * 2 * CT_BYTES;
  static constexpr int OFF_TA = ((OFF_B + 2 * B_BYTES + 127) / 128) * 128;
  static constexpr int OFF_OUT = ((OFF_TA + (TAIL ? 2 * TA_BYTES : 0) + 127) / 128) * 128;
  static constexpr int OFF_BAR = ((OFF_OUT + 2 * CT_BYTES + 127) / 128) * 128;
  static constexpr int SMEM = OFF_BAR + 256;
  static_assert(NDIG == 4 && MT >= 1, "warp-specialised kernel covers 25..31-bit q with >= 128 rows");
  static_assert(B::D_COLS + B::A_COLS <= BUF_COLS, "two TMEM buffers must fit 512 columns");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

// Negated-digit epilogue (A = -bits): d[] are -(digit sums).
template <int ELL, bool PM>
__device__ __forceinline__ uint32_t finish_neg(const uint32_t *d, uint32_t g, const DevParams &p) {
  uint32_t r;
  if constexpr (PM) {
    const uint32_t a = 0u - (d[0] + (d[1] << 8));   // S0 + S1 2^8  (< 2^26)
    const uint32_t b = 0u - (d[2] + (d[3] << 8));   // S2 + S3 2^8
    const uint32_t t = a + ((b & ((1u << (ELL - 16)) - 1u)) << 16) + p.pm_c * (b >> (ELL - 16));
    r = min(t, t - p.q);                            // t < 2q
  } else {
    const int64_t s = -((int64_t)(int32_t)d[0] + ((int64_t)(int32_t)d[1] << 8) +
                        ((int64_t)(int32_t)d[2] << 16) + ((int64_t)(int32_t)d[3] << 24));
    r = mod_u64((uint64_t)s, p.q, p.mu);
  }
  const uint32_t x = g - r;
  return min(x, x + p.q);                           // (g - r) mod q for g, r < q
}

template <int K, int ELL, bool PM>
__global__ void __launch_bounds__(GeoWS<K, ELL, PM>::THREADS, 1)
level_tc_ws_kernel(uint32_t *__restrict__ store, const OpRec *__restrict__ ops, uint32_t n_ops,
                   uint32_t lanes, DevParams p) {
  using G = GeoWS<K, ELL, PM>;
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
  uint64_t *tail_done = main_done + 2;        // [2]
  uint64_t *epi_done = tail_done + 2;         // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(epi_done + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t n_items = n_ops * lanes;     // host guarantees < 2^32

  if (warp == 1) tmem_alloc<512>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < G::S_IN; ++i) {
      mbar_init(&in_full[i], 1);
      mbar_init(&in_empty[i], G::NB_WARPS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&op_full[i], G::NB_WARPS);
      mbar_init(&main_done[i], 1);
      mbar_init(&tail_done[i], 1);
      mbar_init(&epi_done[i], G::NE_WARPS);
    }
    fence_mbar_init();
  }
  for (int w = tid; w < 2 * G::B_BYTES / 4; w += G::THREADS) reinterpret_cast<uint32_t *>(s_b)[w] = 0u;
  if constexpr (G::TAIL > 0)
    for (int w = tid; w < 2 * G::TA_BYTES / 4; w += G::THREADS) reinterpret_cast<uint32_t *>(s_ta)[w] = 0u;
  for (int w = tid; w < 2 * G::CT_WORDS; w += G::THREADS) s_out[w] = 0u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      uint32_t t = 0;
      for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
        const uint32_t s = t % G::S_IN, k = t / G::S_IN;
        mbar_wait(&in_empty[s], (k & 1u) ^ 1u);
        const uint32_t op_i = item / lanes, ln = item - op_i * lanes;
        const OpRec op = ops[op_i];
        uint32_t *dst = s_in + s * 2 * G::CT_WORDS;
        mbar_expect_tx(&in_full[s], 2 * G::CT_BYTES);
        bulk_g2s(dst, store + ((uint64_t)op.left * lanes + ln) * G::CT_WORDS, G::CT_BYTES, &in_full[s]);
        bulk_g2s(dst + G::CT_WORDS, store + ((uint64_t)op.right * lanes + ln) * G::CT_WORDS,
                 G::CT_BYTES, &in_full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      uint32_t t = 0;
      for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
        const uint32_t b = t & 1u, u = t >> 1;
        mbar_wait(&op_full[b], u & 1u);
        tc_fence_after();
        const uint32_t tb = tmem_base + b * G::BUF_COLS;
        const uint32_t b_base = smem_u32(s_b + b * G::B_BYTES);
        const uint32_t idesc = (p.dbg & 8u) ? (G::IDESC & ~(7u << 7)) : G::IDESC;
#pragma unroll
        for (int mt = 0; mt < G::MT; ++mt) {
#pragma unroll
          for (int s = 0; s < K; ++s) {
            const uint64_t bd = smem_desc(b_base + s * 4 * G::LBO, G::LBO, G::SBO);
            mma_i8_ts(tb + mt * G::NPAD, tb + G::D_COLS + mt * 8 * K + 8 * s, bd, idesc,
                      s > 0 ? 1u : 0u);
          }
        }
        mma_commit(&main_done[b]);
        if constexpr (G::TAIL > 0) {
          mbar_wait(&main_done[b], u & 1u);       // tail accumulates into tile-0 A columns
          tc_fence_after();
          const uint32_t ta = smem_u32(s_ta + b * G::TA_BYTES);
#pragma unroll
          for (int s = 0; s < K; ++s) {
            const uint64_t ad = smem_desc(ta + s * 2 * G::TA_LBO, G::TA_LBO, 0u);
            const uint64_t bd = smem_desc(b_base + s * 4 * G::LBO, G::LBO, G::SBO);
            mma_i8_ss(tb + G::D_COLS, ad, bd, idesc, s > 0 ? 1u : 0u);
          }
          mma_commit(&tail_done[b]);
        }
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
    uint32_t t = 0;
    for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
      const uint32_t s = t % G::S_IN, k = t / G::S_IN, b = t & 1u, u = t >> 1;
      const uint32_t flags = ops[item / lanes].flags;
      const bool comp1 = flags & 1u, comp2 = flags & 2u;
      mbar_wait(&in_full[s], k & 1u);
      mbar_wait(&epi_done[b], (u & 1u) ^ 1u);          // gate t-2 is out of buffer b
      tc_fence_after();
      const uint32_t *v1 = s_in + s * 2 * G::CT_WORDS;
      const uint32_t *v2 = v1 + G::CT_WORDS;
      uint8_t *bb = s_b + b * G::B_BYTES;
      // B: K row kr <-> bit j = 8q + o of word w, kk = 4o + q
      for (int kr = bt; kr < G::KB; kr += 128 * G::MT) {
        const int w = kr >> 5, kk = kr & 31;
        const int j = (p.dbg & 8u) ? (kk & ~7) + 7 - (kk & 7) : 8 * (kk & 3) + (kk >> 2);
        if (j >= ELL) continue;                         // padding rows stay zero
        const int c = w * ELL + j;
        uint32_t vals[K];
#pragma unroll
        for (int i = 0; i < K; ++i) vals[i] = v2[c * K + i];
        if (comp2) {
#pragma unroll
          for (int i = 0; i < K; ++i) vals[i] = sub_mod(i == w ? (1u << j) : 0u, vals[i], p.q);
        }
        uint8_t *dst = bb + (kr >> 3) * G::LBO + (kr & 7) * 16;
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
      // A (TMEM tiles): this thread's row
      {
        uint32_t words[K];
#pragma unroll
        for (int i = 0; i < K; ++i) words[i] = v1[row * K + i];
        if (comp1) {
#pragma unroll
          for (int i = 0; i < K; ++i) words[i] = sub_mod(i == row_blk ? (1u << row_bit) : 0u, words[i], p.q);
        }
        const uint32_t a_addr = tmem_base + b * G::BUF_COLS + lane_off + G::D_COLS + tile * 8 * K;
#pragma unroll
        for (int w = 0; w < K; ++w) {
          uint32_t sp[8];
          if (p.dbg & 8u) spread_word(words[w], sp); else spread_word_sr(words[w], sp);
          tmem_st8(a_addr + 8 * w, sp);
        }
      }
      // A (smem tail tile)
      if constexpr (G::TAIL > 0) {
        if (bt < G::TAIL * K) {
          const int m = bt / K, w = bt - m * K;
          const int r = G::MMA_ROWS + m;
          uint32_t v = v1[r * K + w];
          if (comp1) v = sub_mod(w == r / ELL ? (1u << (r % ELL)) : 0u, v, p.q);
          uint32_t sp[8];
          if (p.dbg & 8u) spread_word(v, sp); else spread_word_sr(v, sp);
          uint8_t *dst = s_ta + b * G::TA_BYTES + (2 * w) * G::TA_LBO + m * 16;
          *reinterpret_cast<uint4 *>(dst) = make_uint4(sp[0], sp[1], sp[2], sp[3]);
          *reinterpret_cast<uint4 *>(dst + G::TA_LBO) = make_uint4(sp[4], sp[5], sp[6], sp[7]);
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
    const bool tail_warp = (G::TAIL > 0) && tile == 0 && quad == 0;
    constexpr uint32_t NE_THREADS = 32 * G::NE_WARPS;
    uint32_t t = 0;
    for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
      const uint32_t b = t & 1u, u = t >> 1;
      uint32_t *out_st = s_out + b * G::CT_WORDS;
      if (et == 0) bulk_wait_read_le1();               // gate t-2's store has read its staging
      named_bar(1, NE_THREADS);
      mbar_wait(&main_done[b], u & 1u);
      tc_fence_after();
      const uint32_t tb = tmem_base + b * G::BUF_COLS;
      {
        uint32_t d[G::NPAD];
#pragma unroll
        for (int c = 0; c < G::NCH; ++c) {
          uint32_t chunk[16];
          tmem_ld16(tb + lane_off + tile * G::NPAD + 16 * c, chunk);
#pragma unroll
          for (int x = 0; x < 16; ++x) d[16 * c + x] = chunk[x];
        }
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const uint32_t g = (i == row_blk) ? (1u << row_bit) : 0u;
          out_st[row * K + i] = (p.dbg & 8u) ? finish_value<ELL, 4, PM>(&d[i * 4], g, p)
                                             : finish_neg<ELL, PM>(&d[i * 4], g, p);
        }
      }
      if constexpr (G::TAIL > 0) {
        if (tail_warp) {
          mbar_wait(&tail_done[b], u & 1u);
          tc_fence_after();
          uint32_t d[G::NPAD];
#pragma unroll
          for (int c = 0; c < G::NCH; ++c) {
            uint32_t chunk[16];
            tmem_ld16(tb + G::D_COLS + 16 * c, chunk);
#pragma unroll
            for (int x = 0; x < 16; ++x) d[16 * c + x] = chunk[x];
          }
          tmem_wait_ld();
          if (lane < G::TAIL) {
            const int r = G::MMA_ROWS + lane;
            const int rb = r / ELL, rbit = r - rb * ELL;
#pragma unroll
            for (int i = 0; i < K; ++i)
              out_st[r * K + i] = (p.dbg & 8u)
                                      ? finish_value<ELL, 4, PM>(&d[i * 4], (i == rb) ? (1u << rbit) : 0u, p)
                                      : finish_neg<ELL, PM>(&d[i * 4], (i == rb) ? (1u << rbit) : 0u, p);
          }
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&epi_done[b]);
      named_bar(1, NE_THREADS);
      if (et == 0) {
        const OpRec op = ops[item / lanes];
        const uint32_t ln = item - (item / lanes) * lanes;
        bulk_s2g(store + ((uint64_t)op.out * lanes + ln) * G::CT_WORDS, out_st, G::CT_BYTES);
      }
    }
    if (et == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem_base);
}

}  // namespace tc
}  // namespace fhegpu
