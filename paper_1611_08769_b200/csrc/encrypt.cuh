// encrypt.cuh -- device-side fresh encryption, stream-exact with numpy's PCG64.
//
// Reference: GswScheme._encrypt (fhe.py:227-233):
//     R = rng.integers(0, 2, (N, m));  V = (R @ pk + mu * G) mod q
// numpy's Generator(PCG64) draws integers(0, 2) from 32-bit halves of the
// 64-bit PCG64 output (low half first) and keeps bit 31 of each half (Lemire
// bounded draw with range 2 never rejects).  PCG64 is an LCG on 128 bits
// (state = state * MULT + inc) with the XSL-RR output of the NEW state, so any
// draw can be reached by an O(log n) jump: step^n(s) = MULT^n s + inc * G_n,
// G_n = sum_{i<n} MULT^i.  Every (ciphertext, row) thread jumps to its first
// draw and generates its m bits; the result is bit-identical to the reference
// encrypting with the same Generator.
#pragma once

#include "common.cuh"

namespace fhegpu {

typedef unsigned __int128 u128;

struct JumpTable {
  u128 a[64];  // MULT^(2^j)
  u128 g[64];  // G_(2^j)
};

struct StreamRec {
  uint64_t s_lo, s_hi, inc_lo, inc_hi;
};

__device__ __forceinline__ uint64_t pcg_out(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const uint32_t rot = (uint32_t)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// One thread per (ciphertext, row).  pk is m x k (row-major, values < q).
__global__ void encrypt_kernel(uint32_t *__restrict__ store, const JumpTable *__restrict__ jt,
                               const StreamRec *__restrict__ streams,
                               const uint32_t *__restrict__ stream_idx,
                               const uint64_t *__restrict__ u32_off, const uint32_t *__restrict__ mu,
                               const uint64_t *__restrict__ target, const uint32_t *__restrict__ pk,
                               uint64_t count, uint32_t m, DevParams p) {
  extern __shared__ uint32_t s_pk[];
  for (uint32_t w = threadIdx.x; w < m * p.k; w += blockDim.x) s_pk[w] = pk[w];
  __syncthreads();
  const u128 mult = jt->a[0];
  const uint64_t total = count * p.rows;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = t / p.rows;
    const uint32_t r = (uint32_t)(t - e * p.rows);
    const StreamRec sr = streams[stream_idx[e]];
    const u128 inc = ((u128)sr.inc_hi << 64) | sr.inc_lo;
    u128 s = ((u128)sr.s_hi << 64) | sr.s_lo;
    const uint64_t first = u32_off[e] + (uint64_t)r * m;  // absolute 32-bit draw index
    uint64_t n = first >> 1;                               // 64-bit outputs to skip
    for (int j = 0; n; ++j, n >>= 1)
      if (n & 1) s = jt->a[j] * s + inc * jt->g[j];
    uint64_t acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0;
    uint64_t o = 0;
    uint64_t tdraw = first;
    if (tdraw & 1) {  // row starts on a high half
      s = s * mult + inc;
      o = pcg_out(s);
    }
    for (uint32_t c = 0; c < m; ++c, ++tdraw) {
      uint32_t bit;
      if ((tdraw & 1) == 0) {
        s = s * mult + inc;
        o = pcg_out(s);
        bit = (uint32_t)(o >> 31) & 1u;
      } else {
        bit = (uint32_t)(o >> 63);
      }
      if (bit) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i < (int)p.k) acc[i] += s_pk[c * p.k + i];
      }
    }
    const uint32_t blk = r / p.ell, jb = r - blk * p.ell;
    uint32_t *dst = store + target[e] * p.ct_words + r * p.k;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < (int)p.k) {
        uint64_t v = acc[i];
        if ((uint32_t)i == blk) v += (uint64_t)mu[e] << jb;   // mu * 2^j (mu < q, j < 31)
        dst[i] = mod_u64(v, p.q, p.mu);
      }
    }
    if (r == 0)
      for (uint32_t w = p.words; w < p.ct_words; ++w) store[target[e] * p.ct_words + w] = 0u;
  }
}

}  // namespace fhegpu
