// common.cuh -- shared device helpers for the fhegpu kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fhegpu {

// Parameter block passed by value to every kernel.
struct DevParams {
  uint32_t k;         // Z_q columns per compact row (n + 1)
  uint32_t ell;       // bits per value
  uint32_t q;         // modulus (odd, < 2^31)
  uint32_t rows;      // N = k * ell
  uint32_t ct_words;  // padded u32 stride of one ciphertext
  uint32_t words;     // N * k (dense words)
  uint64_t mu;        // floor(2^64 / q) for Barrett reduction
  uint32_t dbg;       // debug knobs (bit 0: swap B descriptor strides); 0 in production
  uint32_t pm_c;      // 2^ell - q (pseudo-Mersenne epilogue constant)
  uint32_t lanes_magic;  // floor((2^32 - 1) / lanes): item / lanes by multiply (set per launch)
};

// Gadget entry G[r][i] = 2^(r mod ell) if i == r / ell else 0 (fhe.py:200-208, mu = 1).
__device__ __forceinline__ uint32_t gadget(const DevParams &p, uint32_t r, uint32_t i) {
  uint32_t blk = r / p.ell;
  return (blk == i) ? (1u << (r - blk * p.ell)) : 0u;
}

// Same with ell known at compile time (no runtime division).
template <int ELL>
__device__ __forceinline__ uint32_t gadget_ct(uint32_t r, uint32_t i) {
  const uint32_t blk = r / ELL;
  return (blk == i) ? (1u << (r - blk * ELL)) : 0u;
}

// (g - v) mod q for g, v in [0, q).
__device__ __forceinline__ uint32_t sub_mod(uint32_t g, uint32_t v, uint32_t q) {
  return (g >= v) ? (g - v) : (g + (q - v));
}

// x mod q for any 64-bit x (Barrett with mu = floor(2^64 / q); one correction).
__device__ __forceinline__ uint32_t mod_u64(uint64_t x, uint32_t q, uint64_t mu) {
  uint64_t qt = __umul64hi(x, mu);
  uint64_t r = x - qt * (uint64_t)q;
  return (uint32_t)(r >= q ? r - q : r);
}

// item / lanes and item % lanes for 32-bit items (magic = floor((2^32-1)/lanes)).
__device__ __forceinline__ void div_lanes(uint32_t item, uint32_t lanes, uint32_t magic, uint32_t &q,
                                          uint32_t &r) {
  q = __umulhi(item, magic);
  r = item - q * lanes;
  if (r >= lanes) {
    ++q;
    r -= lanes;
  }
}

struct OpRec {
  uint32_t left, right, out, flags;
};

}  // namespace fhegpu
