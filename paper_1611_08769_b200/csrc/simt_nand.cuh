// simt_nand.cuh -- CUDA-core level kernel (reference implementation on the GPU).
//
// One CTA evaluates one (gate, lane) item at a time, grid-striding over the
// level's items.  Compact NAND:
//     out[r][i] = (G[r][i] - sum_c bit_c(row r of V1) * V2[c][i]) mod q
// where bit c of row r is bit (c mod ell) of V1[r][c / ell].  Operands are
// complemented on load ((G - V) mod q) when the op's flags say so -- the fused
// hom_not of fhe.py:343-350.  This kernel serves parameter sets without a
// tensor-core build and is the GPU cross-check of the tcgen05 kernel.
#pragma once

#include "common.cuh"

namespace fhegpu {

template <int KMAX>
__global__ void __launch_bounds__(256)
level_simt_kernel(uint32_t *__restrict__ store, const OpRec *__restrict__ ops, uint32_t n_ops,
                  uint32_t lanes, DevParams p) {
  extern __shared__ uint32_t smem[];
  uint32_t *sA = smem;              // V1 (effective), rows x k
  uint32_t *sB = smem + p.words;    // V2 (effective)
  const uint64_t n_items = (uint64_t)n_ops * lanes;
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint32_t op_i = (uint32_t)(item / lanes);
    const uint32_t lane = (uint32_t)(item - (uint64_t)op_i * lanes);
    const OpRec op = ops[op_i];
    const uint32_t *g1 = store + ((uint64_t)op.left * lanes + lane) * p.ct_words;
    const uint32_t *g2 = store + ((uint64_t)op.right * lanes + lane) * p.ct_words;
    uint32_t *go = store + ((uint64_t)op.out * lanes + lane) * p.ct_words;
    const bool c1 = op.flags & 1u, c2 = op.flags & 2u;
    for (uint32_t w = threadIdx.x; w < p.words; w += blockDim.x) {
      const uint32_t r = w / p.k, i = w - r * p.k;
      const uint32_t g = gadget(p, r, i);
      uint32_t a = g1[w], b = g2[w];
      sA[w] = c1 ? sub_mod(g, a, p.q) : a;
      sB[w] = c2 ? sub_mod(g, b, p.q) : b;
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < p.rows; r += blockDim.x) {
      uint64_t acc[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) acc[i] = 0;
      for (uint32_t blk = 0; blk < p.k; ++blk) {
        uint32_t bits = sA[r * p.k + blk];
        while (bits) {
          const uint32_t j = __ffs(bits) - 1;
          bits &= bits - 1;
          const uint32_t *vrow = sB + (blk * p.ell + j) * p.k;
#pragma unroll
          for (int i = 0; i < KMAX; ++i)
            if (i < (int)p.k) acc[i] += vrow[i];
        }
      }
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        if (i < (int)p.k) {
          const uint32_t s = mod_u64(acc[i], p.q, p.mu);
          go[r * p.k + i] = sub_mod(gadget(p, r, i), s, p.q);
        }
      }
    }
    __syncthreads();
  }
}

// out = (G - in) mod q elementwise over `count` ciphertexts (dense N*k each in
// and out of a staging buffer).
__global__ void complement_kernel(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                                  uint64_t count, DevParams p) {
  const uint64_t total = count * p.words;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w = (uint32_t)(t % p.words);
    const uint32_t r = w / p.k, i = w - r * p.k;
    out[t] = sub_mod(gadget(p, r, i), in[t], p.q);
  }
}

// hom_add in compact form (fhe.py:352-356): out = (a + b) mod q, dense rows of p.words.
__global__ void add_kernel(const uint32_t *__restrict__ a, const uint32_t *__restrict__ b,
                           uint32_t *__restrict__ out, uint64_t count, DevParams p) {
  const uint64_t total = count * p.words;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = a[t] + b[t];               // both < q < 2^31
    out[t] = x >= p.q ? x - p.q : x;
  }
}

// In-place complement of padded store rows: v <- (G - v) mod q.
__global__ void complement_rows_kernel(uint32_t *__restrict__ rows, uint64_t count, DevParams p) {
  const uint64_t total = count * p.words;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = t / p.words;
    const uint32_t w = (uint32_t)(t - c * p.words);
    const uint32_t r = w / p.k, i = w - r * p.k;
    uint32_t *v = rows + c * p.ct_words + w;
    *v = sub_mod(gadget(p, r, i), *v, p.q);
  }
}

// store[idx[c]] <- dense[c] (zero the padding words).
__global__ void scatter_kernel(uint32_t *__restrict__ store, const uint64_t *__restrict__ idx,
                               const uint32_t *__restrict__ dense, uint64_t count, DevParams p) {
  const uint64_t total = count * p.ct_words;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = t / p.ct_words;
    const uint32_t w = (uint32_t)(t - c * p.ct_words);
    store[idx[c] * p.ct_words + w] = (w < p.words) ? dense[c * p.words + w] : 0u;
  }
}

// Slot blocks -> slot blocks (fhegpu_store_copy_slots): slot s holds ciphertexts
// [s * lanes, (s + 1) * lanes), one contiguous run of lanes * ct_words u32, copied as uint4
// (ct_words is a multiple of 4).  blockIdx.y strides the pairs, blockIdx.x the run.
__global__ void copy_slots_kernel(uint32_t *__restrict__ store, const uint32_t *__restrict__ src,
                                  const uint32_t *__restrict__ dst, uint32_t n, uint64_t run_u4) {
  uint4 *st = reinterpret_cast<uint4 *>(store);
  for (uint32_t i = blockIdx.y; i < n; i += gridDim.y) {
    const uint4 *from = st + (uint64_t)src[i] * run_u4;
    uint4 *to = st + (uint64_t)dst[i] * run_u4;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < run_u4;
         t += (uint64_t)gridDim.x * blockDim.x)
      to[t] = from[t];
  }
}

// Host-streaming repack (fhegpu_prog_run_host): rows of `words` u32 (dense, as the host
// holds them) <-> store rows of ct_words (padding zeroed).  One row per block iteration.
__global__ void dense_to_store_kernel(uint32_t *__restrict__ store, const uint32_t *__restrict__ dense,
                                      uint64_t rows, DevParams p) {
  for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x)
    for (uint32_t w = threadIdx.x; w < p.ct_words; w += blockDim.x)
      store[r * p.ct_words + w] = w < p.words ? dense[r * p.words + w] : 0u;
}

__global__ void store_to_dense_kernel(uint32_t *__restrict__ dense, const uint32_t *__restrict__ store,
                                      uint64_t rows, DevParams p) {
  for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x)
    for (uint32_t w = threadIdx.x; w < p.words; w += blockDim.x)
      dense[r * p.words + w] = store[r * p.ct_words + w];
}

// Packed matrix bits: the reference's serialised ciphertext (fileio.py:72-79 / EFT1
// payload): C = decompose(V) row-major, bit j of V[r][i] at stream position
// r*N + i*ell + j, packed 8 per byte MSB first; ceil(N*N/8) bytes per ciphertext.
// Since N = k*ell the stream is simply every value v = r*k + i, ell bits each, LSB first.
//
// Word view: stream bits [32w, 32w + 32) as a u32 X (bit t = stream bit 32w + t) is the
// little-endian load of bytes 4w..4w+3 with the bits of each byte reversed:
//   X = prmt(brev(W), 0x0123)  and  W = prmt(brev(X), 0x0123).
__device__ __forceinline__ uint32_t stream_word(uint32_t w) { return __byte_perm(__brev(w), 0u, 0x0123); }

__global__ void packed_to_store_kernel(uint32_t *__restrict__ store, const uint8_t *__restrict__ packed,
                                       uint64_t rows, uint32_t row_bytes, DevParams p) {
  extern __shared__ uint32_t s_x[];
  const uint32_t mask = (1u << p.ell) - 1u;
  const bool wide = (row_bytes & 3u) == 0;
  const uint32_t n_x = (row_bytes + 3) / 4;
  for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint8_t *src = packed + r * row_bytes;
    if (wide) {                                    // u32 loads (rows 4-byte aligned)
      const uint32_t *src4 = reinterpret_cast<const uint32_t *>(src);
      for (uint32_t x = threadIdx.x; x < n_x; x += blockDim.x) s_x[x] = stream_word(src4[x]);
    } else {
      for (uint32_t x = threadIdx.x; x < n_x; x += blockDim.x) {
        uint32_t w = 0;
        for (uint32_t t = 0; t < 4; ++t)
          if (4 * x + t < row_bytes) w |= (uint32_t)src[4 * x + t] << (8 * t);
        s_x[x] = stream_word(w);
      }
    }
    __syncthreads();
    for (uint32_t v = threadIdx.x; v < p.ct_words; v += blockDim.x) {
      uint32_t val = 0;
      if (v < p.words) {
        const uint32_t bit = v * p.ell, x = bit >> 5;
        const uint32_t hi = x + 1 < n_x ? s_x[x + 1] : 0u;
        val = __funnelshift_r(s_x[x], hi, bit & 31u) & mask;
      }
      store[r * p.ct_words + v] = val;
    }
    __syncthreads();
  }
}

__global__ void store_to_packed_kernel(uint8_t *__restrict__ packed, const uint32_t *__restrict__ store,
                                       uint64_t rows, uint32_t row_bytes, DevParams p) {
  extern __shared__ uint32_t s_vals[];
  const bool wide = (row_bytes & 3u) == 0;
  const uint32_t n_x = (row_bytes + 3) / 4;
  for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    for (uint32_t w = threadIdx.x; w < p.words; w += blockDim.x) s_vals[w] = store[r * p.ct_words + w];
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < n_x; x += blockDim.x) {
      // stream bits [32x, 32x + 32): value v from bit j on, then v+1, v+2 (ell >= 11)
      const uint32_t bit = 32 * x, v = bit / p.ell, j = bit - v * p.ell;
      uint32_t X = v < p.words ? s_vals[v] >> j : 0u;
      uint32_t got = p.ell - j;
      for (uint32_t t = 1; got < 32 && v + t < p.words; ++t, got += p.ell) X |= s_vals[v + t] << got;
      const uint32_t W = stream_word(X);
      if (wide) {
        reinterpret_cast<uint32_t *>(packed + r * row_bytes)[x] = W;
      } else {
        for (uint32_t t = 0; t < 4; ++t)
          if (4 * x + t < row_bytes) packed[r * row_bytes + 4 * x + t] = (uint8_t)(W >> (8 * t));
      }
    }
    __syncthreads();
  }
}

// dense[c] <- store[idx[c]] (complemented when comp[c]); row >= 0 selects one row only.
// Decryption phase of row `row` (fhe.py:267-286): x = sum_{i,b} bit_b(V[row][i]) * pw[i][b] mod q,
// pw[i][b] = (sk_i << b) mod q, centred to (-q/2, q/2].  One thread per ciphertext; the host
// turns x into the bit and checks the noise threshold.
__global__ void decrypt_rows_kernel(const uint32_t *__restrict__ store, const uint64_t *__restrict__ idx,
                                    const uint8_t *__restrict__ comp, const uint32_t *__restrict__ pw,
                                    int32_t *__restrict__ out, uint64_t count, uint32_t row, DevParams p) {
  __shared__ uint32_t s_pw[16 * 32];
  for (uint32_t t = threadIdx.x; t < p.k * p.ell; t += blockDim.x) s_pw[t] = pw[t];
  __syncthreads();
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < count;
       c += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t acc = 0;
    const uint32_t *v_row = store + idx[c] * p.ct_words + (uint64_t)row * p.k;
    for (uint32_t i = 0; i < p.k; ++i) {
      uint32_t v = v_row[i];
      if (comp != nullptr && comp[c]) v = sub_mod(gadget(p, row, i), v, p.q);
      for (uint32_t b = 0; b < p.ell; ++b)
        if ((v >> b) & 1u) acc += s_pw[i * p.ell + b];
    }
    const uint32_t x = (uint32_t)(acc % p.q);
    out[c] = x > p.q / 2 ? (int32_t)((int64_t)x - p.q) : (int32_t)x;
  }
}

__global__ void gather_kernel(const uint32_t *__restrict__ store, const uint64_t *__restrict__ idx,
                              const uint8_t *__restrict__ comp, uint32_t *__restrict__ dense,
                              uint64_t count, int row, DevParams p) {
  const uint32_t per = row < 0 ? p.words : p.k;
  const uint64_t total = count * per;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = t / per;
    const uint32_t j = (uint32_t)(t - c * per);
    const uint32_t w = row < 0 ? j : (uint32_t)row * p.k + j;
    uint32_t v = store[idx[c] * p.ct_words + w];
    if (comp != nullptr && comp[c]) {
      const uint32_t r = w / p.k, i = w - r * p.k;
      v = sub_mod(gadget(p, r, i), v, p.q);
    }
    dense[t] = v;
  }
}

}  // namespace fhegpu
