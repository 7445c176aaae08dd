// Bitsliced cleartext evaluation (the GPU twin of fhefft's CleartextEngine, engine.py:69-121).
//
// A wire holds `lanes` independent plaintext bits packed 32 per u32 word (bit l of word w =
// lane 32 w + l), W = ceil(lanes / 32) words per wire, wire-major: store[slot * W + w].
// NAND(a, b) = ~(a & b) on whole words -- 32 lanes per instruction; a complemented
// operand (the free NOT of engine.py:185-187) is a XOR with all-ones on load.  One launch
// per netlist level; every (gate, word) item is independent, so a level is one coalesced
// pass: HBM-bound integer work, 12 bytes per item.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace fhegpu {

__global__ void bits_level_kernel(uint32_t *__restrict__ store, const OpRec *__restrict__ ops,
                                  uint32_t n_ops, uint32_t words, uint32_t tail_mask) {
  const uint64_t total = (uint64_t)n_ops * words;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t op_i = (uint32_t)(t / words);
    const uint32_t w = (uint32_t)(t - (uint64_t)op_i * words);
    const OpRec op = ops[op_i];
    const uint32_t a = store[(uint64_t)op.left * words + w] ^ (0u - (op.flags & 1u));
    const uint32_t b = store[(uint64_t)op.right * words + w] ^ (0u - ((op.flags >> 1) & 1u));
    uint32_t v = ~(a & b);
    if (w == words - 1) v &= tail_mask;           // lanes past batch_size stay 0
    store[(uint64_t)op.out * words + w] = v;
  }
}

// out[c] = store[slot[c]] (complemented when comp[c]), W words each.
__global__ void bits_gather_kernel(const uint32_t *__restrict__ store, const uint64_t *__restrict__ slots,
                                   const uint8_t *__restrict__ comp, uint32_t *__restrict__ out,
                                   uint64_t count, uint32_t words, uint32_t tail_mask) {
  const uint64_t total = count * words;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = t / words;
    const uint32_t w = (uint32_t)(t - c * words);
    uint32_t v = store[slots[c] * words + w];
    if (comp != nullptr && comp[c]) v = ~v & (w == words - 1 ? tail_mask : 0xFFFFFFFFu);
    out[t] = v;
  }
}

// store[slot[c]] = in[c], W words each.
__global__ void bits_scatter_kernel(uint32_t *__restrict__ store, const uint64_t *__restrict__ slots,
                                    const uint32_t *__restrict__ in, uint64_t count, uint32_t words) {
  const uint64_t total = count * words;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = t / words;
    const uint32_t w = (uint32_t)(t - c * words);
    store[slots[c] * words + w] = in[t];
  }
}

}  // namespace fhegpu
