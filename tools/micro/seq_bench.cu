// Per-gate tcgen05 MMA sequence timing: the production sequence and variants.
#include <cstdio>
#include <cstdint>
#include "../../paper_1611_08769_b200/csrc/tc_nand.cuh"
using namespace fhegpu::tc;

// MODE 0: production (2 tiles x 9 TS + 9 SS tail, SBO=0)     MODE 1: no tail
// MODE 2: tail with SBO=256 (real 128-row block)              MODE 3: all 27 as TS
// MODE 4: tiles interleaved per K-step                        MODE 5: 27 SS (A smem, 128 rows)
template <int MODE>
__global__ void __launch_bounds__(128, 1) seq(uint64_t *out, int gates) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *sb = sm;                    // B 13.8 KB (MN-major, 36 K-groups x 3 chunks)
  uint8_t *sa = sm + 16 * 1024;        // A smem 128 x 288 B = 36 KB
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 56 * 1024);
  uint32_t *slot = reinterpret_cast<uint32_t *>(sm + 56 * 1024 + 64);
  int tid = threadIdx.x;
  for (int i = tid; i < 56 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u * (i & 3);
  if (tid < 32) tmem_alloc<512>(slot);
  if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t LBO = 384, SBO = 128;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 16) | (6u << 17) | (8u << 24);
    const uint32_t bb = smem_u32(sb), ab = smem_u32(sa);
    uint64_t t0 = clock64();
    for (int g = 0; g < gates; ++g) {
      const uint32_t tb = tmem + (g & 1) * 256;
      if (MODE == 4) {
        for (int s = 0; s < 9; ++s)
          for (int mt = 0; mt < 2; ++mt)
            mma_i8_ts(tb + mt * 48, tb + 96 + mt * 72 + 8 * s, smem_desc(bb + s * 4 * LBO, LBO, SBO), idesc, s > 0);
      } else if (MODE == 5) {
        for (int mt = 0; mt < 3; ++mt)
          for (int s = 0; s < 9; ++s)
            mma_i8_ss(tb + mt * 48, smem_desc(ab + s * 256, 128, 2304), smem_desc(bb + s * 4 * LBO, LBO, SBO), idesc, s > 0);
      } else {
        for (int mt = 0; mt < 2; ++mt)
          for (int s = 0; s < 9; ++s)
            mma_i8_ts(tb + mt * 48, tb + 96 + mt * 72 + 8 * s, smem_desc(bb + s * 4 * LBO, LBO, SBO), idesc, s > 0);
        if (MODE == 0 || MODE == 2)
          for (int s = 0; s < 9; ++s)
            mma_i8_ss(tb + 96, smem_desc(ab + s * 256, 128, MODE == 0 ? 0 : 2304), smem_desc(bb + s * 4 * LBO, LBO, SBO), idesc, s > 0);
        if (MODE == 3)
          for (int s = 0; s < 9; ++s)
            mma_i8_ts(tb + 144 + 48 * 0 + 64, tb + 96 + 8 * s, smem_desc(bb + s * 4 * LBO, LBO, SBO), idesc, s > 0);
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid < 32) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char *name, int per_gate) {
  uint64_t *d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(seq<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  const int gates = 200;
  seq<MODE><<<148, 128, 60 * 1024>>>(d, gates);
  cudaError_t e = cudaDeviceSynchronize();
  uint64_t h[148]; cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-44s cycles/gate=%7.1f  cycles/MMA=%6.1f %s\n", name, avg / gates, avg / gates / per_gate,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  run<0>("production: 18 TS + 9 SS tail (SBO=0)", 27);
  run<1>("tiles only: 18 TS", 18);
  run<2>("18 TS + 9 SS tail (SBO=2304, 128 rows)", 27);
  run<3>("27 TS (tail from TMEM)", 27);
  run<4>("18 TS, tiles interleaved per K-step", 18);
  run<5>("27 SS (A from smem)", 27);
  return 0;
}
