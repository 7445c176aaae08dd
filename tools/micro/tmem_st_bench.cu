// tmem_st_bench.cu -- throughput of the operand-builder's data movement on one SM:
// tcgen05.st (register -> TMEM) vs st.shared, the way the A/B builders use them.
//
// One CTA of W warps (lanes quadrant = warp % 4); each warp repeats ITERS times a
// per-gate pattern and the CTA reports cycles per iteration.  Modes:
//   0: A build as in the kernel: 9 words -> 72 u32 (spread) -> 2x st.32x32b.x32 + 1x .x8, wait::st
//   1: the same stores with constant data (no spread ALU work)
//   2: spread ALU only (results folded into a checksum, no stores)
//   3: 72 u32 per thread to shared memory (18 st.shared.v4), same bytes as mode 1
//   4: st.32x32b.x64 + x8 (fewer, wider instructions)
//   5: st.16x256b.x8 shapes (same bytes)
// usage: tmem_st_bench [warps=8] [iters=2000]
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t *v) {
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
__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t *v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void st16x256_x8(uint32_t taddr, const uint32_t *v) {
  // 16 lanes x 256 bits, repeated 8x along columns: 32 registers per thread
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void spread(uint32_t w, uint32_t *out) {
#pragma unroll
  for (int o = 0; o < 8; ++o) out[o] = (w >> o) & 0x01010101u;
}

__global__ void bench(int mode, int iters, uint32_t *res, uint32_t *sink, const uint32_t *src) {
  __shared__ uint32_t tslot;
  extern __shared__ __align__(16) uint32_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tslot;
  const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
  // two A tiles per 8 warps: warps 4..7 write the second tile's columns
  const uint32_t col0 = 256 + ((warp >> 2) & 1) * 72;
  const uint32_t a_addr = tbase + lane_off + col0;
  uint32_t words[9];
  for (int i = 0; i < 9; ++i) words[i] = src[(threadIdx.x * 9 + i) & 4095];
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0 || mode == 1 || mode == 2) {
#pragma unroll
      for (int w0 = 0; w0 < 8; w0 += 4) {
        uint32_t sp[32];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (mode == 1) {
#pragma unroll
            for (int x = 0; x < 8; ++x) sp[8 * j + x] = words[w0 + j] + x;
          } else {
            spread(words[w0 + j] + it, sp + 8 * j);
          }
        }
        if (mode == 2) {
#pragma unroll
          for (int x = 0; x < 32; ++x) acc ^= sp[x];
        } else {
          st32(a_addr + 8 * w0, sp);
        }
      }
      uint32_t sp8[8];
      if (mode == 1) {
#pragma unroll
        for (int x = 0; x < 8; ++x) sp8[x] = words[8] + x;
      } else {
        spread(words[8] + it, sp8);
      }
      if (mode == 2) {
#pragma unroll
        for (int x = 0; x < 8; ++x) acc ^= sp8[x];
      } else {
        st8(a_addr + 64, sp8);
        wait_st();
      }
    } else if (mode == 3) {
      uint4 *dst = reinterpret_cast<uint4 *>(sm) + threadIdx.x;
#pragma unroll
      for (int x = 0; x < 18; ++x) {
        const uint32_t b = words[x % 9] + x + it;
        dst[x * blockDim.x] = make_uint4(b, b + 1, b + 2, b + 3);
      }
      __syncwarp();
    } else if (mode == 4) {
      uint32_t sp[32];
#pragma unroll
      for (int x = 0; x < 32; ++x) sp[x] = words[x % 9] + x + it;
      st32(a_addr, sp);
      st32(a_addr + 32, sp);
      st8(a_addr + 64, sp);
      wait_st();
    } else if (mode == 5) {
      uint32_t sp[32];
#pragma unroll
      for (int x = 0; x < 32; ++x) sp[x] = words[x % 9] + x + it;
      // 16x256b.x8: 16 lanes x 64 columns (8 x 8 cols) per instruction; a warp's 32 lanes
      // need 2 (lanes 0-15, 16-31)
      st16x256_x8(a_addr, sp);
      st16x256_x8(a_addr + (16u << 16), sp);
      uint32_t sp8[8];
      for (int x = 0; x < 8; ++x) sp8[x] = sp[x];
      st8(a_addr + 64, sp8);
      wait_st();
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) res[0] = (uint32_t)(t1 - t0);
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main(int argc, char **argv) {
  int warps = argc > 1 ? atoi(argv[1]) : 8;
  int iters = argc > 2 ? atoi(argv[2]) : 2000;
  uint32_t *res, *sink, *src;
  cudaMalloc(&res, 4);
  cudaMalloc(&sink, 4096 * 4);
  cudaMalloc(&src, 4096 * 4);
  cudaMemset(src, 0x5a, 4096 * 4);
  int smem = 18 * 16 * 32 * warps;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char *names[] = {"spread+tmem st (kernel A build)", "tmem st only (x32,x32,x8)", "spread ALU only",
                         "st.shared.v4 same bytes", "tmem st x32,x32,x8 no spread", "tmem st 16x256b.x8"};
  for (int mode = 0; mode < 6; ++mode) {
    bench<<<1, 32 * warps, smem>>>(mode, 10, res, sink, src);
    bench<<<1, 32 * warps, smem>>>(mode, iters, res, sink, src);
    uint32_t cyc = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&cyc, res, 4, cudaMemcpyDeviceToHost);
    double per = (double)cyc / iters;
    double bytes = (mode == 2) ? 0 : 32.0 * warps * 288;
    printf("mode %d %-34s warps=%2d cycles/iter=%8.1f  B/clk=%6.1f %s\n", mode, names[mode], warps, per,
           bytes / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
