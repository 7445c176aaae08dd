// tcgen05.mma kind::i8 throughput microbenchmark: cycles per MMA for several shapes and
// operand sources (A in TMEM vs smem, B MN-major vs K-major), one CTA per SM.
#include <cstdio>
#include <cstdint>
#include "../../paper_1611_08769_b200/csrc/tc_nand.cuh"
using namespace fhegpu::tc;

template <int N, bool A_TMEM, bool B_MN, int NACC = 1, int M = 128>
__global__ void __launch_bounds__(128, 1) bench(uint64_t *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *sb = sm;                 // B: 32 x N bytes
  uint8_t *sa = sm + 32 * 1024;     // A smem: 128 x 32 bytes
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 48 * 1024);
  uint32_t *slot = reinterpret_cast<uint32_t *>(sm + 48 * 1024 + 64);
  int tid = threadIdx.x;
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u * (i & 3);
  if (tid < 32) tmem_alloc<512>(slot);
  if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    uint64_t bd;
    if (B_MN) bd = smem_desc(smem_u32(sb), (N / 16) * 128, 128);   // LBO: K-group stride, SBO: N-chunk
    else bd = smem_desc(smem_u32(sb), 128, 256);                   // K-major: LBO K-chunk, SBO 8-row group
    uint64_t ad = smem_desc(smem_u32(sa), 128, (M == 64 && NACC < 0) ? 0 : 256);
    uint64_t t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t dcol = (uint32_t)(i % NACC) * 64u;
      if (A_TMEM) mma_i8_ts(tmem + dcol, tmem + 256 + 8 * (i % NACC), bd, idesc, i >= NACC);
      else mma_i8_ss(tmem + dcol, ad, bd, idesc, i >= NACC);
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
    uint64_t t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid < 32) tmem_dealloc<512>(tmem);
}

template <int N, bool A_TMEM, bool B_MN, int NACC = 1, int M = 128>
void run(const char *name, int sms) {
  uint64_t *d; cudaMalloc(&d, sms * 8);
  auto k = bench<N, A_TMEM, B_MN, NACC, M>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  const int iters = 2000;
  k<<<sms, 128, 50 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  uint64_t h[148]; cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  double cyc = avg / iters;
  printf("%-34s sms=%3d  cycles/MMA=%7.2f  MAC/clk/SM=%7.0f  %s\n", name, sms, cyc, (double)M * N * 32 / cyc,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

// Dense i8 tensor peak as a rate: every SM issues back-to-back M128 N256 K32 MMAs (A and B in
// shared memory, the shape that reaches the full datapath), timed with CUDA events.
void peak(int sms) {
  uint64_t *d; cudaMalloc(&d, sms * 8);
  auto k = bench<256, false, false, 1, 128>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  const int iters = 200000;
  k<<<sms, 128, 50 * 1024>>>(d, 1000);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 128, 50 * 1024>>>(d, iters);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  uint64_t h[148]; cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  const double macs = (double)sms * iters * 128.0 * 256 * 32;
  printf("{\"i8_dense_tops\": %.1f, \"mac_per_clk_per_sm\": %.0f, \"ms\": %.3f, \"sms\": %d, "
         "\"shape\": \"M128 N256 K32 kind::i8, A and B smem\", \"err\": \"%s\"}\n",
         2.0 * macs / (ms * 1e-3) / 1e12, 128.0 * 256 * 32 / (avg / iters), ms, sms,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char **argv) {
  if (argc > 1 && argv[1][0] == 'p') { peak(148); return 0; }
  for (int sms : {148}) {
    run<48, false, true, 1, 64>("M64 N48 smemA", sms);
    run<48, true, true, 1, 64>("M64 N48 tmemA", sms);
    run<16, false, true, 1, 64>("M64 N16 smemA", sms);
    run<96, false, true, 1, 64>("M64 N96 smemA", sms);
    run<48, false, true, 1, 128>("M128 N48 smemA (ref)", sms);
    run<48, true, true, 2>("N48 tmemA, 2 interleaved accumulators", sms);
    run<48, true, true, 3>("N48 tmemA, 3 interleaved accumulators", sms);
    run<48, true, true, 4>("N48 tmemA, 4 interleaved accumulators", sms);
    run<48, false, true, 2>("N48 smemA, 2 interleaved accumulators", sms);
    run<48, false, true, 4>("N48 smemA, 4 interleaved accumulators", sms);
    run<16, true, true, 4>("N16 tmemA, 4 interleaved accumulators", sms);
    run<48, true, true>("M128 N48  A=tmem B=MN (current)", sms);
    run<48, true, false>("M128 N48  A=tmem B=K", sms);
    run<48, false, true>("M128 N48  A=smem B=MN", sms);
    run<48, false, false>("M128 N48  A=smem B=K", sms);
    run<16, true, true>("M128 N16  A=tmem B=MN", sms);
    run<32, true, true>("M128 N32  A=tmem B=MN", sms);
    run<64, true, true>("M128 N64  A=tmem B=MN", sms);
    run<96, true, true>("M128 N96  A=tmem B=MN", sms);
    run<128, true, true>("M128 N128 A=tmem B=MN", sms);
    run<256, true, true>("M128 N256 A=tmem B=MN", sms);
    run<256, true, false>("M128 N256 A=tmem B=K", sms);
    run<256, false, false>("M128 N256 A=smem B=K", sms);
  }
  return 0;
}
