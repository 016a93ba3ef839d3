// Microbenchmark: aggregate tcgen05.ld (TMEM -> registers) bandwidth per SM, to decide
// whether TMEM-staged X can beat the 128 B/clk/SM shared-memory ceiling.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_tmem micro_tmem.cu
#include <cstdio>
#include <cstdint>

template <int X>
__device__ __forceinline__ void ldtm(uint32_t taddr, uint32_t (&r)[X]);

template <>
__device__ __forceinline__ void ldtm<4>(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void ldtm<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}

template <int X, int BATCH>
__global__ void __launch_bounds__(1024) ldtm_bw(float* out, int iters) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase + (((uint32_t)(warp & 3) * 32) << 16);
  float acc = 0.f;
  int col = (warp >> 2) * 8;
  for (int i = 0; i < iters; ++i) {
    uint32_t r[BATCH][X];
#pragma unroll
    for (int b = 0; b < BATCH; ++b) ldtm<X>(t + ((col + b * X) & (511 & ~(X - 1))), r[b]);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int b = 0; b < BATCH; ++b)
#pragma unroll
      for (int j = 0; j < X; ++j) acc += __uint_as_float(r[b][j]);
    col += BATCH * X;
  }
  if (acc == 1.2345f) out[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{");
  auto run = [&](const char* name, auto kern, int threads, int x, int batch) {
    const int iters = 20000;
    kern<<<sms, threads>>>(out, 10);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<sms, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)sms * threads * iters * batch * x * 4;
    printf("\"%s\": {\"TBps\": %.2f, \"B_per_clk_per_sm\": %.1f, \"err\": \"%s\"}, ", name, bytes / ms / 1e9,
           bytes / (ms * 1e-3) / (clk * 1e3) / sms, cudaGetErrorString(cudaGetLastError()));
  };
  run("x4_b4_w4", ldtm_bw<4, 4>, 128, 4, 4);
  run("x4_b4_w8", ldtm_bw<4, 4>, 256, 4, 4);
  run("x4_b4_w16", ldtm_bw<4, 4>, 512, 4, 4);
  run("x4_b4_w32", ldtm_bw<4, 4>, 1024, 4, 4);
  run("x4_b8_w16", ldtm_bw<4, 8>, 512, 4, 8);
  run("x4_b8_w32", ldtm_bw<4, 8>, 1024, 4, 8);
  run("x16_b2_w8", ldtm_bw<16, 2>, 256, 16, 2);
  run("x16_b2_w16", ldtm_bw<16, 2>, 512, 16, 2);
  printf("\"sms\": %d}\n", sms);
  return 0;
}
