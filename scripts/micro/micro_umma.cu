// Back-to-back tcgen05.mma throughput, cta_group::1, operands resident in shared memory (no TMA):
// the tensor-pipe ceiling of the tcgen05 block executor (kernel 5d) for kind::f16 M128 N256 K16
// and kind::tf32 M128 N256 K8 (one K-major SW128 A, one MN-major B), 1 CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_umma micro_umma.cu && ./micro_umma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | ((uint64_t)lay << 61);
}
template <int KIND>  // 0 = f16, 1 = tf32
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t d = tslot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(sm), sb = sa + 16384;
    const uint32_t fmt = KIND == 1 ? 2u : 0u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 16) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t da = desc(sa + 32u * kk, 16u, 1024u, 2u);
        const uint64_t db = KIND == 1 ? desc(sb + 1024u * kk, 4096u, 512u, 1u) : desc(sb + 2048u * kk, 8192u, 1024u, 2u);
        const uint32_t dd = d + (uint32_t)((it & 1) * 256);
        if (KIND == 1)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(dd), "l"(da), "l"(db), "r"(idesc), "r"(1u));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(dd), "l"(da), "l"(db), "r"(idesc), "r"(1u));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
}

template <int KIND>
void run(const char* name, double flop_per_mma) {
  const int iters = 20000, nblk = 148;
  unsigned long long* cyc;
  cudaMalloc(&cyc, nblk * 8);
  cudaFuncSetAttribute(k<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  k<KIND><<<nblk, 128, 50 * 1024>>>(100, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<KIND><<<nblk, 128, 50 * 1024>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, cyc, nblk * 8, cudaMemcpyDeviceToHost);
  const double flops = (double)nblk * iters * 4 * flop_per_mma;
  printf("%-28s %s  %.1f us  %.1f TFLOP/s  (%.1f cycles per MMA on SM 0)\n", name, cudaGetErrorString(e), ms * 1e3,
         flops / (ms * 1e-3) / 1e12, (double)h[0] / (iters * 4.0));
  cudaFree(cyc);
}

int main() {
  run<0>("f16 M128 N256 K16 cta1", 2.0 * 128 * 256 * 16);
  run<1>("tf32 M128 N256 K8 cta1", 2.0 * 128 * 256 * 8);
  return 0;
}
