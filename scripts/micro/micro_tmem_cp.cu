// Check: tcgen05.cp.cta_group::1.32x128b.warpx4 of one 512-byte smem row (32 x 16 B) into
// TMEM column c, replicated to the 4 lane quarters; read back with tcgen05.ld.32x32b.x4 by
// 4 warps.  Tries both descriptor encodings (SBO vs LBO = 128 B between 8-row core matrices).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // sm100 descriptor version
  return d;                 // base offset 0, lbo mode 0, layout 0 = SWIZZLE_NONE
}
__global__ void k(int* out, int variant) {
  __shared__ __align__(128) float row[4][128];
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&row[0][0])[i] = (float)i;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    for (int r = 0; r < 4; ++r) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&row[r][0]);
      const uint64_t d = variant == 0 ? desc(sa, 0, 128) : desc(sa, 128, 0);
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tb + 4 * r + 8), "l"(d));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  int bad = 0;
  for (int r = 0; r < 4; ++r) {
    uint32_t a, b, c, d;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(tb + ((uint32_t)(warp * 32) << 16) + 4 * r + 8));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const float e = (float)(r * 128 + lane * 4);
    bad += (__uint_as_float(a) != e) + (__uint_as_float(b) != e + 1) + (__uint_as_float(c) != e + 2) + (__uint_as_float(d) != e + 3);
    if (lane == 5 && r == 1 && warp == 2) out[8] = (int)__uint_as_float(a);
  }
  atomicAdd(out + variant, bad);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
int main() {
  int* o; cudaMalloc(&o, 64); cudaMemset(o, 0, 64);
  k<<<1, 128>>>(o, 0); k<<<1, 128>>>(o, 1);
  int h[16]; cudaMemcpy(h, o, 64, cudaMemcpyDeviceToHost);
  printf("mismatches sbo=128: %d, lbo=128: %d (of 2048); sample %d (expect %d); %s\n", h[0], h[1], h[8], 128 + 20,
         cudaGetErrorString(cudaGetLastError()));
}
