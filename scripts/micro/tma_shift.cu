// Probe: a 2-D TMA box whose innermost start coordinate is NOT 16-byte aligned (shift by 1..3
// elements), with the 128-byte swizzles the tcgen05 executor uses.  Prints ok / mismatch / error.
//   fp32: box {32, 32}, SWIZZLE_128B_ATOM_32B;  fp16: box {64, 64}, SWIZZLE_128B
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap m, int x0, int y0, unsigned bytes, unsigned* out) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((unsigned long long)smraw + 1023) & ~1023ull);
  __shared__ __align__(8) unsigned long long bar;
  unsigned ba = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"((unsigned long long)&m), "r"(x0), "r"(y0), "r"(ba) : "memory");
    unsigned done = 0;
    while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(ba));
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = ((unsigned*)sm)[i];
}
int main() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  const int W = 4096, H = 128;
  for (int es : {4, 2}) {
    const int bx = 128 / es, by = bx;  // 128-byte rows
    std::vector<unsigned char> h((size_t)W * H * es);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (unsigned char)(i * 7 + (i >> 8) * 13);
    void* d; cudaMalloc(&d, h.size()); cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    unsigned* out; cudaMalloc(&out, 65536);
    CUtensorMap m; memset(&m, 0, sizeof m);
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    cuuint64_t str[1] = {(cuuint64_t)W * es};
    cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
    cuuint32_t est[2] = {1, 1};
    CUresult r = enc(&m, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, dims, str, box, est,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, es == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const unsigned bytes = bx * by * es;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int x0 : {64, 65, 66, 67, 63, -1}) {
      k<<<1, 128, bytes + 1024>>>(m, x0, 3, bytes, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("es %d x0 %d -> %s\n", es, x0, cudaGetErrorString(e)); return 0; }
      std::vector<unsigned char> g(bytes);
      cudaMemcpy(g.data(), out, bytes, cudaMemcpyDeviceToHost);
      // reference: row y (k), element x: 128-byte row r of the box = y; swizzle 128B: 16-byte chunk
      // c of row r at c ^ (r % 8); ATOM_32B: 32-byte chunks (c2) at c2 ^ (r % 4)... compare unswizzled
      int bad = 0;
      for (int y = 0; y < by; ++y)
        for (int x = 0; x < bx; ++x) {
          const int gx = x0 + x, gy = 3 + y;
          unsigned char ref[4] = {0, 0, 0, 0};
          if (gx >= 0 && gx < W) memcpy(ref, &h[((size_t)gy * W + gx) * es], es);
          const int b = x * es;
          size_t off;
          if (es == 4) off = (size_t)y * 128 + (((b / 32) ^ (y % 4)) * 32) + (b % 32);
          else off = (size_t)y * 128 + (((b / 16) ^ (y % 8)) * 16) + (b % 16);
          if (memcmp(ref, &g[off], es)) ++bad;
        }
      printf("es %d x0 %d -> %s, %d mismatches of %d\n", es, x0, r == CUDA_SUCCESS ? "ok" : "encode error", bad, bx * by);
    }
  }
  return 0;
}
