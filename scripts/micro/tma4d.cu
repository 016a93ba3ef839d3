// Probe: one 4-D TMA box load {wp, rows, 1, cc} with variant knobs (argv), prints ok / error.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
__global__ void k(const __grid_constant__ CUtensorMap m, int x0, int y0, int b, int c0, unsigned bytes, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned ba = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"((unsigned long long)&m), "r"(x0), "r"(y0), "r"(b), "r"(c0), "r"(ba) : "memory");
    unsigned done = 0;
    while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(ba));
    out[0] = ((float*)sm)[17];
  }
}
int main(int argc, char** argv) {
  int wp = 16, H = 14, B = 256, Cin = 256, rows = atoi(argv[1]), cc = atoi(argv[2]);
  int x0 = atoi(argv[3]), y0 = atoi(argv[4]), b = atoi(argv[5]), prom = atoi(argv[6]);
  const int tw = argc > 7 ? atoi(argv[7]) : wp;
  float* xp; cudaMalloc(&xp, (size_t)tw * H * B * Cin * 4); cudaMemset(xp, 0, (size_t)tw * H * B * Cin * 4);
  float* out; cudaMalloc(&out, 4);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m; memset(&m, 0, sizeof m);
  cuuint64_t dims[4] = {(cuuint64_t)tw, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)Cin};
  cuuint64_t str[3] = {(cuuint64_t)tw * 4, (cuuint64_t)tw * 4 * H, (cuuint64_t)tw * 4 * H * B};
  cuuint32_t box[4] = {(cuuint32_t)wp, (cuuint32_t)rows, 1u, (cuuint32_t)cc};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, xp, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned bytes = wp * rows * cc * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<1, 32, bytes + 1024>>>(m, x0, y0, b, 0, bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("tw %d rows %d cc %d x0 %d y0 %d b %d prom %d encode %d -> %s\n", tw, rows, cc, x0, y0, b, prom, (int)r, cudaGetErrorString(e));
  return 0;
}
