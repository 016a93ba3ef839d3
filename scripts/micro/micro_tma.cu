// Microbenchmark: per-SM streaming throughput of TMA 2-D boxes (the X-staging pattern of
// spmm_kernel) vs 1-D bulk copies, one CTA per SM, ring of `stages` buffers, a single
// thread issues and waits (no compute).  Answers: how many bytes in flight per SM does
// HBM / L2 streaming need, and does the box shape matter?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_tma micro_tma.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(done) : "r"(bar), "r"(ph) : "memory");
  } while (!done);
}

template <bool BOX>
__global__ void stream(const __grid_constant__ CUtensorMap map, const uint8_t* src, int64_t bytes_per_chunk,
                       int chunks_total, int stages, int box_rows, int box_cols, int64_t row_stride) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // chunk c of this CTA: global chunk id = blockIdx.x + c * gridDim.x
  const int mine = (chunks_total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  auto issue = [&](int c) {
    const int s = c % stages;
    const int id = blockIdx.x + c * gridDim.x;
    const uint32_t bar = su32(&bars[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)bytes_per_chunk) : "memory");
    uint8_t* dst = smem + (int64_t)s * bytes_per_chunk;
    if (BOX) {
      // chunks tile the tensor: x = (id % ncolt) * box_cols, y = (id / ncolt) * box_rows
      const int ncolt = (int)(row_stride / 4 / box_cols);
      const int x = (id % ncolt) * box_cols, y = (id / ncolt) * box_rows;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(dst)), "l"((uint64_t)&map), "r"(x), "r"(y), "r"(bar) : "memory");
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(dst)), "l"(src + (int64_t)id * bytes_per_chunk), "r"((uint32_t)bytes_per_chunk), "r"(bar) : "memory");
    }
  };
  for (int c = 0; c < mine && c < stages; ++c) issue(c);
  for (int c = 0; c < mine; ++c) {
    wait(su32(&bars[c % stages]), (c / stages) & 1);
    if (c + stages < mine) issue(c + stages);
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 256ll << 20;  // 256 MiB: larger than L2 (HBM) ; also 32 MiB (L2)
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("[\n");
  for (int64_t span : {32ll << 20, 256ll << 20}) {
    for (int cols : {128, 256}) {          // fp32 elements per box row
      const int64_t row_stride = 25088 * 4;  // RN50 p1 X row (fp32, N = 25088)
      for (int rows : {16, 32, 64, 128}) {
        const int64_t chunk = (int64_t)rows * cols * 4;
        for (int stages : {2, 4, 6}) {
          if (chunk * stages > 200 * 1024) continue;
          const int64_t nrows = span / row_stride;
          CUtensorMap map;
          cuuint64_t dims[2] = {(cuuint64_t)(row_stride / 4), (cuuint64_t)nrows};
          cuuint64_t strides[1] = {(cuuint64_t)row_stride};
          cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)rows};
          cuuint32_t es[2] = {1, 1};
          enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          const int chunks = (int)((nrows / rows) * (row_stride / 4 / cols));
          const int smem = (int)(chunk * stages);
          for (int box = 1; box >= 0; --box) {
            auto k = box ? stream<true> : stream<false>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
            k<<<sms, 32, smem>>>(map, buf, chunk, chunks, stages, rows, cols, row_stride);
            cudaEventRecord(e0);
            for (int r = 0; r < 5; ++r) k<<<sms, 32, smem>>>(map, buf, chunk, chunks, stages, rows, cols, row_stride);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = (double)chunks * chunk * 5;
            printf(" {\"span_MB\": %lld, \"box\": %d, \"rows\": %d, \"cols\": %d, \"chunk_KB\": %lld, \"stages\": %d, \"GBps\": %.0f, \"err\": \"%s\"},\n",
                   (long long)(span >> 20), box, rows, cols, (long long)(chunk >> 10), stages, bytes / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
          }
        }
      }
    }
  }
  printf("{}]\n");
  return 0;
}
