// Microbenchmark: the row-stationary SpMM inner loop (Alg. 3) with X rows read from TMEM
// (tcgen05.ld.32x32b.x4, warp-uniform column = 4*k) vs from shared memory (LDS.128), plan
// entries from shared memory in both.  fp32, R rows per warp walked jointly, 16 warps/CTA,
// one CTA per SM.  Reports lane-FMA throughput (TFLOP/s = 2 flops per lane-FMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_tmem_loop micro_tmem_loop.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void ldtm4(uint32_t taddr, float4& v) {
  uint32_t a, b, c, d;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(taddr));
  v = make_float4(__uint_as_float(a), __uint_as_float(b), __uint_as_float(c), __uint_as_float(d));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int R, bool TMEM>
__global__ void __launch_bounds__(512, 1) loop(float* out, int iters, int units_per_row) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // plan: units_per_row * R units per warp-row set, each unit {xoff, w, xoff, w} with pseudo-random k < 64
  uint4* ents = (uint4*)smem;
  const int nunits = units_per_row * R;
  for (int i = threadIdx.x; i < nunits; i += blockDim.x) {
    uint32_t h = i * 2654435761u;
    const uint32_t k0 = (h >> 8) & 63, k1 = (h >> 16) & 63;
    ents[i] = make_uint4(k0 * 512, __float_as_uint(1.0f + (h & 7)), k1 * 512, __float_as_uint(0.5f));
  }
  uint8_t* xs = smem + 16 * 4096;  // 64 rows x 512 B
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) ((float*)xs)[i] = (float)(i & 15);
  if (TMEM && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = TMEM ? tbase_s + (((uint32_t)(warp & 3) * 32) << 16) : 0;
  if (TMEM) {  // fill TMEM columns 4k..4k+3 of every lane with X row k (lane's 4 floats)
    for (int k = 0; k < 64; ++k) {
      const float4 v = *(const float4*)(xs + k * 512 + lane * 16);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tb + 4 * k),
                   "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                   "r"(__float_as_uint(v.w)));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  __syncthreads();
  float acc[R][4] = {};
  const uint8_t* xl = xs + lane * 16;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int u = 0; u < units_per_row; ++u) {
      uint4 q[R];
#pragma unroll
      for (int r = 0; r < R; ++r) q[r] = ents[r * units_per_row + u];
      float4 x0[R], x1[R];
      if (TMEM) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ldtm4(tb + (q[r].x >> 7), x0[r]);
          ldtm4(tb + (q[r].z >> 7), x1[r]);
        }
        wait_ld();
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          x0[r] = *(const float4*)(xl + q[r].x);
          x1[r] = *(const float4*)(xl + q[r].z);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float w0 = __uint_as_float(q[r].y), w1 = __uint_as_float(q[r].w);
        acc[r][0] = fmaf(w0, x0[r].x, acc[r][0]); acc[r][1] = fmaf(w0, x0[r].y, acc[r][1]);
        acc[r][2] = fmaf(w0, x0[r].z, acc[r][2]); acc[r][3] = fmaf(w0, x0[r].w, acc[r][3]);
        acc[r][0] = fmaf(w1, x1[r].x, acc[r][0]); acc[r][1] = fmaf(w1, x1[r].y, acc[r][1]);
        acc[r][2] = fmaf(w1, x1[r].z, acc[r][2]); acc[r][3] = fmaf(w1, x1[r].w, acc[r][3]);
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < R; ++r) s += acc[r][0] + acc[r][1] + acc[r][2] + acc[r][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (TMEM && warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase_s));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = 16 * 4096 + 64 * 512;
  auto run = [&](const char* name, auto k, int threads, int R) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 200, upr = 64;
    k<<<sms, threads, smem>>>(out, 2, upr);
    cudaEventRecord(e0);
    k<<<sms, threads, smem>>>(out, iters, upr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)sms * threads * iters * upr * R * 2 * 4;
    printf("%s threads=%d R=%d: %.2f TFLOP/s (%s)\n", name, threads, R, 2 * fmas / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("smem", loop<2, false>, 512, 2);
  run("tmem", loop<2, true>, 512, 2);
  run("smem", loop<4, false>, 512, 4);
  run("tmem", loop<4, true>, 512, 4);
  run("smem", loop<8, false>, 512, 8);
  run("tmem", loop<8, true>, 512, 8);
  run("smem", loop<4, false>, 256, 4);
  run("tmem", loop<4, true>, 256, 4);
  return 0;
}
