// Microbenchmarks that ground the executor design: FMA pipe rates for the
// operand forms the executors use, shared-memory load bandwidth, and the cost of a
// warp-uniform indirect-branch dispatch (column-stationary accumulation).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro micro.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void ffma_reg(float* out, float w, int iters) {
  float a[8], x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 0.001f + j; x[j] = j * 0.5f; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(w, x[j], a[j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __int_as_float(__float_as_int(x[j]) ^ 1);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.0f) out[threadIdx.x] = s;
}

__global__ void ffma_imm(float* out, int iters) {
  float a[8], x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 0.001f + j; x[j] = j * 0.5f; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(1.0001f + 0.37f * u, x[j], a[j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __int_as_float(__float_as_int(x[j]) ^ 1);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.0f) out[threadIdx.x] = s;
}

__device__ __forceinline__ void fma_h2(float& a0, float& a1, uint16_t w, uint32_t x2) {
  asm("{\n\t.reg .b16 xl, xh;\n\tmov.b32 {xl, xh}, %3;\n\t"
      "fma.rn.f32.f16 %0, %2, xl, %0;\n\tfma.rn.f32.f16 %1, %2, xh, %1;\n\t}"
      : "+f"(a0), "+f"(a1) : "h"(w), "r"(x2));
}

__global__ void fhfma(float* out, int iters) {
  float a[8];
  uint32_t x[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 0.001f + j;
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = 0x3c003c00u + j;
  uint16_t w = 0x3c01;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int j = 0; j < 4; ++j) fma_h2(a[2 * j], a[2 * j + 1], w, x[j]);
      w ^= 1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] ^= 0x00010001u;
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.0f) out[threadIdx.x] = s;
}

// LDS.128: each warp reads row k (uniform) of a [rows][32*16B] tile, lane-contiguous.
__global__ void lds128(float* out, int iters) {
  __shared__ float4 t[64][32];
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) t[i / 32][i % 32] = make_float4(i, 1, 2, 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float4 acc = make_float4(0, 0, 0, 0);
  int k = threadIdx.x >> 5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4 v = t[(k + u * 7) & 63][lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    k += 3;
  }
  if (acc.x == 1234.5f) out[threadIdx.x] = acc.y;
}

// Column-stationary dispatch: per entry (r, w) jump to the block updating acc[r][0..7].
template <int NR>
__global__ void brx_dispatch(const uint32_t* __restrict__ ent, int nent, float* out, int iters) {
  __shared__ uint32_t se[2048];
  __shared__ float4 xs[32][64];  // [k][lane pair]
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) se[i] = ent[i % nent];
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) xs[i / 64][i % 64] = make_float4(i, 1, 2, 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc[NR][8];
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0;
  for (int it = 0; it < iters; ++it) {
    // entry: bits 0..4 r, bits 5..10 k, bit 11 new-k flag, upper 16 bits = weight (half)
    float4 x0 = xs[0][2 * lane], x1 = xs[0][2 * lane + 1];
    for (int e = 0; e < 2048; ++e) {
      const uint32_t en = se[e];
      if (en & 0x800u) {
        const int k = (en >> 5) & 31;
        x0 = xs[k][2 * lane];
        x1 = xs[k][2 * lane + 1];
      }
      const float w = __half2float(__ushort_as_half((unsigned short)(en >> 16)));
      const int r = en & 31;
#define UPD(RR) case RR: \
      acc[RR][0] = fmaf(w, x0.x, acc[RR][0]); acc[RR][1] = fmaf(w, x0.y, acc[RR][1]); \
      acc[RR][2] = fmaf(w, x0.z, acc[RR][2]); acc[RR][3] = fmaf(w, x0.w, acc[RR][3]); \
      acc[RR][4] = fmaf(w, x1.x, acc[RR][4]); acc[RR][5] = fmaf(w, x1.y, acc[RR][5]); \
      acc[RR][6] = fmaf(w, x1.z, acc[RR][6]); acc[RR][7] = fmaf(w, x1.w, acc[RR][7]); break;
      switch (r) {
        UPD(0) UPD(1) UPD(2) UPD(3) UPD(4) UPD(5) UPD(6) UPD(7)
        UPD(8) UPD(9) UPD(10) UPD(11) UPD(12) UPD(13) UPD(14) UPD(15)
        default: break;
      }
#undef UPD
    }
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Row-stationary inner loop as in spmm_kernel v1 (fp32): entries {k, w} broadcast, LDS.128 of X.
__global__ void rowstat(const uint2* __restrict__ ent, int nent, float* out, int iters) {
  __shared__ uint2 se[1024];
  __shared__ float4 xs[64][32];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) se[i] = ent[i % nent];
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) xs[i / 32][i % 32] = make_float4(i, 1, 2, 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int it = 0; it < iters; ++it) {
    for (int e = 0; e < 1024; e += 4) {
      uint2 en[4];
      float4 xv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) en[j] = se[e + j];
#pragma unroll
      for (int j = 0; j < 4; ++j) xv[j] = xs[en[j].x & 63][lane];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float w = __uint_as_float(en[j].y);
        a0 = fmaf(w, xv[j].x, a0); a1 = fmaf(w, xv[j].y, a1);
        a2 = fmaf(w, xv[j].z, a2); a3 = fmaf(w, xv[j].w, a3);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  float* out;
  CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
  };
  const int blocks = sms * 8, threads = 256, iters = 4096;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  {
    float ms = timeit([&] { ffma_reg<<<blocks, threads>>>(out, 1.0001f, iters); });
    double fl = 2.0 * blocks * threads * iters * 32;
    printf(", \"ffma_reg_tflops\": %.2f", fl / ms / 1e9);
  }
  {
    float ms = timeit([&] { ffma_imm<<<blocks, threads>>>(out, iters); });
    double fl = 2.0 * blocks * threads * iters * 32;
    printf(", \"ffma_imm_tflops\": %.2f", fl / ms / 1e9);
  }
  {
    float ms = timeit([&] { fhfma<<<blocks, threads>>>(out, iters); });
    double fl = 2.0 * blocks * threads * iters * 32;
    printf(", \"fhfma_tflops\": %.2f", fl / ms / 1e9);
  }
  {
    float ms = timeit([&] { lds128<<<blocks, threads>>>(out, iters); });
    double by = 16.0 * blocks * threads * iters * 8;
    printf(", \"lds128_TBps\": %.2f, \"lds128_B_per_clk_per_sm\": %.1f", by / ms / 1e9,
           by / (ms * 1e-3) / (clk * 1e3) / sms);
  }
  // entries for dispatch: random r in [0,16), new-k every ~4 entries
  std::vector<uint32_t> h(2048);
  uint32_t s = 12345;
  for (int i = 0; i < 2048; ++i) {
    s = s * 1664525u + 1013904223u;
    uint32_t r = (s >> 8) & 15, k = (s >> 16) & 63, nk = (i % 4 == 0) ? 1 : 0;
    h[i] = r | (k << 5) | (nk << 11) | (0x3c00u << 16);
  }
  uint32_t* dent;
  CK(cudaMalloc(&dent, 2048 * 4));
  CK(cudaMemcpy(dent, h.data(), 2048 * 4, cudaMemcpyHostToDevice));
  {
    const int it2 = 64;
    float ms = timeit([&] { brx_dispatch<16><<<blocks, threads>>>(dent, 2048, out, it2); });
    double fl = 2.0 * blocks * threads * it2 * 2048 * 8;
    printf(", \"brx_dispatch_tflops\": %.2f", fl / ms / 1e9);
  }
  std::vector<uint2> h2(1024);
  for (int i = 0; i < 1024; ++i) {
    s = s * 1664525u + 1013904223u;
    h2[i] = make_uint2((s >> 10) & 63, 0x3f800000u);
  }
  uint2* dent2;
  CK(cudaMalloc(&dent2, 1024 * 8));
  CK(cudaMemcpy(dent2, h2.data(), 1024 * 8, cudaMemcpyHostToDevice));
  {
    const int it2 = 128;
    float ms = timeit([&] { rowstat<<<blocks, threads>>>(dent2, 1024, out, it2); });
    double fl = 2.0 * blocks * threads * it2 * 1024 * 4;
    printf(", \"rowstat_tflops\": %.2f", fl / ms / 1e9);
  }
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
