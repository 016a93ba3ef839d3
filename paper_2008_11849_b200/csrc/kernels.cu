// Executor kernels for sm_100a (B200): the paper's Alg. 3 "SpMM for thread
// group" as a plan-driven CUDA-core kernel, and its
// implicit-im2col 3x3 convolution variant (Sec. 3.6).
//
// Mapping of the paper's tiling (Sec. 3.3) onto the B200 kernel:
//   thread block (M_blocks x N_blocks grid)  -> CTA (row panel, N tile)
//   thread group of Gsy threads               -> warp (or 32/G_k-lane group)
//   Gsy = N / N_blocks ("inner loop fixed to 1") -> lane owns C contiguous
//        columns so every X access is one 128-bit shared-memory load
//   ACC register array                        -> acc[R][C] fp32 registers,
//        statically indexed (R unrolled), never local memory
//   "Cache B[b, N_list]"                       -> X chunk staged in smem by
//        cp.async (double buffered), shared by all rows of the panel
//   A values "broadcast across the thread group" -> packed plan
//        entries staged in smem and read with warp-uniform (broadcast) loads
//   reduction of group accumulators   -> fixed-order __shfl_xor tree
//   C written once per tile           -> one store per output, no atomics
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>

#include "../../include/sparsert.h"
#include "plan.h"

namespace srt {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// acc += w * x for fp16 w, x with the product exact in fp32 and an fp32
// accumulator: mixed-precision FMA (sm_100 "fma.rn.f32.f16", SASS FHFMA).
__device__ __forceinline__ void fma_h(float& acc, uint16_t w, uint16_t x) {
  asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(w), "h"(x));
}
__device__ __forceinline__ void fma_h2(float& a0, float& a1, uint16_t w, uint32_t x2) {
  asm("{\n\t.reg .b16 xl, xh;\n\tmov.b32 {xl, xh}, %3;\n\t"
      "fma.rn.f32.f16 %0, %2, xl, %0;\n\tfma.rn.f32.f16 %1, %2, xh, %1;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "h"(w), "r"(x2));
}

// ------------------------------------------------------------------ SpMM
struct SpmmArgs {
  const uint8_t* blob;
  const int64_t* blk_off;
  const int32_t* row_id;
  const uint8_t* X;
  uint8_t* Y;
  int64_t ldx, ldy, N;
  int32_t K, kc, nchunks, Mp;
  int32_t x_stage_bytes, stage_bytes, hdr_bytes;
  int32_t vec_x, vec_y;
};

template <int R, int GK, bool F16>
__global__ void __launch_bounds__(256) spmm_kernel(const SpmmArgs a) {
  constexpr int C = F16 ? 8 : 4;   // columns per lane (16 bytes of X)
  constexpr int S = F16 ? 2 : 4;   // element bytes
  constexpr int L = 32 / GK;       // lanes per thread group
  constexpr int NT = L * C;        // columns per CTA
  constexpr int ROWB = NT * S;     // bytes per staged X row
  constexpr int SEG = ROWB / 16;   // 16-byte segments per staged X row
  constexpr int EB = F16 ? 4 : 8;  // plan entry bytes
  extern __shared__ __align__(16) uint8_t smem[];

  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane / L, li = lane % L;
  const int panel = blockIdx.x;
  const int64_t n0 = (int64_t)blockIdx.y * NT;
  const int ncol = (int)min((int64_t)NT, a.N - n0);

  float acc[R][C];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0.0f;

  auto stage = [&](int chunk, int buf) {
    uint8_t* st = smem + buf * a.stage_bytes;
    const int64_t bi = (int64_t)panel * a.nchunks + chunk;
    const int64_t b0 = a.blk_off[bi];
    const int nb = (int)((a.blk_off[bi + 1] - b0) >> 4);
    const uint32_t dblk = smem_u32(st + a.x_stage_bytes);
    for (int i = tid; i < nb; i += nthr) cp_async16(dblk + 16 * i, a.blob + b0 + 16 * i, 16);
    const int k0 = chunk * a.kc;
    const int kr = min(a.kc, a.K - k0);
    if (a.vec_x) {
      const int total = kr * SEG;
      for (int i = tid; i < total; i += nthr) {
        const int r = i / SEG, s = i % SEG;
        const int64_t n = n0 + s * (16 / S);
        const int64_t rem = (a.N - n) * S;
        const int bytes = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
        const uint8_t* gp = bytes > 0 ? a.X + ((int64_t)(k0 + r) * a.ldx + n) * S : a.X;
        cp_async16(smem_u32(st + r * ROWB + s * 16), gp, bytes);
      }
    } else {
      const int total = kr * NT;
      for (int i = tid; i < total; i += nthr) {
        const int r = i / NT, cc = i % NT;
        const int64_t n = n0 + cc;
        const uint8_t* gp = a.X + ((int64_t)(k0 + r) * a.ldx + n) * S;
        if (F16) {
          uint16_t v = 0;
          if (n < a.N) v = __ldg((const unsigned short*)gp);
          *(uint16_t*)(st + r * ROWB + cc * 2) = v;
        } else {
          cp_async4(smem_u32(st + r * ROWB + cc * 4), n < a.N ? gp : a.X, n < a.N ? 4 : 0);
        }
      }
    }
  };

  stage(0, 0);
  cp_async_commit();
  for (int c = 0; c < a.nchunks; ++c) {
    if (c + 1 < a.nchunks) {
      stage(c + 1, (c + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint8_t* st = smem + (c & 1) * a.stage_bytes;
    const uint8_t* xs = st + li * (C * S);
    const uint16_t* soff = (const uint16_t*)(st + a.x_stage_bytes);
    const uint8_t* ents = st + a.x_stage_bytes + a.hdr_bytes;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int slot = warp * R + r;
      int beg = soff[slot];
      int end = soff[slot + 1];
      if (GK > 1) {  // contiguous k-ascending pieces, all but the last of equal size
        const int cnt = end - beg;
        const int per = (cnt + GK - 1) / GK;
        const int lo = min(g * per, cnt);
        const int hi = min(lo + per, cnt);
        end = beg + hi;
        beg = beg + lo;
      }
      int e = beg;
      if (!F16) {
        for (; e + 4 <= end; e += 4) {
          uint2 en[4];
          float4 xv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) en[j] = *(const uint2*)(ents + (e + j) * EB);
#pragma unroll
          for (int j = 0; j < 4; ++j) xv[j] = *(const float4*)(xs + en[j].x * ROWB);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float w = __uint_as_float(en[j].y);
            acc[r][0] = fmaf(w, xv[j].x, acc[r][0]);
            acc[r][1] = fmaf(w, xv[j].y, acc[r][1]);
            acc[r][2] = fmaf(w, xv[j].z, acc[r][2]);
            acc[r][3] = fmaf(w, xv[j].w, acc[r][3]);
          }
        }
        for (; e < end; ++e) {
          const uint2 en = *(const uint2*)(ents + e * EB);
          const float4 xv = *(const float4*)(xs + en.x * ROWB);
          const float w = __uint_as_float(en.y);
          acc[r][0] = fmaf(w, xv.x, acc[r][0]);
          acc[r][1] = fmaf(w, xv.y, acc[r][1]);
          acc[r][2] = fmaf(w, xv.z, acc[r][2]);
          acc[r][3] = fmaf(w, xv.w, acc[r][3]);
        }
      } else {
        for (; e + 4 <= end; e += 4) {
          uint32_t en[4];
          uint4 xv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) en[j] = *(const uint32_t*)(ents + (e + j) * EB);
#pragma unroll
          for (int j = 0; j < 4; ++j) xv[j] = *(const uint4*)(xs + (en[j] & 0xffffu) * ROWB);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint16_t w = (uint16_t)(en[j] >> 16);
            fma_h2(acc[r][0], acc[r][1], w, xv[j].x);
            fma_h2(acc[r][2], acc[r][3], w, xv[j].y);
            fma_h2(acc[r][4], acc[r][5], w, xv[j].z);
            fma_h2(acc[r][6], acc[r][7], w, xv[j].w);
          }
        }
        for (; e < end; ++e) {
          const uint32_t en = *(const uint32_t*)(ents + e * EB);
          const uint4 xv = *(const uint4*)(xs + (en & 0xffffu) * ROWB);
          const uint16_t w = (uint16_t)(en >> 16);
          fma_h2(acc[r][0], acc[r][1], w, xv.x);
          fma_h2(acc[r][2], acc[r][3], w, xv.y);
          fma_h2(acc[r][4], acc[r][5], w, xv.z);
          fma_h2(acc[r][6], acc[r][7], w, xv.w);
        }
      }
    }
    __syncthreads();
  }

  // cross-group reduction: fixed binary tree over group index, no atomics
  if (GK > 1) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int off = 16; off >= L; off >>= 1)
          acc[r][c] += __shfl_xor_sync(0xffffffffu, acc[r][c], off);
  }
  if (g != 0) return;
  const int col = li * C;
  if (col >= ncol) return;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = a.row_id[(int64_t)panel * a.Mp + warp * R + r];
    if (row < 0) continue;
    uint8_t* yp = a.Y + ((int64_t)row * a.ldy + n0 + col) * S;
    if (F16) {
      __half h[C];
#pragma unroll
      for (int c = 0; c < C; ++c) h[c] = __float2half_rn(acc[r][c]);
      if (a.vec_y && col + C <= ncol) {
        *(uint4*)yp = *(const uint4*)h;
      } else {
        for (int c = 0; c < C && col + c < ncol; ++c) ((__half*)yp)[c] = h[c];
      }
    } else {
      if (a.vec_y && col + C <= ncol) {
        *(float4*)yp = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      } else {
        for (int c = 0; c < C && col + c < ncol; ++c) ((float*)yp)[c] = acc[r][c];
      }
    }
  }
}

// ------------------------------------------------------------------ conv 3x3
struct ConvArgs {
  const uint8_t* blob;
  const int64_t* blk_off;
  const int32_t* row_id;
  const uint8_t* x;
  uint8_t* y;
  int32_t B, H, W, c_in, cc, nchunks, Mp;
  int32_t x_stage_bytes, stage_bytes, hdr_bytes;
  int32_t rb, ipt, wp, simg, sci, guard, stage_elems, T, bands;
};

template <int R, int CP, bool F16>
__global__ void __launch_bounds__(256) conv3x3_kernel(const ConvArgs a) {
  constexpr int S = F16 ? 2 : 4;
  constexpr int EB = F16 ? 4 : 8;
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int panel = blockIdx.x;
  const int tile = blockIdx.y;
  const int ig = tile / a.bands, yb = tile % a.bands;
  const int y0 = yb * a.rb, b0 = ig * a.ipt;
  const int64_t plane = (int64_t)a.B * a.H * a.W;

  int pos[CP];      // smem element index of each output position (padded grid)
  int64_t out[CP];  // offset inside an output channel plane, -1 = not stored
#pragma unroll
  for (int j = 0; j < CP; ++j) {
    const int t = lane + 32 * j;
    pos[j] = a.guard;
    out[j] = -1;
    if (t < a.T) {
      const int per_img = a.rb * a.wp;
      const int i = t / per_img, rem = t % per_img;
      const int yy = rem / a.wp, xx = rem % a.wp;
      pos[j] = a.guard + i * a.simg + (yy + 1) * a.wp + xx;
      const int b = b0 + i;
      if (b < a.B && xx >= 1 && xx <= a.W)
        out[j] = ((int64_t)b * a.H + (y0 + yy)) * a.W + (xx - 1);
    }
  }

  float acc[R][CP];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < CP; ++j) acc[r][j] = 0.0f;

  // zero both stages once: the halo (padding 1) is never overwritten
  for (int i = tid; i < 2 * a.stage_bytes / 4; i += nthr) ((uint32_t*)smem)[i] = 0u;
  __syncthreads();

  auto stage = [&](int chunk, int buf) {
    uint8_t* st = smem + buf * a.stage_bytes;
    const int64_t bi = (int64_t)panel * a.nchunks + chunk;
    const int64_t blk0 = a.blk_off[bi];
    const int nb = (int)((a.blk_off[bi + 1] - blk0) >> 4);
    const uint32_t dblk = smem_u32(st + a.x_stage_bytes);
    for (int i = tid; i < nb; i += nthr) cp_async16(dblk + 16 * i, a.blob + blk0 + 16 * i, 16);
    const int ci0 = chunk * a.cc;
    const int ncc = min(a.cc, a.c_in - ci0);
    const int rows = a.rb + 2;
    const int total = ncc * a.ipt * rows * a.W;
    for (int idx = tid; idx < total; idx += nthr) {
      const int xc = idx % a.W;
      int q = idx / a.W;
      const int r = q % rows;
      q /= rows;
      const int i = q % a.ipt;
      const int cl = q / a.ipt;
      const int b = b0 + i, yr = y0 - 1 + r;
      if (b >= a.B || yr < 0 || yr >= a.H) continue;
      const int64_t src = (((int64_t)(ci0 + cl) * a.B + b) * a.H + yr) * a.W + xc;
      const int dst = a.guard + cl * a.sci + i * a.simg + r * a.wp + xc + 1;
      if (F16) {
        *(uint16_t*)(st + dst * 2) = __ldg((const unsigned short*)(a.x + src * 2));
      } else {
        cp_async4(smem_u32(st + dst * 4), a.x + src * 4, 4);
      }
    }
  };

  stage(0, 0);
  cp_async_commit();
  for (int c = 0; c < a.nchunks; ++c) {
    if (c + 1 < a.nchunks) {
      stage(c + 1, (c + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint8_t* st = smem + (c & 1) * a.stage_bytes;
    const uint16_t* soff = (const uint16_t*)(st + a.x_stage_bytes);
    const uint8_t* ents = st + a.x_stage_bytes + a.hdr_bytes;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int slot = warp * R + r;
      const int beg = soff[slot], end = soff[slot + 1];
      for (int e = beg; e < end; ++e) {
        if (F16) {
          const uint32_t en = *(const uint32_t*)(ents + e * EB);
          const int off = (int)(int16_t)(en & 0xffffu);
          const uint16_t w = (uint16_t)(en >> 16);
#pragma unroll
          for (int j = 0; j < CP; ++j) {
            const uint16_t xv = *(const uint16_t*)(st + (pos[j] + off) * 2);
            fma_h(acc[r][j], w, xv);
          }
        } else {
          const uint2 en = *(const uint2*)(ents + e * EB);
          const int off = (int)en.x;
          const float w = __uint_as_float(en.y);
#pragma unroll
          for (int j = 0; j < CP; ++j) {
            const float xv = *(const float*)(st + (pos[j] + off) * 4);
            acc[r][j] = fmaf(w, xv, acc[r][j]);
          }
        }
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = a.row_id[(int64_t)panel * a.Mp + warp * R + r];
    if (row < 0) continue;
#pragma unroll
    for (int j = 0; j < CP; ++j) {
      if (out[j] < 0) continue;
      const int64_t o = (int64_t)row * plane + out[j];
      if (F16)
        ((__half*)a.y)[o] = __float2half_rn(acc[r][j]);
      else
        ((float*)a.y)[o] = acc[r][j];
    }
  }
}

// ------------------------------------------------------------------ dispatch
using SpmmFn = void (*)(const SpmmArgs);
using ConvFn = void (*)(const ConvArgs);

template <bool F16>
static SpmmFn pick_spmm(int R, int GK) {
#define SRT_S(RR, GG) \
  if (R == RR && GK == GG) return spmm_kernel<RR, GG, F16>;
#define SRT_SR(RR) SRT_S(RR, 1) SRT_S(RR, 2) SRT_S(RR, 4) SRT_S(RR, 8)
  SRT_SR(1) SRT_SR(2) SRT_SR(4) SRT_SR(8)
#undef SRT_SR
#undef SRT_S
  return nullptr;
}

template <bool F16>
static ConvFn pick_conv(int R, int CP) {
#define SRT_C(RR, CC) \
  if (R == RR && CP == CC) return conv3x3_kernel<RR, CC, F16>;
#define SRT_CR(RR) SRT_C(RR, 2) SRT_C(RR, 4) SRT_C(RR, 7) SRT_C(RR, 8)
  SRT_CR(1) SRT_CR(2) SRT_CR(4) SRT_CR(8)
#undef SRT_CR
#undef SRT_C
  return nullptr;
}

static std::mutex g_attr_mu;

template <typename Fn>
static cudaError_t ensure_smem_attr(Fn fn, int bytes) {
  // Opt in to > 48 KB dynamic shared memory once per kernel (idempotent).
  if (bytes <= 48 * 1024) return cudaSuccess;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  return cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              227 * 1024);
}

struct DeviceGuard {
  int prev = -1;
  bool switched = false;
  cudaError_t st = cudaSuccess;
  explicit DeviceGuard(int dev) {
    st = cudaGetDevice(&prev);
    if (st == cudaSuccess && prev != dev) {
      st = cudaSetDevice(dev);
      switched = st == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (switched) cudaSetDevice(prev);
  }
};

static int cuda_fail(cudaError_t e, const char* what, std::string& err) {
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return SPARSE_ECUDA;
}

int upload_plan(Plan& p, std::string& err) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e, "no CUDA device", err);
  if (p.device < 0) {
    e = cudaGetDevice(&p.device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice", err);
  }
  if (p.device >= ndev) {
    err = "device ordinal out of range";
    return SPARSE_EINVAL;
  }
  DeviceGuard dg(p.device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  const size_t nrow = p.row_id.size() * 4, noff = p.blk_off.size() * 8, nblob = p.blob.size();
  const size_t o_off = 0, o_row = (noff + 255) & ~size_t(255),
               o_blob = (o_row + nrow + 255) & ~size_t(255);
  const size_t total = o_blob + nblob;
  void* mem = nullptr;
  e = cudaMalloc(&mem, total);
  if (e != cudaSuccess) {
    cudaGetLastError();
    err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
    return SPARSE_ENOMEM;
  }
  uint8_t* b = (uint8_t*)mem;
  if ((e = cudaMemcpy(b + o_off, p.blk_off.data(), noff, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(b + o_row, p.row_id.data(), nrow, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(b + o_blob, p.blob.data(), nblob, cudaMemcpyHostToDevice)) != cudaSuccess) {
    cudaFree(mem);
    return cuda_fail(e, "cudaMemcpy(plan)", err);
  }
  p.d_mem = mem;
  p.d_blk_off = (const int64_t*)(b + o_off);
  p.d_row_id = (const int32_t*)(b + o_row);
  p.d_blob = b + o_blob;
  return SPARSE_OK;
}

void free_plan_device(Plan& p) {
  if (p.d_mem) {
    DeviceGuard dg(p.device);
    cudaFree(p.d_mem);
    p.d_mem = nullptr;
  }
}

int launch_spmm(const Plan& p, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy,
                void* stream, std::string& err) {
  const bool f16 = p.dtype == SPARSE_F16;
  const int S = f16 ? 2 : 4;
  SpmmFn fn = f16 ? pick_spmm<true>(p.R, p.gk) : pick_spmm<false>(p.R, p.gk);
  if (!fn) {
    err = "internal: no kernel instance for this tile configuration";
    return SPARSE_EINTERNAL;
  }
  DeviceGuard dg(p.device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  cudaError_t e = ensure_smem_attr(fn, p.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
  SpmmArgs a;
  a.blob = p.d_blob;
  a.blk_off = p.d_blk_off;
  a.row_id = p.d_row_id;
  a.ldx = ldx;
  a.ldy = ldy;
  a.K = p.K;
  a.kc = p.kc;
  a.nchunks = p.nchunks;
  a.Mp = p.Mp;
  a.x_stage_bytes = p.x_stage_bytes;
  a.stage_bytes = p.x_stage_bytes + p.max_blk_bytes;
  a.hdr_bytes = ((p.Mp + 1) * 2 + 15) & ~15;
  a.vec_x = ((uintptr_t)X % 16 == 0) && ((ldx * S) % 16 == 0);
  a.vec_y = ((uintptr_t)Y % 16 == 0) && ((ldy * S) % 16 == 0);
  const int64_t ntiles = (N + p.n_tile - 1) / p.n_tile;
  const int64_t kMaxY = 65535;
  for (int64_t t0 = 0; t0 < ntiles; t0 += kMaxY) {
    const int64_t nt = std::min(kMaxY, ntiles - t0);
    const int64_t c0 = t0 * p.n_tile;
    a.X = (const uint8_t*)X + c0 * S;
    a.Y = (uint8_t*)Y + c0 * S;
    a.N = N - c0;
    dim3 grid((unsigned)p.npanels, (unsigned)nt);
    fn<<<grid, p.warps * 32, p.smem_bytes, (cudaStream_t)stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "spmm launch", err);
  }
  return SPARSE_OK;
}

int launch_conv3x3(const Plan& p, int64_t batch, const void* x, void* y, void* stream,
                   std::string& err) {
  const bool f16 = p.dtype == SPARSE_F16;
  ConvFn fn = f16 ? pick_conv<true>(p.R, p.C) : pick_conv<false>(p.R, p.C);
  if (!fn) {
    err = "internal: no conv kernel instance for this tile configuration";
    return SPARSE_EINTERNAL;
  }
  if (batch > INT32_MAX) {
    err = "batch too large";
    return SPARSE_EUNSUPPORTED;
  }
  DeviceGuard dg(p.device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  cudaError_t e = ensure_smem_attr(fn, p.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
  ConvArgs a;
  a.blob = p.d_blob;
  a.blk_off = p.d_blk_off;
  a.row_id = p.d_row_id;
  a.x = (const uint8_t*)x;
  a.y = (uint8_t*)y;
  a.B = (int32_t)batch;
  a.H = p.h;
  a.W = p.w;
  a.c_in = p.c_in;
  a.cc = p.cc;
  a.nchunks = p.nchunks;
  a.Mp = p.Mp;
  a.x_stage_bytes = p.x_stage_bytes;
  a.stage_bytes = p.x_stage_bytes + p.max_blk_bytes;
  a.hdr_bytes = ((p.Mp + 1) * 2 + 15) & ~15;
  a.rb = p.conv_rb;
  a.ipt = p.conv_ipt;
  a.wp = p.conv_wp;
  a.simg = p.conv_simg;
  a.sci = p.conv_sci;
  a.guard = p.conv_guard;
  a.stage_elems = p.conv_stage_elems;
  a.T = p.n_tile;
  a.bands = p.h / p.conv_rb;
  const int64_t groups = (batch + p.conv_ipt - 1) / p.conv_ipt;
  const int64_t ntiles = groups * a.bands;
  if (ntiles > 65535) {
    err = "conv: too many tiles for one launch (batch too large)";
    return SPARSE_EUNSUPPORTED;
  }
  dim3 grid((unsigned)p.npanels, (unsigned)ntiles);
  fn<<<grid, p.warps * 32, p.smem_bytes, (cudaStream_t)stream>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "conv3x3 launch", err);
  return SPARSE_OK;
}

}  // namespace srt
