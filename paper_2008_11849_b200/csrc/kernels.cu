// Executor kernels for sm_100a (B200): the paper's Alg. 3 "SpMM for thread
// group" as a plan-driven CUDA-core kernel, and its
// implicit-im2col 3x3 convolution variant (Sec. 3.6).
//
// Mapping of the paper's tiling (Sec. 3.3) onto the B200 kernel:
//   thread block (M_blocks x N_blocks grid)  -> CTA (row panel, N tile); with
//        k_split > 1 a thread-block CLUSTER of k_split CTAs shares one
//        (panel, N tile) and splits its K chunks ("different thread blocks can
//        have different portions of the reduction axis", Fig. 2a)
//   thread group of Gsy threads               -> warp (or 32/G_k-lane group)
//   Gsy = N / N_blocks ("inner loop fixed to 1") -> lane owns C contiguous
//        columns so every X access is one 128-bit shared-memory load
//   ACC register array                        -> acc[R][C] fp32 registers,
//        statically indexed (R unrolled), never local memory
//   "Cache B[b, N_list]"                       -> X chunk [Kc x N tile] staged
//        in smem by TMA (cp.async.bulk.tensor) with the chunk's packed plan
//        block (cp.async.bulk), an mbarrier ring filled by a producer warp
//   A values "broadcast across the thread group" -> packed plan
//        entries read with warp-uniform 128-bit broadcast shared loads
//   reduction of group accumulators   -> fixed-order __shfl_xor tree
//        inside a warp; fixed-rank-order sum over distributed shared memory
//        across the CTAs of a cluster
//   C written once per tile           -> one store per output, no atomics
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>
#include <string>

#include "../../include/sparsert.h"
#include "plan.h"

namespace cg = cooperative_groups;

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

// mbarrier (shared::cta) primitives
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
// TMA: 2-D tile of X (coordinates {n, k}) -> smem, completion on an mbarrier
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// 1-D bulk copy global -> smem (16-byte multiple), completion on an mbarrier
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
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

template <bool F16>
struct EntryOps;

template <>
struct EntryOps<false> {  // {uint32 k_local, float w}; 2 per 16 bytes
  static constexpr int EB = 8;
  static constexpr int A = 2;
  template <int C, int ROWB>
  __device__ __forceinline__ static void run(float (&acc)[C], const uint8_t* ents, int beg,
                                             int cnt, const uint8_t* xs) {
    int e = 0;
    for (; e + 4 <= cnt; e += 4) {
      const uint4 p0 = *(const uint4*)(ents + (beg + e) * EB);
      const uint4 p1 = *(const uint4*)(ents + (beg + e + 2) * EB);
      const uint32_t k[4] = {p0.x, p0.z, p1.x, p1.z};
      const uint32_t w[4] = {p0.y, p0.w, p1.y, p1.w};
      float4 xv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) xv[j] = *(const float4*)(xs + k[j] * ROWB);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float wf = __uint_as_float(w[j]);
        acc[0] = fmaf(wf, xv[j].x, acc[0]);
        acc[1] = fmaf(wf, xv[j].y, acc[1]);
        acc[2] = fmaf(wf, xv[j].z, acc[2]);
        acc[3] = fmaf(wf, xv[j].w, acc[3]);
      }
    }
    for (; e < cnt; ++e) {
      const uint2 en = *(const uint2*)(ents + (beg + e) * EB);
      const float4 xv = *(const float4*)(xs + en.x * ROWB);
      const float wf = __uint_as_float(en.y);
      acc[0] = fmaf(wf, xv.x, acc[0]);
      acc[1] = fmaf(wf, xv.y, acc[1]);
      acc[2] = fmaf(wf, xv.z, acc[2]);
      acc[3] = fmaf(wf, xv.w, acc[3]);
    }
  }
};

template <>
struct EntryOps<true> {  // {uint16 k_local, half w}; 4 per 16 bytes
  static constexpr int EB = 4;
  static constexpr int A = 4;
  __device__ __forceinline__ static void one(float (&acc)[8], uint32_t en, const uint8_t* xs,
                                             int ROWB) {
    const uint4 xv = *(const uint4*)(xs + (en & 0xffffu) * ROWB);
    const uint16_t w = (uint16_t)(en >> 16);
    fma_h2(acc[0], acc[1], w, xv.x);
    fma_h2(acc[2], acc[3], w, xv.y);
    fma_h2(acc[4], acc[5], w, xv.z);
    fma_h2(acc[6], acc[7], w, xv.w);
  }
  template <int C, int ROWB>
  __device__ __forceinline__ static void run(float (&acc)[C], const uint8_t* ents, int beg,
                                             int cnt, const uint8_t* xs) {
    int e = 0;
    for (; e + 4 <= cnt; e += 4) {
      const uint4 q = *(const uint4*)(ents + (beg + e) * EB);
      const uint32_t en[4] = {q.x, q.y, q.z, q.w};
      uint4 xv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) xv[j] = *(const uint4*)(xs + (en[j] & 0xffffu) * ROWB);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint16_t w = (uint16_t)(en[j] >> 16);
        fma_h2(acc[0], acc[1], w, xv[j].x);
        fma_h2(acc[2], acc[3], w, xv[j].y);
        fma_h2(acc[4], acc[5], w, xv[j].z);
        fma_h2(acc[6], acc[7], w, xv[j].w);
      }
    }
    for (; e < cnt; ++e) one(acc, *(const uint32_t*)(ents + (beg + e) * EB), xs, ROWB);
  }
};

// ------------------------------------------------------------------ SpMM
struct SpmmArgs {
  const uint8_t* blob;
  const int64_t* blk_off;
  const int32_t* row_id;
  const uint8_t* X;
  uint8_t* Y;
  int64_t ldx, ldy, N;
  int32_t K, kc, nchunks, Mp, ks, stages, npanels;
  int32_t x_stage_bytes, stage_bytes, hdr_bytes, bar_off;
  int32_t use_tma, vec_y;
};

template <int R, int GK, bool F16>
__global__ void __launch_bounds__(288) spmm_kernel(const __grid_constant__ CUtensorMap tmap,
                                                   const SpmmArgs a) {
  constexpr int C = F16 ? 8 : 4;  // columns per lane (16 bytes of X)
  constexpr int S = F16 ? 2 : 4;  // element bytes
  constexpr int L = 32 / GK;      // lanes per thread group
  constexpr int NT = L * C;       // columns per CTA
  constexpr int ROWB = NT * S;    // bytes per staged X row
  using E = EntryOps<F16>;
  extern __shared__ __align__(1024) uint8_t smem[];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nwarps = (blockDim.x >> 5) - 1;  // consumer warps; warp `nwarps` is the producer
  const int g = lane / L, li = lane % L;
  const int col = li * C;
  // Work decomposition.  k_split == 1: persistent CTAs walk the (panel, N tile) tiles
  // t = blockIdx.x + j * gridDim.x with the panel index fastest, so CTAs running together
  // read the same X tile (L2 reuse) and the producer prefetches across tile boundaries.
  // k_split > 1: one tile per cluster; CTA rank r of the cluster takes chunk slice r.
  const bool persistent = a.ks == 1;
  const int rank = persistent ? 0 : (int)(blockIdx.x % a.ks);
  const int ntn = (int)((a.N + NT - 1) / NT);
  const int np = a.npanels;
  const int ntiles = persistent ? np * ntn : 1;
  const int cps = (a.nchunks + a.ks - 1) / a.ks;
  const int c_begin = rank * cps;
  const int nloc = max(0, min(a.nchunks, c_begin + cps) - c_begin);
  // tile walker without divisions in the loop (64-bit / runtime-divisor division is
  // emulated on the GPU and used to dominate small-K layers)
  struct TileIter {
    int t, panel, nt, step, sd, sm;
  };
  auto tile_begin = [&]() {
    TileIter it;
    if (persistent) {
      it.t = (int)blockIdx.x;
      it.panel = it.t % np;
      it.nt = it.t / np;
      it.step = (int)gridDim.x;
      it.sd = it.step / np;
      it.sm = it.step % np;
    } else {
      it.t = 0;
      it.panel = (int)(blockIdx.x / a.ks);
      it.nt = (int)blockIdx.y;
      it.step = 1;
      it.sd = 0;
      it.sm = 0;
    }
    return it;
  };
  auto tile_next = [&](TileIter& it) {
    it.t += it.step;
    it.nt += it.sd;
    it.panel += it.sm;
    if (it.panel >= np) {
      it.panel -= np;
      it.nt += 1;
    }
  };
  const uint32_t full0 = smem_u32(smem + a.bar_off);
  const uint32_t empty0 = full0 + 8 * 4;

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(full0 + 8 * s, a.use_tma ? 1 : 33);
      mbar_init(empty0 + 8 * s, nwarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  float acc[R][C];

  // Y[row][n0 + col ...] <- acc (fp16: RN once), group-0 lanes only
  auto store_tile = [&](int panel, int64_t n0, const int (&rows)[R]) {
    const int ncol = (int)min((int64_t)NT, a.N - n0);
    if (g != 0 || col >= ncol) return;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = rows[r];
      if (row < 0) continue;
      uint8_t* yp = a.Y + ((int64_t)row * a.ldy + n0 + col) * S;
      if (F16) {
        __half h[C];
#pragma unroll
        for (int c = 0; c < C; ++c) h[c] = __float2half_rn(acc[r][c]);
        if (a.vec_y && col + C <= ncol) {
          *(uint4*)yp = *(const uint4*)h;
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (col + c < ncol) ((__half*)yp)[c] = h[c];
        }
      } else {
        if (a.vec_y && col + C <= ncol) {
          *(float4*)yp = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (col + c < ncol) ((float*)yp)[c] = acc[r][c];
        }
      }
    }
  };

  if (warp == nwarps) {
    // ---------------- producer warp: TMA X tile + bulk plan block per chunk, running
    // ahead of the consumers by up to `stages` chunks (across tile boundaries)
    int s = 0, uses = 0;  // ring slot and how many times it has been filled (phase)
    uint32_t ph = 0;
    for (TileIter it = tile_begin(); it.t < ntiles; tile_next(it)) {
      const int panel = it.panel;
      const int64_t n0 = (int64_t)it.nt * NT;
      for (int j = 0; j < nloc; ++j) {
        const int c = c_begin + j;
        if (uses > 0) mbar_wait(empty0 + 8 * s, ph ^ 1u);
        uint8_t* st = smem + s * a.stage_bytes;
        const int64_t bi = (int64_t)panel * a.nchunks + c;
        const int64_t b0 = a.blk_off[bi];
        const uint32_t bbytes = (uint32_t)(a.blk_off[bi + 1] - b0);
        const uint32_t fb = full0 + 8 * s;
        if (a.use_tma) {
          if (lane == 0) {
            mbar_arrive_expect_tx(fb, (uint32_t)a.x_stage_bytes + bbytes);
            tma_load_2d(smem_u32(st), &tmap, (int)n0, c * a.kc, fb);
            bulk_load(smem_u32(st + a.x_stage_bytes), a.blob + b0, bbytes, fb);
          }
        } else {
          if (lane == 0) {
            mbar_arrive_expect_tx(fb, bbytes);
            bulk_load(smem_u32(st + a.x_stage_bytes), a.blob + b0, bbytes, fb);
          }
          const int k0 = c * a.kc;
          const int kr = min(a.kc, a.K - k0);
          const int total = kr * NT;
          for (int idx = lane; idx < total; idx += 32) {
            const int r = idx / NT, cc = idx % NT;
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
          if (F16)
            mbar_arrive(fb);
          else
            cp_async_mbar_arrive_noinc(fb);
        }
        if (++s == a.stages) {
          s = 0;
          ph ^= 1u;
          uses = 1;
        }
      }
    }
  } else {
    // ---------------- consumer warps: Alg. 3 over each staged chunk
    int s = 0;
    uint32_t ph = 0;
    for (TileIter it = tile_begin(); it.t < ntiles; tile_next(it)) {
      const int panel = it.panel;
      const int64_t n0 = (int64_t)it.nt * NT;
      int rows[R];
#pragma unroll
      for (int r = 0; r < R; ++r) rows[r] = a.row_id[(int64_t)panel * a.Mp + warp * R + r];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[r][c] = 0.0f;
      for (int j = 0; j < nloc; ++j) {
        mbar_wait(full0 + 8 * s, ph);
        const uint8_t* st = smem + s * a.stage_bytes;
        const uint8_t* xs = st + li * (C * S);
        const uint32_t* shdr = (const uint32_t*)(st + a.x_stage_bytes);
        const uint8_t* ents = st + a.x_stage_bytes + a.hdr_bytes;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t h = shdr[warp * R + r];
          int beg = (int)(h & 0xffffu);
          int cnt = (int)(h >> 16);
          if (GK > 1) {  // contiguous k-ascending pieces, all but the last of equal size
            int per = (cnt + GK - 1) / GK;
            per = (per + E::A - 1) / E::A * E::A;
            const int lo = min(g * per, cnt);
            const int hi = min(lo + per, cnt);
            beg += lo;
            cnt = hi - lo;
          }
          E::template run<C, ROWB>(acc[r], ents, beg, cnt, xs);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * s);
        if (++s == a.stages) {
          s = 0;
          ph ^= 1u;
        }
      }
      // cross-group reduction inside the warp: fixed binary tree over group index
      if (GK > 1) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int c = 0; c < C; ++c)
#pragma unroll
            for (int off = 16; off >= L; off >>= 1)
              acc[r][c] += __shfl_xor_sync(0xffffffffu, acc[r][c], off);
      }
      if (persistent) store_tile(panel, n0, rows);
    }
  }
  if (persistent) return;

  const TileIter it0 = tile_begin();
  const int panel = it0.panel;
  const int64_t n0 = (int64_t)it0.nt * NT;
  const int ncol = (int)min((int64_t)NT, a.N - n0);
  // ---------------- k_split > 1: partial tiles reduced across the cluster through DSMEM,
  // summed in rank order 0, 1, ..., ks-1 for every output (deterministic).
  __syncthreads();  // every consumer is done with the stage buffers that `red` overlays
  float* red = (float*)smem;  // [Mp][NT] fp32
  if (warp < nwarps && g == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float* dst = red + (warp * R + r) * NT + col;
#pragma unroll
      for (int c = 0; c < C; c += 4)
        *(float4*)(dst + c) = make_float4(acc[r][c], acc[r][c + 1], acc[r][c + 2], acc[r][c + 3]);
    }
  }
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  const int rows_per_rank = (a.Mp + a.ks - 1) / a.ks;
  const int s0 = rank * rows_per_rank;
  const int s1 = min(a.Mp, s0 + rows_per_rank);
  const int items = (s1 - s0) * (NT / 4);
  for (int it = tid; it < items; it += blockDim.x) {
    const int slot = s0 + it / (NT / 4);
    const int c4 = (it % (NT / 4)) * 4;
    const int row = a.row_id[(int64_t)panel * a.Mp + slot];
    if (row < 0 || c4 >= ncol) continue;
    float4 v = *(const float4*)(cluster.map_shared_rank(red, 0) + slot * NT + c4);
    for (int q = 1; q < a.ks; ++q) {
      const float4 u = *(const float4*)(cluster.map_shared_rank(red, q) + slot * NT + c4);
      v.x += u.x;
      v.y += u.y;
      v.z += u.z;
      v.w += u.w;
    }
    uint8_t* yp = a.Y + ((int64_t)row * a.ldy + n0 + c4) * S;
    const float vv[4] = {v.x, v.y, v.z, v.w};
    if (F16) {
      __half h[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) h[c] = __float2half_rn(vv[c]);
      if (a.vec_y && c4 + 4 <= ncol) {
        *(uint2*)yp = *(const uint2*)h;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c4 + c < ncol) ((__half*)yp)[c] = h[c];
      }
    } else {
      if (a.vec_y && c4 + 4 <= ncol) {
        *(float4*)yp = v;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c4 + c < ncol) ((float*)yp)[c] = vv[c];
      }
    }
  }
  cluster.sync();  // keep every CTA's smem alive until all remote reads are done
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
  extern __shared__ __align__(1024) uint8_t smem[];
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
    const uint32_t* shdr = (const uint32_t*)(st + a.x_stage_bytes);
    const uint8_t* ents = st + a.x_stage_bytes + a.hdr_bytes;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t h = shdr[warp * R + r];
      const int beg = (int)(h & 0xffffu), cnt = (int)(h >> 16);
      int e = 0;
      if (F16) {
        for (; e + 4 <= cnt; e += 4) {  // 4 entries per 128-bit broadcast load
          const uint4 q = *(const uint4*)(ents + (beg + e) * EB);
          const uint32_t en[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int off = (int)(int16_t)(en[u] & 0xffffu);
            const uint16_t w = (uint16_t)(en[u] >> 16);
            uint16_t xv[CP];
#pragma unroll
            for (int j = 0; j < CP; ++j) xv[j] = *(const uint16_t*)(st + (pos[j] + off) * 2);
#pragma unroll
            for (int j = 0; j < CP; ++j) fma_h(acc[r][j], w, xv[j]);
          }
        }
        for (; e < cnt; ++e) {
          const uint32_t en = *(const uint32_t*)(ents + (beg + e) * EB);
          const int off = (int)(int16_t)(en & 0xffffu);
          const uint16_t w = (uint16_t)(en >> 16);
#pragma unroll
          for (int j = 0; j < CP; ++j) fma_h(acc[r][j], w, *(const uint16_t*)(st + (pos[j] + off) * 2));
        }
      } else {
        for (; e + 2 <= cnt; e += 2) {  // 2 entries per 128-bit broadcast load
          const uint4 q = *(const uint4*)(ents + (beg + e) * EB);
          const int off0 = (int)q.x, off1 = (int)q.z;
          const float w0 = __uint_as_float(q.y), w1 = __uint_as_float(q.w);
          float x0[CP], x1[CP];
#pragma unroll
          for (int j = 0; j < CP; ++j) {
            x0[j] = *(const float*)(st + (pos[j] + off0) * 4);
            x1[j] = *(const float*)(st + (pos[j] + off1) * 4);
          }
#pragma unroll
          for (int j = 0; j < CP; ++j) {
            acc[r][j] = fmaf(w0, x0[j], acc[r][j]);
            acc[r][j] = fmaf(w1, x1[j], acc[r][j]);
          }
        }
        for (; e < cnt; ++e) {
          const uint2 en = *(const uint2*)(ents + (beg + e) * EB);
          const int off = (int)en.x;
          const float w = __uint_as_float(en.y);
#pragma unroll
          for (int j = 0; j < CP; ++j)
            acc[r][j] = fmaf(w, *(const float*)(st + (pos[j] + off) * 4), acc[r][j]);
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
using SpmmFn = void (*)(const __grid_constant__ CUtensorMap, const SpmmArgs);
using ConvFn = void (*)(const ConvArgs);

template <bool F16>
static SpmmFn pick_spmm(int R, int GK) {
#define SRT_S(RR, GG) \
  if (R == RR && GK == GG) return spmm_kernel<RR, GG, F16>;
#define SRT_SR(RR) SRT_S(RR, 1) SRT_S(RR, 2) SRT_S(RR, 4) SRT_S(RR, 8)
  SRT_SR(1) SRT_SR(2) SRT_SR(4) SRT_SR(8)
  if constexpr (!F16) { SRT_SR(16) }
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
  // Opt in to > 48 KB dynamic shared memory once per (kernel, device); cached so that
  // launches inside CUDA-graph capture make no driver calls.
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  static std::set<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  const auto key = std::make_pair((const void*)fn, dev);
  if (done.count(key)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute((const void*)fn,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) done.insert(key);
  return e;
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

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// Row repack of an X whose base or row stride is not 16-byte aligned (TMA needs both):
// Xp[k][0..N) = X[k][0..N), Xp with a padded row stride.  Pure data movement.
__global__ void repack_rows(const uint8_t* __restrict__ X, int64_t ldx_b, uint8_t* __restrict__ Xp,
                            int64_t ldp_b, int64_t N, int S) {
  const int64_t k = blockIdx.y;
  const uint8_t* src = X + k * ldx_b;
  uint8_t* dst = Xp + k * ldp_b;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < N;
       n += (int64_t)gridDim.x * blockDim.x) {
    if (S == 2)
      ((uint16_t*)dst)[n] = __ldg((const unsigned short*)src + n);
    else
      ((float*)dst)[n] = __ldg((const float*)src + n);
  }
}

int launch_repack(int device, int64_t K, int64_t N, int S, const void* X, int64_t ldx, void** Xp,
                  int64_t* ldp, void* stream, std::string& err) {
  DeviceGuard dg(device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  const int64_t per16 = 16 / S;
  *ldp = (N + per16 - 1) / per16 * per16;
  cudaError_t e = cudaMallocAsync(Xp, (size_t)(K * *ldp * S), (cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *Xp = nullptr;
    return cuda_fail(e, "cudaMallocAsync(repack)", err);
  }
  const unsigned gx = (unsigned)std::min<int64_t>((N + 255) / 256, 64);
  for (int64_t k0 = 0; k0 < K; k0 += 65535) {
    const int64_t kk = std::min<int64_t>(65535, K - k0);
    repack_rows<<<dim3(gx, (unsigned)kk), 256, 0, (cudaStream_t)stream>>>(
        (const uint8_t*)X + k0 * ldx * S, ldx * S, (uint8_t*)*Xp + k0 * *ldp * S, *ldp * S, N, S);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "repack launch", err);
  return SPARSE_OK;
}

void free_repack(int device, void* Xp, void* stream) {
  DeviceGuard dg(device);
  cudaFreeAsync(Xp, (cudaStream_t)stream);
}

int upload_plan(Plan& p, std::string& err) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e, "no CUDA device", err);
  }
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
  a.ks = p.ks;
  a.stages = p.stages;
  a.x_stage_bytes = p.x_stage_bytes;
  a.stage_bytes = (p.x_stage_bytes + p.max_blk_bytes + 127) & ~127;
  a.hdr_bytes = p.hdr_bytes;
  a.bar_off = p.smem_bytes - 128;
  const int smem = p.smem_bytes;
  const bool vec_x = ((uintptr_t)X % 16 == 0) && ((ldx * S) % 16 == 0);
  a.vec_y = ((uintptr_t)Y % 16 == 0) && ((ldy * S) % 16 == 0);
  a.npanels = p.npanels;
  auto encode = tensor_map_encoder();
  const int threads = (p.warps + 1) * 32;
  auto make_map = [&](CUtensorMap& tmap) {
    std::memset(&tmap, 0, sizeof tmap);
    a.use_tma = 0;
    if (vec_x && encode) {
      cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)p.K};
      cuuint64_t strides[1] = {(cuuint64_t)(ldx * S)};
      cuuint32_t box[2] = {(cuuint32_t)p.n_tile, (cuuint32_t)p.kc};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = encode(&tmap, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                          2, (void*)a.X, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      a.use_tma = r == CUDA_SUCCESS ? 1 : 0;
    }
  };
  const int64_t ntn = (N + p.n_tile - 1) / p.n_tile;
  if (p.ks == 1) {
    // persistent: one wave of CTAs, each walking tiles blockIdx.x + j * gridDim.x
    a.X = (const uint8_t*)X;
    a.Y = (uint8_t*)Y;
    a.N = N;
    CUtensorMap tmap;
    make_map(tmap);
    const int64_t ntiles = (int64_t)p.npanels * ntn;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
    fn<<<(unsigned)grid, threads, smem, (cudaStream_t)stream>>>(tmap, a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "spmm launch", err);
    return SPARSE_OK;
  }
  const int64_t kMaxY = 65535;
  for (int64_t t0 = 0; t0 < ntn; t0 += kMaxY) {
    const int64_t nt = std::min(kMaxY, ntn - t0);
    const int64_t c0 = t0 * p.n_tile;
    a.X = (const uint8_t*)X + c0 * S;
    a.Y = (uint8_t*)Y + c0 * S;
    a.N = N - c0;
    CUtensorMap tmap;
    make_map(tmap);
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3((unsigned)(p.npanels * p.ks), (unsigned)nt, 1);
    cfg.blockDim = dim3((unsigned)threads, 1, 1);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)p.ks;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, fn, tmap, a);
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
  a.hdr_bytes = p.hdr_bytes;
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
