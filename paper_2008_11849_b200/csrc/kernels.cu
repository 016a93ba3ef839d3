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
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <mutex>
#include <set>
#include <type_traits>
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
// the wait with cluster-scope acquire: the phase was completed (also) by a release.cluster
// arrive of another CTA of the cluster (CTA pairs: rank 1 forwards its stages to rank 0)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
// arrive on an mbarrier of another CTA of the cluster (shared::cluster address)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// the same wait with a suspend-time hint: the warp sleeps until the phase completes (or the
// hint elapses) instead of re-polling, so waiting warps do not steal issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(0x100000u)
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

// ---- thread-block-cluster helpers (X multicast clusters)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address of this CTA -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t bar_cluster, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(
                   bar_cluster), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint32_t atom_add_cluster(uint32_t addr_cluster, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr_cluster), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// TMA 2-D box multicast to the CTAs of `mask` (same smem offset and mbarrier offset in each)
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                               uint32_t bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
      : "memory");
}

// acc += w * x for fp16 w, x with the product exact in fp32 and an fp32
// accumulator: mixed-precision FMA (sm_100 "fma.rn.f32.f16", SASS FHFMA).
__device__ __forceinline__ void fma_h(float& acc, uint16_t w, uint16_t x) {
  asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(w), "h"(x));
}
template <bool BF = false>
__device__ __forceinline__ void fma_h2(float& a0, float& a1, uint16_t w, uint32_t x2) {
  if (BF)  // bfloat16 inputs (SASS FHFMA.BF16), fp32 accumulate
    asm("{\n\t.reg .b16 xl, xh;\n\tmov.b32 {xl, xh}, %3;\n\t"
        "fma.rn.f32.bf16 %0, %2, xl, %0;\n\tfma.rn.f32.bf16 %1, %2, xh, %1;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "h"(w), "r"(x2));
  else
    asm("{\n\t.reg .b16 xl, xh;\n\tmov.b32 {xl, xh}, %3;\n\t"
        "fma.rn.f32.f16 %0, %2, xl, %0;\n\tfma.rn.f32.f16 %1, %2, xh, %1;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "h"(w), "r"(x2));
}

// Inner loop of Alg. 3 for one thread group, one row and one staged chunk: `cnt`
// 16-byte units of packed entries (plan.h), each one warp-uniform broadcast load;
// per entry one 128-bit shared load of the lane's C columns of X row k and C FMAs.
// Entries are applied in storage (k-ascending) order; neutral padding entries
// (-0 times the zero row) leave acc unchanged bit for bit.
__device__ __forceinline__ void fma4(float (&acc)[4], uint32_t wbits, const float4 x) {
  const float w = __uint_as_float(wbits);
  acc[0] = fmaf(w, x.x, acc[0]);
  acc[1] = fmaf(w, x.y, acc[1]);
  acc[2] = fmaf(w, x.z, acc[2]);
  acc[3] = fmaf(w, x.w, acc[3]);
}
template <bool BF = false>
__device__ __forceinline__ void fma8h(float (&acc)[8], uint32_t en, const uint4 xv) {
  const uint16_t w = (uint16_t)(en >> 16);
  fma_h2<BF>(acc[0], acc[1], w, xv.x);
  fma_h2<BF>(acc[2], acc[3], w, xv.y);
  fma_h2<BF>(acc[4], acc[5], w, xv.z);
  fma_h2<BF>(acc[6], acc[7], w, xv.w);
}
// fp32 -> 16-bit output bits, round to nearest even (fp16 or bf16)
template <bool BF>
__device__ __forceinline__ uint16_t to16(float v) {
  if (BF) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
  return __half_as_ushort(__float2half_rn(v));
}
template <bool BF>
__device__ __forceinline__ float from16(const void* p) {
  if (BF) return __bfloat162float(*(const __nv_bfloat16*)p);
  return __half2float(*(const __half*)p);
}

template <bool F16, bool BF = false>
struct EntryOps;

template <>
struct EntryOps<false, false> {  // unit = 2 x {uint32 xoff (bytes), float w}
  static constexpr int C = 4;
  __device__ __forceinline__ static void unit(float (&acc)[4], const uint4 p, const uint8_t* xs) {
    const float4 x0 = *(const float4*)(xs + p.x);
    const float4 x1 = *(const float4*)(xs + p.z);
    fma4(acc, p.y, x0);
    fma4(acc, p.w, x1);
  }
};

template <bool BF>
struct EntryOps<true, BF> {  // unit = 4 x {uint16 xoff (16-byte units), half / bf16 w}
  static constexpr int C = 8;
  __device__ __forceinline__ static const uint8_t* xrow(const uint8_t* xs, uint32_t en) {
    return xs + ((en & 0xffffu) << 4);
  }
  __device__ __forceinline__ static void unit(float (&acc)[8], const uint4 q, const uint8_t* xs) {
    const uint4 x0 = *(const uint4*)xrow(xs, q.x);
    const uint4 x1 = *(const uint4*)xrow(xs, q.y);
    const uint4 x2 = *(const uint4*)xrow(xs, q.z);
    const uint4 x3 = *(const uint4*)xrow(xs, q.w);
    fma8h<BF>(acc, q.x, x0);
    fma8h<BF>(acc, q.y, x1);
    fma8h<BF>(acc, q.z, x2);
    fma8h<BF>(acc, q.w, x3);
  }
};

// One thread group's R rows over one staged chunk.  The rows are walked jointly for
// their common unit count (R independent load->FMA chains per step: the latency of the
// broadcast plan load and of the X load of one row hides behind the others), then each
// row's remaining units.  Every row still applies its own entries in storage
// (k-ascending) order, so the result is the same as walking the rows one by one.
#ifndef SRT_JOINT
#define SRT_JOINT 1
#endif
#ifndef SRT_MINB
#define SRT_MINB 1
#endif
#ifndef SRT_TAILMERGE
#define SRT_TAILMERGE 1
#endif
template <bool F16, bool BF = false>
__device__ __forceinline__ void run_one_row(float (&acc)[F16 ? 8 : 4], const uint4* up, int u, int cnt,
                                            const uint8_t* xs) {
  using E = EntryOps<F16, BF>;
#pragma unroll 1
  for (; u + 2 <= cnt; u += 2) {
    const uint4 q0 = up[u], q1 = up[u + 1];
    E::unit(acc, q0, xs);
    E::unit(acc, q1, xs);
  }
  if (u < cnt) E::unit(acc, up[u], xs);
}

template <bool F16, int R, bool BF = false, int JP = R>
__device__ __forceinline__ void run_rows(float (&acc)[R][F16 ? 8 : 4], const uint32_t (&h)[R],
                                         const uint4* ents, const uint8_t* xs) {
  using E = EntryOps<F16, BF>;
#if SRT_JOINT == 0
#pragma unroll
  for (int r = 0; r < R; ++r) run_one_row<F16, BF>(acc[r], ents + (h[r] & 0xffffu), 0, (int)(h[r] >> 16), xs);
#else
  // rows walked jointly (JP < R: in groups of JP rows, fewer live plan registers)
  constexpr int P = (SRT_JOINT == 2 && R > 2) ? 2 : JP;
#pragma unroll
  for (int r0 = 0; r0 < R; r0 += P) {
    int mn = (int)(h[r0] >> 16);
#pragma unroll
    for (int r = 1; r < P; ++r) mn = min(mn, (int)(h[r0 + r] >> 16));
    const uint4* pr[P];
#pragma unroll
    for (int r = 0; r < P; ++r) pr[r] = ents + (h[r0 + r] & 0xffffu);
    int u = 0;
#pragma unroll 1
    for (; u + 2 <= mn; u += 2) {  // two steps per trip: both steps' loads in flight
      uint4 q[P], q2[P];
#pragma unroll
      for (int r = 0; r < P; ++r) {
        q[r] = pr[r][0];
        q2[r] = pr[r][1];
        pr[r] += 2;
      }
#pragma unroll
      for (int r = 0; r < P; ++r) E::unit(acc[r0 + r], q[r], xs);
#pragma unroll
      for (int r = 0; r < P; ++r) E::unit(acc[r0 + r], q2[r], xs);
    }
    if (u < mn) {
#pragma unroll
      for (int r = 0; r < P; ++r) E::unit(acc[r0 + r], pr[r][0], xs);
      ++u;
    }
#pragma unroll
    for (int r = 0; r < P; ++r)
      run_one_row<F16, BF>(acc[r0 + r], ents + (h[r0 + r] & 0xffffu), mn, (int)(h[r0 + r] >> 16), xs);
  }
#endif
}

// ---- TMEM X source (tcgen05): X rows of a chunk live in tensor memory, replicated to the
// four 32-lane quarters, so every warp reads row k of its 32 lanes with one warp-uniform
// tcgen05.ld (X row k of a 512-byte staged row -> TMEM columns 4k..4k+3 of each lane).
__device__ __forceinline__ void ldtm4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// shared-memory matrix descriptor (sm_100, SWIZZLE_NONE) of one 512-byte X row seen as a
// 32 x 16-byte matrix: 8-row core matrices 128 bytes apart (stride byte offset)
__device__ __forceinline__ uint64_t tm_row_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void tm_cp_row(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}
__device__ __forceinline__ void tm_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

template <bool F16>
struct TmOps;
template <>
struct TmOps<false> {  // unit = 2 x {uint32 xoff = 512 k, float w}: TMEM column 4k = xoff >> 7
  __device__ __forceinline__ static void load(const uint4 q, uint32_t tq, uint32_t (&x)[2][4]) {
    ldtm4(tq + (q.x >> 7), x[0]);
    ldtm4(tq + (q.z >> 7), x[1]);
  }
  __device__ __forceinline__ static void fma(float (&acc)[4], const uint4 q, const uint32_t (&x)[2][4]) {
    fma4(acc, q.y, make_float4(__uint_as_float(x[0][0]), __uint_as_float(x[0][1]),
                               __uint_as_float(x[0][2]), __uint_as_float(x[0][3])));
    fma4(acc, q.w, make_float4(__uint_as_float(x[1][0]), __uint_as_float(x[1][1]),
                               __uint_as_float(x[1][2]), __uint_as_float(x[1][3])));
  }
  static constexpr int NL = 2;
};
template <>
struct TmOps<true> {  // unit = 4 x {uint16 xoff16 = 32 k, half w}: TMEM column 4k = xoff16 >> 3
  __device__ __forceinline__ static void load(const uint4 q, uint32_t tq, uint32_t (&x)[4][4]) {
    ldtm4(tq + ((q.x & 0xffffu) >> 3), x[0]);
    ldtm4(tq + ((q.y & 0xffffu) >> 3), x[1]);
    ldtm4(tq + ((q.z & 0xffffu) >> 3), x[2]);
    ldtm4(tq + ((q.w & 0xffffu) >> 3), x[3]);
  }
  __device__ __forceinline__ static void fma(float (&acc)[8], const uint4 q, const uint32_t (&x)[4][4]) {
    fma8h(acc, q.x, make_uint4(x[0][0], x[0][1], x[0][2], x[0][3]));
    fma8h(acc, q.y, make_uint4(x[1][0], x[1][1], x[1][2], x[1][3]));
    fma8h(acc, q.z, make_uint4(x[2][0], x[2][1], x[2][2], x[2][3]));
    fma8h(acc, q.w, make_uint4(x[3][0], x[3][1], x[3][2], x[3][3]));
  }
  static constexpr int NL = 4;
};

// run_rows with X from TMEM (tq = this warp's lane quarter + the chunk's buffer column): the
// R rows are walked jointly for their common unit count (one tcgen05.wait::ld per step of R
// rows), then each row's remaining units.
template <bool F16, int R>
__device__ __forceinline__ void run_rows_tm(float (&acc)[R][F16 ? 8 : 4], const uint32_t (&h)[R],
                                            const uint4* ents, uint32_t tq) {
  using T = TmOps<F16>;
  int mn = (int)(h[0] >> 16);
#pragma unroll
  for (int r = 1; r < R; ++r) mn = min(mn, (int)(h[r] >> 16));
#pragma unroll 1
  for (int u = 0; u < mn; ++u) {
    uint4 q[R];
    uint32_t x[R][T::NL][4];
#pragma unroll
    for (int r = 0; r < R; ++r) q[r] = ents[(h[r] & 0xffffu) + u];
#pragma unroll
    for (int r = 0; r < R; ++r) T::load(q[r], tq, x[r]);
    tm_wait_ld();
#pragma unroll
    for (int r = 0; r < R; ++r) T::fma(acc[r], q[r], x[r]);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint4* up = ents + (h[r] & 0xffffu);
    const int cnt = (int)(h[r] >> 16);
#pragma unroll 1
    for (int u = mn; u < cnt; ++u) {
      const uint4 q = up[u];
      uint32_t x[T::NL][4];
      T::load(q, tq, x);
      tm_wait_ld();
      T::fma(acc[r], q, x);
    }
  }
}

// Fused epilogue on one output value: act(acc + bias[row] + beta * y_old), fp32.
template <bool F16, bool BF = false>
__device__ __forceinline__ float epilogue_one(float v, const uint8_t* bias, int row, float beta,
                                              const uint8_t* yold, int relu) {
  if (bias) v += F16 ? from16<BF>((const uint16_t*)bias + row) : ((const float*)bias)[row];
  if (beta != 0.0f) v = fmaf(beta, F16 ? from16<BF>(yold) : *(const float*)yold, v);
  if (relu) v = v < 0.0f ? 0.0f : v;
  return v;
}

// ------------------------------------------------------------------ SpMM
struct SpmmArgs {
  const uint8_t* blob;
  const int64_t* blk_off;
  const int32_t* row_id;
  const uint8_t* X;
  uint8_t* Y;
  int64_t ldx, ldy, N;
  int32_t K, kc, nchunks, Mp, ks, stages, npanels;
  int32_t x_stage_bytes, stage_bytes, hdr_bytes, bar_off, blk_bytes;
  int32_t use_tma, vec_y, cm;
  const uint8_t* bias;  // fused epilogue (plan.h Epilogue)
  float beta;
  int32_t relu;
  const float* tcws;    // tensor-core sub-block partial sums (fp32, ldws), or null
  const int32_t* ws_row;
  int64_t ldws;
};

template <int R, int GK, bool F16, bool TM, bool BF = false>
__global__ void __launch_bounds__(512, SRT_MINB) spmm_kernel(const __grid_constant__ CUtensorMap tmap,
                                                   const SpmmArgs a) {
  constexpr int C = F16 ? 8 : 4;  // columns per lane (16 bytes of X)
  constexpr int S = F16 ? 2 : 4;  // element bytes
  constexpr int L = 32 / GK;      // lanes per thread group
  constexpr int NT = L * C;       // columns per CTA
  constexpr int ROWB = NT * S;    // bytes per staged X row
  extern __shared__ __align__(1024) uint8_t smem[];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;  // every warp consumes (no dedicated producer warp)
  const int g = lane / L, li = lane % L;
  const int col = li * C;
  // Work decomposition.  k_split == 1: persistent CTAs walk the (panel, N tile) tiles
  // t = blockIdx.x + i * gridDim.x with the panel index fastest, so CTAs running together
  // read the same X tile (L2 reuse); the ring of stages runs across tile boundaries.
  // k_split > 1: one tile per cluster; CTA rank r of the cluster takes chunk slice r.
  const bool persistent = a.ks == 1;
  const int rank = persistent ? 0 : (int)(blockIdx.x % a.ks);
  const int np = a.npanels;
  // X multicast cluster (persistent only): cm CTAs take panels pg*cm + crank of the same tile
  const int cm = a.cm;
  const uint32_t crank = cm > 1 ? cluster_rank() : 0u;
  const int cid = (int)blockIdx.x / cm, ncl = (int)gridDim.x / cm;
  const int npg = np / cm;
  const int ntiles = persistent ? npg * (int)((a.N + NT - 1) / NT) : 1;
  const int my_tiles = !persistent ? 1 : (ntiles > cid ? (ntiles - 1 - cid) / ncl + 1 : 0);
  const int cps = (a.nchunks + a.ks - 1) / a.ks;
  const int c_begin = rank * cps;
  const int nloc = max(0, min(a.nchunks, c_begin + cps) - c_begin);
  const int total = my_tiles * nloc;  // chunks this CTA consumes, in ring order
  // tile ti of this CTA (cluster): panel group fastest, so clusters running together read
  // the same X tile (L2 reuse); the ring of stages runs across tile boundaries
  auto tile_of = [&](int ti, int& pg, int64_t& n0) {
    if (persistent) {
      const int t = cid + ti * ncl;
      pg = t % npg;
      n0 = (int64_t)(t / npg) * NT;
    } else {
      pg = (int)(blockIdx.x / a.ks);
      n0 = (int64_t)blockIdx.y * NT;
    }
  };
  const uint32_t full0 = smem_u32(smem + a.bar_off);
  // smem tail (256 B): full[8] mbarriers | cluster-empty[8] mbarriers (multicast leader) |
  // release counters[8] | TMEM base
  const uint32_t cempty0 = full0 + 8 * kMaxStages;
  uint32_t* ctr = (uint32_t*)(smem + a.bar_off + 16 * kMaxStages);  // releases per ring slot

  // the zero row after the kc X rows of every stage (target of neutral padding entries)
  for (int s = 0; s < a.stages; ++s)
    for (int i = tid; i < ROWB / 16; i += blockDim.x)
      *(uint4*)(smem + s * a.stage_bytes + a.kc * ROWB + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
  if (tid < kMaxStages) ctr[tid] = 0u;
  // TMEM X source: chunk q lives in TMEM buffer q & 1 (columns 256 b .. 256 b + 4 kc, zero
  // row at column 256 b + 4 kc), replicated in the four 32-lane quarters
  uint32_t* tslot = (uint32_t*)(smem + a.bar_off + 16 * kMaxStages + 4 * kMaxStages);
  if (TM && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(full0 + 8 * s, a.use_tma ? 1 : 33);
    for (int s = 0; cm > 1 && s < a.stages; ++s) mbar_init(cempty0 + 8 * s, (uint32_t)cm);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (TM) tm_fence_before();
  __syncthreads();
  if (TM) tm_fence_after();
  if (cm > 1) cluster_sync_all();  // every CTA's barriers exist before anyone fills them
  const uint32_t tbase = TM ? *tslot : 0u;
  if (TM && warp < 4) {  // zero rows of both TMEM buffers, one lane quarter per warp
    const uint32_t tz = tbase + (((uint32_t)warp * 32u) << 16) + 4u * (uint32_t)a.kc;
#pragma unroll
    for (int b = 0; b < 2; ++b)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tz + 256u * b),
                   "r"(0u)
                   : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  if (TM) {
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
  }
  // TMEM fill of staged chunk q (smem ring slot) into buffer q & 1 of this warp's lane
  // quarter: the nwarps / 4 warps of a quarter split the kc X rows (LDS.128 of the lane's
  // 16 bytes -> tcgen05.st), then meet at the quarter's named barrier.
  const int tq_id = warp & 3, tq_idx = warp >> 2, tq_n = nwarps >> 2;
  const uint32_t tq_base = TM ? tbase + (((uint32_t)tq_id * 32u) << 16) : 0u;
  auto tm_fill = [&](const uint8_t* st, int q) {
    const uint32_t dst = tq_base + 256u * (uint32_t)(q & 1);
    for (int k = tq_idx; k < a.kc; k += tq_n) {
      const uint4 v = *(const uint4*)(st + k * ROWB + lane * 16);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 4u * k),
                   "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tm_fence_before();
    asm volatile("bar.sync %0, %1;" ::"r"(1 + tq_id), "r"(tq_n * 32) : "memory");
    tm_fence_after();
  };
  // Stage chunk q of the (cluster's) sequence into ring slot q % stages of every CTA of the
  // cluster: one TMA 2-D box of X (kc rows x NT columns, OOB zero-filled), multicast to the
  // cm CTAs when cm > 1, and each CTA's own plan block (1-D bulk copy), all completing on
  // the slot's mbarrier of the receiving CTA.  Called by one whole warp.
  auto refill = [&](int q) {
    const int slot = q % a.stages;
    const int ti = q / nloc, j = q - ti * nloc;
    int pg;
    int64_t n0;
    tile_of(ti, pg, n0);
    const int c = c_begin + j;
    const uint32_t bbytes = (uint32_t)a.blk_bytes;  // fixed block stride (plan.h)
    uint8_t* st = smem + slot * a.stage_bytes;
    const uint32_t fb = full0 + 8 * slot;
    if (a.use_tma && cm > 1) {
      if (lane < cm) {  // lane d serves cluster rank d (its panel's plan block)
        const int64_t bi = (int64_t)(pg * cm + lane) * a.nchunks + c;
        const uint32_t bar_d = map_rank(fb, (uint32_t)lane);
        mbar_arrive_expect_tx_cluster(bar_d, (uint32_t)(a.kc * ROWB) + bbytes);
        bulk_load(map_rank(smem_u32(st + a.x_stage_bytes), (uint32_t)lane), a.blob + bi * a.blk_bytes,
                  bbytes, bar_d);
      }
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_load_2d_mc(smem_u32(st), &tmap, (int)n0, c * a.kc, fb, (uint16_t)((1u << cm) - 1u));
      }
      return;
    }
    const int64_t bi = (int64_t)(persistent ? pg * cm + (int)crank : pg) * a.nchunks + c;
    const int64_t b0 = bi * a.blk_bytes;
    if (a.use_tma) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(fb, (uint32_t)(a.kc * ROWB) + bbytes);
        tma_load_2d(smem_u32(st), &tmap, (int)n0, c * a.kc, fb);
        bulk_load(smem_u32(st + a.x_stage_bytes), a.blob + b0, bbytes, fb);
      }
      return;
    }
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(fb, bbytes);
      bulk_load(smem_u32(st + a.x_stage_bytes), a.blob + b0, bbytes, fb);
    }
    const int k0 = c * a.kc;
    const int kr = min(a.kc, a.K - k0);
    const int cnt = kr * NT;
    for (int idx = lane; idx < cnt; idx += 32) {
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
  };
  // Programmatic dependent launch: everything above (barriers, zero rows, TMEM allocation)
  // overlapped the previous kernel's tail; global X / Y are touched only after it completed.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 0 && crank == 0)
    for (int q = 0; q < min(a.stages, total); ++q) refill(q);

  float acc[R][C];

  // Y[row][n0 + col ...] <- acc (fp16: RN once), group-0 lanes only
  auto store_tile = [&](int64_t n0, const int (&rows)[R]) {
    const int ncol = (int)min((int64_t)NT, a.N - n0);
    if (g != 0 || col >= ncol) return;
    const bool epi = a.bias != nullptr || a.beta != 0.0f || a.relu;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = rows[r];
      if (row < 0) continue;
      uint8_t* yp = a.Y + ((int64_t)row * a.ldy + n0 + col) * S;
      if (a.tcws) {  // + the row's dense-tile contribution (tensor cores), before rounding
        const int wr = a.ws_row[row];
        if (wr >= 0) {
          const float* wp = a.tcws + (int64_t)wr * a.ldws + n0 + col;
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (col + c < ncol) acc[r][c] += wp[c];
        }
      }
      if (epi) {
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (col + c < ncol)
            acc[r][c] = epilogue_one<F16, BF>(acc[r][c], a.bias, row, a.beta, yp + c * S, a.relu);
      }
      if (F16) {
        alignas(16) uint16_t h[C];
#pragma unroll
        for (int c = 0; c < C; ++c) h[c] = to16<BF>(acc[r][c]);
        if (a.vec_y && col + C <= ncol) {
          *(uint4*)yp = *(const uint4*)h;
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (col + c < ncol) ((uint16_t*)yp)[c] = h[c];
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

  // ---------------- Alg. 3 over each staged chunk; the last warp to release a ring slot
  // refills it with chunk q + stages (no producer warp, no blocking wait on an empty barrier)
  int q = 0, slot = 0;
  uint32_t ph = 0;
  int panel = 0;
  int64_t n0 = 0;
  for (int ti = 0; ti < my_tiles; ++ti) {
    tile_of(ti, panel, n0);
    if (persistent) panel = panel * cm + (int)crank;
    int rows[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rows[r] = __ldg(a.row_id + (int64_t)panel * a.Mp + warp * R + r);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[r][c] = 0.0f;
    // lanes past the ragged end of N read lane 0's columns (never stored): their loads
    // merge into lane 0's wavefront, so a tile with n valid lanes costs ceil(n / 8)
    // shared-memory wavefronts per X load instead of 4 (N = 49: 2, N tail of 8: 1)
#if SRT_TAILMERGE
    // (decided per quarter-warp: a 128-bit load is served 8 lanes at a time, and a junk lane
    // of a partly valid quarter reading lane 0's banks would conflict with a valid lane)
    const int xoff = (li & ~7) * C < (int)min((int64_t)NT, a.N - n0) ? li * (C * S) : 0;
#else
    const int xoff = li * (C * S);
#endif
    for (int j = 0; j < nloc; ++j) {
      mbar_wait(full0 + 8 * slot, ph);
      const uint8_t* st = smem + slot * a.stage_bytes;
      if (TM) tm_fill(st, q);
      const uint8_t* xs = st + xoff;
      const uint32_t* shdr = (const uint32_t*)(st + a.x_stage_bytes);
      const uint4* ents = (const uint4*)(st + a.x_stage_bytes + a.hdr_bytes);
      uint32_t h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = shdr[(warp * R + r) * GK + g];
      if (TM) {
        run_rows_tm<F16, R>(acc, h, ents, tq_base + 256u * (uint32_t)(q & 1));
        tm_fence_before();
      } else {
        run_rows<F16, R, BF>(acc, h, ents, xs);
      }
      __syncwarp();
      uint32_t old = 0;
      if (lane == 0)  // release: this warp's reads of the slot precede the count
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old) : "r"(smem_u32(ctr + slot)) : "memory");
      old = __shfl_sync(0xffffffffu, old, 0);
      const bool last_local = (old + 1u) % (uint32_t)nwarps == 0u;
      if (cm == 1) {  // the CTA's last releasing warp refills the slot
        if (last_local && q + a.stages < total) refill(q + a.stages);
      } else if (last_local) {
        // multicast cluster: one remote arrive per CTA on the leader's cluster-empty barrier;
        // the leader's last warp waits for all cm CTAs, then refills the slot cluster-wide
        if (lane == 0) {
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           map_rank(cempty0 + 8 * slot, 0u))
                       : "memory");
        }
        if (crank == 0 && q + a.stages < total) {
          mbar_wait(cempty0 + 8 * slot, (uint32_t)((q / a.stages) & 1));
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
          refill(q + a.stages);
        }
      }

      ++q;
      if (++slot == a.stages) {
        slot = 0;
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
    if (persistent) store_tile(n0, rows);
  }
  if (persistent) {
    if (cm > 1) cluster_sync_all();  // no CTA leaves while peers may still touch its smem
    if (TM) {
      tm_fence_before();
      __syncthreads();
      if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    }
    return;
  }

  const int ncol = (int)min((int64_t)NT, a.N - n0);
  // ---------------- k_split > 1: partial tiles reduced across the cluster through DSMEM,
  // summed in rank order 0, 1, ..., ks-1 for every output (deterministic).
  __syncthreads();  // every consumer is done with the stage buffers that `red` overlays
  float* red = (float*)smem;  // [Mp][NT] fp32
  if (g == 0) {
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
    if (a.tcws && a.ws_row[row] >= 0) {
      const float* wp = a.tcws + (int64_t)a.ws_row[row] * a.ldws + n0 + c4;
      if (c4 + 0 < ncol) v.x += wp[0];
      if (c4 + 1 < ncol) v.y += wp[1];
      if (c4 + 2 < ncol) v.z += wp[2];
      if (c4 + 3 < ncol) v.w += wp[3];
    }
    if (a.bias != nullptr || a.beta != 0.0f || a.relu) {
      if (c4 + 0 < ncol) v.x = epilogue_one<F16, BF>(v.x, a.bias, row, a.beta, yp + 0 * S, a.relu);
      if (c4 + 1 < ncol) v.y = epilogue_one<F16, BF>(v.y, a.bias, row, a.beta, yp + 1 * S, a.relu);
      if (c4 + 2 < ncol) v.z = epilogue_one<F16, BF>(v.z, a.bias, row, a.beta, yp + 2 * S, a.relu);
      if (c4 + 3 < ncol) v.w = epilogue_one<F16, BF>(v.w, a.bias, row, a.beta, yp + 3 * S, a.relu);
    }
    const float vv[4] = {v.x, v.y, v.z, v.w};
    if (F16) {
      alignas(8) uint16_t h[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) h[c] = to16<BF>(vv[c]);
      if (a.vec_y && c4 + 4 <= ncol) {
        *(uint2*)yp = *(const uint2*)h;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c4 + c < ncol) ((uint16_t*)yp)[c] = h[c];
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

// ------------------------------------------------------------------ SpMM, plan in kernel parameters
// The paper keeps the sparse values in the constant cache (baked into the code, P:185, P:379:
// "the value of the sparse matrix A is broadcast across the thread group, it is an ideal use case
// for the constant cache").  plan_source = 1 is that idea for the plan-driven executor: a plan of
// at most kParamPlanBytes travels as a __grid_constant__ kernel parameter (constant bank 0), so
// every warp-uniform plan read is an LDC from the constant cache instead of a shared-memory
// broadcast load, and the ring stages carry X only (no per-chunk bulk copy of plan blocks).
// Same tiles, ring, FMA order and epilogue as spmm_kernel (k_split = 1, no multicast / TMEM):
// results are bitwise equal.
constexpr int kParamPlanBytes = 30 * 1024;
struct ParamPlan {
  uint4 d[kParamPlanBytes / 16];
};

template <int R, bool F16, bool BF = false>
__global__ void __launch_bounds__(512, SRT_MINB) spmm_param_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                   const SpmmArgs a,
                                                                   const __grid_constant__ ParamPlan pp) {
  constexpr int C = F16 ? 8 : 4;
  constexpr int S = F16 ? 2 : 4;
  constexpr int NT = 32 * C;
  constexpr int ROWB = NT * S;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;
  const int np = a.npanels;
  const int ntiles = np * (int)((a.N + NT - 1) / NT);
  const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = my_tiles * a.nchunks;
  const uint32_t full0 = smem_u32(smem + a.bar_off);
  uint32_t* ctr = (uint32_t*)(smem + a.bar_off + 16 * kMaxStages);
  for (int s = 0; s < a.stages; ++s)  // the zero row after the kc X rows of every stage
    for (int i = tid; i < ROWB / 16; i += blockDim.x)
      *(uint4*)(smem + s * a.stage_bytes + a.kc * ROWB + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
  if (tid < kMaxStages) ctr[tid] = 0u;
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(full0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  auto tile_of = [&](int ti, int& panel, int64_t& n0) {
    const int t = (int)blockIdx.x + ti * (int)gridDim.x;
    panel = t % np;
    n0 = (int64_t)(t / np) * NT;
  };
  auto refill = [&](int q) {  // lane 0 of one warp: the X box of chunk q only
    const int slot = q % a.stages;
    const int ti = q / a.nchunks, c = q - ti * a.nchunks;
    int panel;
    int64_t n0;
    tile_of(ti, panel, n0);
    const uint32_t fb = full0 + 8 * slot;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(fb, (uint32_t)(a.kc * ROWB));
    tma_load_2d(smem_u32(smem + slot * a.stage_bytes), &tmap, (int)n0, c * a.kc, fb);
  };
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 0 && lane == 0)
    for (int q = 0; q < min(a.stages, total); ++q) refill(q);
  float acc[R][C];
  int q = 0, slot = 0;
  uint32_t ph = 0;
  for (int ti = 0; ti < my_tiles; ++ti) {
    int panel;
    int64_t n0;
    tile_of(ti, panel, n0);
    int rows[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rows[r] = __ldg(a.row_id + (int64_t)panel * a.Mp + warp * R + r);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[r][c] = 0.0f;
    const int xoff = ((lane & ~7) * C < (int)min((int64_t)NT, a.N - n0)) ? lane * (C * S) : 0;
    for (int j = 0; j < a.nchunks; ++j) {
      mbar_wait(full0 + 8 * slot, ph);
      const uint8_t* xs = smem + slot * a.stage_bytes + xoff;
      // plan block of (panel, chunk j): fixed stride a.blk_bytes in the parameter blob
      const int b16 = (panel * a.nchunks + j) * (a.blk_bytes / 16);
      const uint32_t* shdr = (const uint32_t*)&pp.d[b16];
      const uint4* ents = &pp.d[b16 + a.hdr_bytes / 16];
      uint32_t h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = shdr[warp * R + r];
      run_rows<F16, R, BF>(acc, h, ents, xs);
      __syncwarp();
      uint32_t old = 0;
      if (lane == 0)
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old) : "r"(smem_u32(ctr + slot)) : "memory");
      old = __shfl_sync(0xffffffffu, old, 0);
      if ((old + 1u) % (uint32_t)nwarps == 0u && q + a.stages < total && lane == 0) refill(q + a.stages);
      ++q;
      if (++slot == a.stages) {
        slot = 0;
        ph ^= 1u;
      }
    }
    const int ncol = (int)min((int64_t)NT, a.N - n0);
    const int col = lane * C;
    if (col >= ncol) continue;
    const bool epi = a.bias != nullptr || a.beta != 0.0f || a.relu;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = rows[r];
      if (row < 0) continue;
      uint8_t* yp = a.Y + ((int64_t)row * a.ldy + n0 + col) * S;
      if (epi) {
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (col + c < ncol) acc[r][c] = epilogue_one<F16, BF>(acc[r][c], a.bias, row, a.beta, yp + c * S, a.relu);
      }
      if (F16) {
        alignas(16) uint16_t hv[C];
#pragma unroll
        for (int c = 0; c < C; ++c) hv[c] = to16<BF>(acc[r][c]);
        if (a.vec_y && col + C <= ncol) {
          *(uint4*)yp = *(const uint4*)hv;
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (col + c < ncol) ((uint16_t*)yp)[c] = hv[c];
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
  int32_t rb, ipt, wp, simg, sci, guard, stage_elems, T, bands, cs;
  int32_t npanels, stages;  // TMA-fed kernel
  const uint8_t* bias;  // fused epilogue (plan.h Epilogue)
  float beta;
  int32_t relu;
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
      const float v = epilogue_one<F16>(acc[r][j], a.bias, row, a.beta, a.y + o * S, a.relu);
      if (F16)
        ((__half*)a.y)[o] = __float2half_rn(v);
      else
        ((float*)a.y)[o] = v;
    }
  }
}

// ------------------------------------------------------------------ conv 3x3, vectorised
// Implicit im2col (Sec. 3.6) on the SpMM inner loop.  CTA = (panel of output
// channels, image b, band of rb output rows).  Output positions p = r * wp + c (row r of the
// band, padded column c, pixel x = c - 1); lane owns C consecutive positions (16 bytes).
// The staged input of a chunk of cc channels is the zero-halo band (rows y0-1 .. y0+rb)
// stored three times, copy d shifted by d - 1 elements, so tap (ci, dy, dx) of position p is
// copy_dx[ci][G + p + dy * wp]: every entry is one aligned 128-bit shared load per lane
// (plan entry offset = dx * cs + ci * sci + dy * wp elements).  Halo, guard and junk
// positions are zero / discarded; no bounds checks in the FMA loop.
template <int R, bool F16>
__global__ void __launch_bounds__(512) conv3x3_vec_kernel(const ConvArgs a) {
  constexpr int C = F16 ? 8 : 4;
  constexpr int S = F16 ? 2 : 4;
  constexpr int MAXE = 8;  // staged input elements per thread and chunk (inspector bound)
  using T = typename std::conditional<F16, uint16_t, float>::type;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int panel = blockIdx.x;
  const int b = (int)blockIdx.y / a.bands, band = (int)blockIdx.y % a.bands;
  const int y0 = band * a.rb;
  const int64_t plane = (int64_t)a.H * a.W;
  const int per_ch = (a.rb + 2) * a.W;

  for (int i = tid; i < 2 * a.stage_bytes / 16; i += nthr) ((uint4*)smem)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();

  T v[MAXE];
  auto load = [&](int chunk) {  // global -> registers (coalesced along x)
    const int ci0 = chunk * a.cc, n = min(a.cc, a.c_in - ci0) * per_ch;
#pragma unroll
    for (int j = 0; j < MAXE; ++j) {
      const int e = tid + j * nthr;
      v[j] = T(0);
      if (e < n) {
        const int cl = e / per_ch, r = e - cl * per_ch;
        const int hr = r / a.W, x = r - hr * a.W;
        const int y = y0 - 1 + hr;
        if (y >= 0 && y < a.H)
          v[j] = ((const T*)a.x)[((int64_t)(ci0 + cl) * a.B + b) * plane + (int64_t)y * a.W + x];
      }
    }
  };
  auto store = [&](int buf, int chunk) {  // registers -> the three shifted copies
    T* st = (T*)(smem + buf * a.stage_bytes);
    const int n = min(a.cc, a.c_in - chunk * a.cc) * per_ch;
#pragma unroll
    for (int j = 0; j < MAXE; ++j) {
      const int e = tid + j * nthr;
      if (e < n) {
        const int cl = e / per_ch, r = e - cl * per_ch;
        const int hr = r / a.W, x = r - hr * a.W;
        const int ebase = cl * a.sci + a.guard + hr * a.wp + x + 2;  // halo h + G + 1 - d, d = 0
        st[ebase] = v[j];
        st[a.cs + ebase - 1] = v[j];
        st[2 * a.cs + ebase - 2] = v[j];
      }
    }
  };
  auto plan_copy = [&](int buf, int chunk) {
    uint8_t* st = smem + buf * a.stage_bytes;
    const int64_t bi = (int64_t)panel * a.nchunks + chunk;
    const int64_t blk0 = a.blk_off[bi];
    const int nb = (int)((a.blk_off[bi + 1] - blk0) >> 4);
    const uint32_t dblk = smem_u32(st + a.x_stage_bytes);
    for (int i = tid; i < nb; i += nthr) cp_async16(dblk + 16 * i, a.blob + blk0 + 16 * i, 16);
  };

  float acc[R][C];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0.0f;
  const bool junk = ((lane & ~7) * C) / a.wp >= min(a.rb, a.H - y0);  // whole quarter-warp

  load(0);
  store(0, 0);
  plan_copy(0, 0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int c = 0; c < a.nchunks; ++c) {
    const int buf = c & 1;
    if (c + 1 < a.nchunks) {
      load(c + 1);
      plan_copy(buf ^ 1, c + 1);
      cp_async_commit();
    }
    const uint8_t* st = smem + buf * a.stage_bytes;
    const uint32_t* shdr = (const uint32_t*)(st + a.x_stage_bytes);
    const uint4* ents = (const uint4*)(st + a.x_stage_bytes + a.hdr_bytes);
    uint32_t h[R];
#pragma unroll
    for (int r = 0; r < R; ++r) h[r] = shdr[warp * R + r];
    // lanes whose C positions all lie below the band's last image row read lane 0's address:
    // their loads merge into lane 0's wavefront (no shared-memory bandwidth for junk rows)
    run_rows<F16, R>(acc, h, ents, st + (a.guard + (junk ? 0 : lane * C)) * S);
    if (c + 1 < a.nchunks) {
      store(buf ^ 1, c + 1);
      cp_async_wait<0>();
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = a.row_id[(int64_t)panel * a.Mp + warp * R + r];
    if (row < 0) continue;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int p = lane * C + c;
      const int rr = p / a.wp, x = p - rr * a.wp - 1;
      const int y = y0 + rr;
      if (rr >= a.rb || y >= a.H || x < 0 || x >= a.W) continue;
      const int64_t o = ((int64_t)row * a.B + b) * plane + (int64_t)y * a.W + x;
      const float v = epilogue_one<F16>(acc[r][c], a.bias, row, a.beta, a.y + o * S, a.relu);
      if (F16)
        ((__half*)a.y)[o] = __float2half_rn(v);
      else
        ((float*)a.y)[o] = v;
    }
  }
}

// ------------------------------------------------------------------ conv 3x3, TMA-fed
// The vectorised implicit im2col above with the staging done by the TMA engine instead of
// registers.  TMA rows must be 16-byte aligned (H8) and so must the innermost box coordinate
// (a box starting 1 element off raises an illegal-instruction fault on B200:
// scripts/micro/tma4d.cu), so the shift cannot be done by the TMA engine: a pre-pass
// (pad_conv_input) writes the three shifted, zero-haloed copies to global memory,
// xp3[dx][ci][b][r][c] = x[ci][b][r - 1][c + dx - 2] (zero outside), rows of wp elements.  Copy
// dx of a chunk is then ONE 5-D TMA box {wp, rb + 2, 1, cc, 1} at {0, y0, b, ci0, dx}; rows and
// channels past the end arrive as zeros, so the zero halo of P:215 costs nothing in the loop.  Persistent CTAs walk the tiles (panel fastest, then image band) through an
// mbarrier ring refilled by the last releasing warp (as spmm_kernel); the FMA loop is
// run_rows on the same plan format (offset dx * cs + ci * sci + dy * wp, guard 0).
template <int R, bool F16, bool BF = false>
__global__ void __launch_bounds__(512) conv3x3_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          const ConvArgs a) {
  constexpr int C = F16 ? 8 : 4;
  constexpr int S = F16 ? 2 : 4;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;
  const int np = a.npanels;
  const int64_t ntiles = (int64_t)np * a.B * a.bands;
  const int my_tiles = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
  const int total = my_tiles * a.nchunks;
  const int64_t plane = (int64_t)a.H * a.W;
  const uint32_t full0 = smem_u32(smem + (size_t)a.stages * a.stage_bytes);
  uint32_t* ctr = (uint32_t*)(smem + (size_t)a.stages * a.stage_bytes + 8 * kMaxStages);
  // zero block after the three copies of every stage (target of neutral padding entries)
  for (int s = 0; s < a.stages; ++s)
    for (int i = tid; i < (a.T + 16) * S / 16; i += blockDim.x)
      *(uint4*)(smem + (size_t)s * a.stage_bytes + (size_t)3 * a.cs * S + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
  if (tid < kMaxStages) ctr[tid] = 0u;
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(full0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  auto tile_of = [&](int ti, int& panel, int& b, int& band) {
    const int64_t t = blockIdx.x + (int64_t)ti * gridDim.x;
    panel = (int)(t % np);
    const int64_t ib = t / np;
    b = (int)(ib / a.bands);
    band = (int)(ib % a.bands);
  };
  const uint32_t box_bytes = (uint32_t)(a.cc * a.sci * S);
  auto refill = [&](int q) {  // lane 0 of one warp
    const int slot = q % a.stages;
    const int ti = q / a.nchunks, c = q - ti * a.nchunks;
    int panel, b, band;
    tile_of(ti, panel, b, band);
    const int64_t bi = (int64_t)panel * a.nchunks + c;
    const int64_t blk0 = a.blk_off[bi];
    const uint32_t nb = (uint32_t)(a.blk_off[bi + 1] - blk0);
    uint8_t* st = smem + (size_t)slot * a.stage_bytes;
    const uint32_t fb = full0 + 8 * slot;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(fb, 3 * box_bytes + nb);
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(st + (size_t)dx * a.cs * S)),
          "l"((uint64_t)&tmap), "r"(0), "r"(band * a.rb), "r"(b), "r"(c * a.cc), "r"(dx), "r"(fb)
          : "memory");
    }
    if (nb) bulk_load(smem_u32(st + a.x_stage_bytes), a.blob + blk0, nb, fb);
  };
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 0 && lane == 0)
    for (int q = 0; q < min(a.stages, total); ++q) refill(q);

  float acc[R][C];
  int q = 0, slot = 0;
  uint32_t ph = 0;
  for (int ti = 0; ti < my_tiles; ++ti) {
    int panel, b, band;
    tile_of(ti, panel, b, band);
    const int y0 = band * a.rb;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[r][c] = 0.0f;
    // lanes whose C positions all lie below the band's last image row read lane 0's address
    // (per quarter-warp: a junk lane of a partly valid quarter keeps its own address, which
    // shares the quarter's wavefront, instead of conflicting with a valid lane on lane 0's banks)
    const bool junk = ((lane & ~7) * C) / a.wp >= min(a.rb, a.H - y0);
    const int xoff = junk ? 0 : lane * C * S;
    for (int j = 0; j < a.nchunks; ++j) {
      mbar_wait(full0 + 8 * slot, ph);
      const uint8_t* st = smem + (size_t)slot * a.stage_bytes;
      const uint32_t* shdr = (const uint32_t*)(st + a.x_stage_bytes);
      const uint4* ents = (const uint4*)(st + a.x_stage_bytes + a.hdr_bytes);
      uint32_t h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = shdr[warp * R + r];
      run_rows<F16, R, BF>(acc, h, ents, st + xoff);
      __syncwarp();
      uint32_t old = 0;
      if (lane == 0)
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old) : "r"(smem_u32(ctr + slot)) : "memory");
      old = __shfl_sync(0xffffffffu, old, 0);
      if ((old + 1u) % (uint32_t)nwarps == 0u && q + a.stages < total && lane == 0) refill(q + a.stages);
      ++q;
      if (++slot == a.stages) {
        slot = 0;
        ph ^= 1u;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = a.row_id[(int64_t)panel * a.Mp + warp * R + r];
      if (row < 0) continue;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int p = lane * C + c;
        const int rr = p / a.wp, x = p - rr * a.wp - 1;
        const int y = y0 + rr;
        if (rr >= a.rb || y >= a.H || x < 0 || x >= a.W) continue;
        const int64_t o = ((int64_t)row * a.B + b) * plane + (int64_t)y * a.W + x;
        const float v = epilogue_one<F16, BF>(acc[r][c], a.bias, row, a.beta, a.y + o * S, a.relu);
        if (F16)
          ((uint16_t*)a.y)[o] = to16<BF>(v);
        else
          ((float*)a.y)[o] = v;
      }
    }
  }
}

// ------------------------------------------------------------------ conv 3x3, interleaved
// Implicit im2col (Sec. 3.6) with NO junk positions.  The padded-row layout of
// conv3x3_tma_kernel spends 2 of every wp = 16 positions (and a partial band) on halo columns /
// rows: 23 % of its FMAs at 14 x 14.  Here g images are interleaved row by row ("image group"
// q = images q g .. q g + g - 1): group row r holds row r - 1 of each of the g images side by
// side, pitch P = g W, with one zero row above and below each group (stride Sg = (H + 2) P).
// Output positions n = (q H + y) P + xx (xx = j W + x, image b = q g + j) are all real pixels
// (except the padding images of a batch that is not a multiple of g), a lane owns C = 4
// consecutive ones, and g is the smallest group whose pitch keeps every tap shift (dy - 1) P of
// a lane's 4 positions aligned for one vector load (16 B fp32, 8 B 16-bit; P % 4 == 0; the span
// start is rounded down to 16 bytes and the lanes' offsets follow).  A device pre-pass
// (il_pad_input) writes the three dx-shifted copies in this layout, copy_dx[ci][h] =
// x[ci][b][r - 1][x + dx - 1] (zero outside the image, per position: the zero padding of
// P:215 is resolved there, never in the FMA loop); per chunk of cc channels the TMA engine
// stages, for each copy, the span of h the tile's 128 positions touch (one box of lc <= 256
// elements per channel).  Tap (ci, dy, dx) of a lane's positions is then one aligned load at
// u + dx cs + ci lc + (dy - 1) P (u = the lane's offset in the span), the same mbarrier ring
// and Alg. 3 FMA loop as conv3x3_tma_kernel.  Summation order per output: k ascending, chunks
// ascending -- bitwise equal to the other conv kernels.
struct IlArgs {
  const uint8_t* blob;
  const int64_t* blk_off;
  const int32_t* row_id;
  uint8_t* y;
  int64_t npos;   // image groups x H x P positions
  int64_t plane;  // B H W: output channel stride (CNHW)
  int32_t H, W, P, g, Bt, Sg;
  int32_t cc, nchunks, Mp, npanels, stages, stage_bytes;
  int32_t lc, cs, blk_at, hdr_bytes, bar_off;
  const uint8_t* bias;
  float beta;
  int32_t relu;
  // overlap with the pre-pass (programmatic dependent launch): group q's copies are complete
  // when ready[q] == ready_target (= C_in); nullptr = the pre-pass completed before launch
  const uint32_t* ready;
  uint32_t ready_target;
  int32_t ngroups;
};

// 16-bit entries for 4 positions per lane: unit = 4 x {uint16 xoff (8-byte units), half / bf16 w}
template <bool BF>
__device__ __forceinline__ void unit_h4(float (&acc)[4], const uint4 q, const uint8_t* xs) {
  const uint32_t en[4] = {q.x, q.y, q.z, q.w};
  uint2 x[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) x[e] = *(const uint2*)(xs + ((en[e] & 0xffffu) << 3));
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    fma_h2<BF>(acc[0], acc[1], (uint16_t)(en[e] >> 16), x[e].x);
    fma_h2<BF>(acc[2], acc[3], (uint16_t)(en[e] >> 16), x[e].y);
  }
}
template <bool F16, bool BF, int R>
__device__ __forceinline__ void run_rows_il(float (&acc)[R][4], const uint32_t (&h)[R], const uint4* ents,
                                            const uint8_t* xs) {
  if (!F16) {
    run_rows<false, R>(acc, h, ents, xs);
    return;
  }
  int mn = (int)(h[0] >> 16);
#pragma unroll
  for (int r = 1; r < R; ++r) mn = min(mn, (int)(h[r] >> 16));
  const uint4* pr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) pr[r] = ents + (h[r] & 0xffffu);
#pragma unroll 1
  for (int u = 0; u < mn; ++u) {
    uint4 q[R];
#pragma unroll
    for (int r = 0; r < R; ++r) q[r] = pr[r][u];
#pragma unroll
    for (int r = 0; r < R; ++r) unit_h4<BF>(acc[r], q[r], xs);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int cnt = (int)(h[r] >> 16);
#pragma unroll 1
    for (int u = mn; u < cnt; ++u) unit_h4<BF>(acc[r], pr[r][u], xs);
  }
}

template <int R, bool F16, bool BF = false>
__global__ void __launch_bounds__(512) conv3x3_il_kernel(const __grid_constant__ CUtensorMap tmap,
                                                         const IlArgs a) {
  constexpr int C = 4, NT = 128;  // positions per lane / per tile
  constexpr int S = F16 ? 2 : 4;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;
  const int np = a.npanels;
  const int64_t ntiles = (int64_t)np * ((a.npos + NT - 1) / NT);
  const int my_tiles = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
  const int total = my_tiles * a.nchunks;
  const uint32_t full0 = smem_u32(smem + a.bar_off);
  uint32_t* ctr = (uint32_t*)(smem + a.bar_off + 8 * kMaxStages);
  // the zero block after the three copies of every stage (target of neutral padding entries)
  for (int s = 0; s < a.stages; ++s)
    for (int i = tid; i < a.lc * S / 16; i += blockDim.x)
      *(uint4*)(smem + (size_t)s * a.stage_bytes + (size_t)3 * a.cs * S + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
  if (tid < kMaxStages) ctr[tid] = 0u;
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(full0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const int64_t HP = (int64_t)a.H * a.P;
  auto hcoord = [&](int64_t n) -> int64_t {  // span coordinate of position n
    const int64_t q = n / HP;
    return q * a.Sg + a.P + (n - q * HP);
  };
  auto tile_of = [&](int ti, int& panel, int64_t& n0) {
    const int64_t t = blockIdx.x + (int64_t)ti * gridDim.x;
    panel = (int)(t % np);
    n0 = (t / np) * NT;
  };
  auto refill = [&](int q) {  // lane 0 of one warp
    const int slot = q % a.stages;
    const int ti = q / a.nchunks, c = q - ti * a.nchunks;
    int panel;
    int64_t n0;
    tile_of(ti, panel, n0);
    const int64_t bi = (int64_t)panel * a.nchunks + c;
    const int64_t blk0 = a.blk_off[bi];
    const uint32_t nb = (uint32_t)(a.blk_off[bi + 1] - blk0);
    uint8_t* st = smem + (size_t)slot * a.stage_bytes;
    const uint32_t fb = full0 + 8 * slot;
    const int hb = (int)((hcoord(n0) - a.P) & ~(int64_t)(16 / S - 1));  // 16-byte aligned span start
    if (a.ready) {
      // the span's image groups must be complete in the copies (written by the concurrently
      // running pre-pass): acquire their counters, then order the async-proxy (TMA) reads
      // after them; bounded spin (a missing producer traps instead of hanging the GPU)
      const int q0 = hb / a.Sg, q1 = min(a.ngroups - 1, (hb + a.lc - 1) / a.Sg);
      for (int qq = q0; qq <= q1; ++qq) {
        uint32_t v, spins = 0;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.ready + qq) : "memory");
          if (v >= a.ready_target) break;
          __nanosleep(64);
          if (++spins > (1u << 26)) __trap();
        } while (true);
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(fb, (uint32_t)(3 * a.cc * a.lc * S) + nb);
#pragma unroll
    for (int dx = 0; dx < 3; ++dx)  // copy dx: box {lc, cc, 1} at {hb, ci0, dx}
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(st + (size_t)dx * a.cs * S)),
          "l"((uint64_t)&tmap), "r"(hb), "r"(c * a.cc), "r"(dx), "r"(fb)
          : "memory");
    if (nb) bulk_load(smem_u32(st + a.blk_at), a.blob + blk0, nb, fb);
  };
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // overlapped with the pre-pass: do not wait for its completion (per-group counters instead)
  if (!a.ready) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 0 && lane == 0)
    for (int q = 0; q < min(a.stages, total); ++q) refill(q);

  float acc[R][C];
  int q = 0, slot = 0;
  uint32_t ph = 0;
  for (int ti = 0; ti < my_tiles; ++ti) {
    int panel;
    int64_t n0;
    tile_of(ti, panel, n0);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[r][c] = 0.0f;
    const int64_t hb = (hcoord(n0) - a.P) & ~(int64_t)(16 / S - 1);  // as refill
    const int64_t nl = n0 + lane * C;
    // lanes past the end read the tile's first positions (never stored), per quarter-warp
    const int64_t u = (n0 + (lane & ~7) * C < a.npos ? hcoord(nl) : hcoord(n0)) - hb;
    const intptr_t xoff = (intptr_t)(u - a.P) * S;  // + dx cs + ci lc + dy P (plan entry)
    for (int j = 0; j < a.nchunks; ++j) {
      mbar_wait(full0 + 8 * slot, ph);
      const uint8_t* st = smem + (size_t)slot * a.stage_bytes;
      const uint32_t* shdr = (const uint32_t*)(st + a.blk_at);
      const uint4* ents = (const uint4*)(st + a.blk_at + a.hdr_bytes);
      uint32_t h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = shdr[warp * R + r];
      run_rows_il<F16, BF, R>(acc, h, ents, st + xoff);
      __syncwarp();
      uint32_t old = 0;
      if (lane == 0)
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old) : "r"(smem_u32(ctr + slot)) : "memory");
      old = __shfl_sync(0xffffffffu, old, 0);
      if ((old + 1u) % (uint32_t)nwarps == 0u && q + a.stages < total && lane == 0) refill(q + a.stages);
      ++q;
      if (++slot == a.stages) {
        slot = 0;
        ph ^= 1u;
      }
    }
    // epilogue: position n -> image b = q g + xx / W, pixel (y, xx % W) of the CNHW output
    int64_t oidx[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int64_t n = nl + c;
      const int64_t gq = n / HP;
      const int rem = (int)(n - gq * HP), yy = rem / a.P, xx = rem - yy * a.P;
      const int jj = xx / a.W;
      const int64_t b = gq * a.g + jj;
      oidx[c] = (n < a.npos && b < a.Bt) ? (b * a.H + yy) * a.W + (xx - jj * a.W) : -1;
    }
    const bool epi = a.bias != nullptr || a.beta != 0.0f || a.relu;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = a.row_id[(int64_t)panel * a.Mp + warp * R + r];
      if (row < 0) continue;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (oidx[c] < 0) continue;
        uint8_t* yp = a.y + ((int64_t)row * a.plane + oidx[c]) * S;
        float v = acc[r][c];
        if (epi) v = epilogue_one<F16, BF>(v, a.bias, row, a.beta, yp, a.relu);
        if (F16)
          *(uint16_t*)yp = to16<BF>(v);
        else
          *(float*)yp = v;
      }
    }
  }
}

// a / b for 0 <= a < 2^22 and a runtime divisor b with its reciprocal: one float multiply and
// a +-1 correction instead of an integer division (pre-pass index math is instruction bound)
__device__ __forceinline__ int div_rcp(int a, int b, float rb) {
  int q = (int)((float)a * rb);
  if (q * b > a) --q;
  else if ((q + 1) * b <= a) ++q;
  return q;
}

// fp32 -> nearest TF32 value (round to nearest even on the 13 dropped mantissa bits), in an fp32
// container (finite inputs; 3xTF32 operand splits)
__device__ __forceinline__ float tf32_rn_dev(float f) {
  uint32_t u = __float_as_uint(f);
  u += 0xfffu + ((u >> 13) & 1u);
  return __uint_as_float(u & 0xffffe000u);
}

// Shared-memory staging of `count` contiguous elements (16-byte vectors when the source and the
// count allow it, 4 in flight per thread), zero-filled past `valid`.
template <typename T>
__device__ __forceinline__ void stage_contig(T* dst, const T* __restrict__ src, int count, int valid) {
  constexpr int V = 16 / sizeof(T);
  if (((uintptr_t)src % 16) == 0 && (count % V) == 0 && (valid % V) == 0) {
    const int nv = count / V, vv = valid / V;
    for (int i = threadIdx.x; i < nv; i += 4 * blockDim.x) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int iv = i + u * blockDim.x;
        v[u] = iv < vv ? __ldg((const uint4*)src + iv) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * blockDim.x < nv) ((uint4*)dst)[i + u * blockDim.x] = v[u];
    }
  } else {
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = i < valid ? __ldg(src + i) : T(0);
  }
}

// Image-group interleaved, zero-haloed, dx-shifted copies for conv3x3_il_kernel:
// xp[dx][ci][q Sg + r P + j W + x] = x[ci][q g + j][r - 1][x + dx - 1] (zero outside the
// image, for the halo rows r = 0, H + 1 and for padding images b >= B).  Pure data movement:
// a CTA stages `pp` (channel, group) blocks of g contiguous input planes in shared memory
// (16-byte loads), then writes every (block, copy) output of Sg contiguous elements with
// 16-byte stores, thread t at elements 4 t .. 4 t + 3 (P % 4 == 0: a vector never leaves its row).
template <typename T>
__global__ void __launch_bounds__(256) il_pad_input(const T* __restrict__ x, T* __restrict__ xp, int cin, int B,
                                                    int H, int W, int g, int ngroups, int Sg, int pp,
                                                    uint32_t* ready, T* __restrict__ xlo = nullptr) {
  extern __shared__ __align__(16) uint8_t il_smem[];
  T* sp = (T*)il_smem;  // [pp][g][H][W]
  const int HW = H * W, P = g * W, blk = g * HW;
  const int nblk = cin * ngroups;
  const int64_t span = (int64_t)ngroups * Sg;
  // overlap mode: the conv kernel may start now (it waits on the per-group counters, not on
  // this grid).  Sequential mode: no early trigger -- a conv CTA launched early would sit on
  // an SM (in griddepcontrol.wait) and take the resources this pre-pass needs (measured 70 ->
  // 89 us).
  if (ready) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // block order: overlap mode group-major (bb = q cin + ci: the first image groups complete
  // first, in the order the conv kernel's tiles consume them); sequential mode channel-major
  // (bb = ci ngroups + q: a CTA's consecutive blocks are one contiguous run of the input)
  const float rcin = 1.0f / cin, rng = 1.0f / ngroups, rP = 1.0f / P, rW = 1.0f / W;
  auto decode = [&](int bb, int& q, int& ci) {
    if (ready) {
      q = div_rcp(bb, cin, rcin);
      ci = bb - q * cin;
    } else {
      ci = div_rcp(bb, ngroups, rng);
      q = bb - ci * ngroups;
    }
  };
  // vectors of V elements never leave their row: fp32 V = 4 (16 B); 16-bit V = 8 (16 B) when
  // P % 8 == 0, else V = 4 (8-byte stores)
  auto write_copies = [&](int b0, int nb, auto vtag) {
    constexpr int V = decltype(vtag)::value;
    const int nvv = Sg / V;
    const float rnv = 1.0f / nvv;
    for (int i = threadIdx.x; i < 3 * nb * nvv; i += blockDim.x) {
      const int t = div_rcp(i, nvv, rnv), e0 = (i - t * nvv) * V;
      const int k = div_rcp(t, 3, 1.0f / 3.0f), dx = t - 3 * k;
      int q, ci;
      decode(b0 + k, q, ci);
      const int r = div_rcp(e0, P, rP), xx = e0 - r * P;
      int j = div_rcp(xx, W, rW), xw = xx - j * W;
      const T* sb = sp + (size_t)k * blk + (size_t)(r - 1) * W;
      alignas(16) T v[V];
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int xs = xw + dx - 1;
        v[c] = (r >= 1 && r <= H && xs >= 0 && xs < W) ? sb[j * HW + xs] : T(0);
        if (++xw == W) xw = 0, ++j;
      }
      T* dst = xp + ((int64_t)dx * cin + ci) * span + (int64_t)q * Sg + e0;
      if (V * sizeof(T) == 16)
        *(uint4*)dst = *(const uint4*)v;
      else
        *(uint2*)dst = *(const uint2*)v;
    }
  };
  const bool v8 = sizeof(T) == 2 && P % 8 == 0;
  for (int b0 = blockIdx.x * pp; b0 < nblk; b0 += gridDim.x * pp) {
    const int nb = min(pp, nblk - b0);
    for (int k = 0; k < nb;) {  // block (q, ci): g contiguous planes (zero past the batch)
      int q, ci;
      decode(b0 + k, q, ci);
      // sequential mode: the run of this channel's blocks is contiguous in x
      const int run = ready ? 1 : min(nb - k, ngroups - q);
      const int valid = max(0, min(run * g, B - q * g)) * HW;
      stage_contig<T>(sp + (size_t)k * blk, x + ((int64_t)ci * B + (int64_t)q * g) * HW, run * blk, valid);
      k += run;
    }
    __syncthreads();
    if (v8) {
      write_copies(b0, nb, std::integral_constant<int, 8>{});
    } else {  // (the round-2 fp32 loop, kept verbatim: the generic form measured 19 us slower)
      const int nv = Sg / 4;
      const float rnv = 1.0f / nv;
      for (int i = threadIdx.x; i < 3 * nb * nv; i += blockDim.x) {
        const int t = div_rcp(i, nv, rnv), e0 = (i - t * nv) * 4;
        const int k = div_rcp(t, 3, 1.0f / 3.0f), dx = t - 3 * k;
          int q, ci;
        decode(b0 + k, q, ci);
        const int r = div_rcp(e0, P, rP), xx = e0 - r * P;
        int j = div_rcp(xx, W, rW), xw = xx - j * W;
        const T* sb = sp + (size_t)k * blk + (size_t)(r - 1) * W;
        alignas(16) T v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int xs = xw + dx - 1;
          v[c] = (r >= 1 && r <= H && xs >= 0 && xs < W) ? sb[j * HW + xs] : T(0);
          if (++xw == W) xw = 0, ++j;
        }
        const int64_t di = ((int64_t)dx * cin + ci) * span + (int64_t)q * Sg + e0;
        if constexpr (sizeof(T) == 4) {
          if (xlo) {  // 3xTF32 operand split (conv on the tcgen05 block executor): v = hi + lo
            float h[4], l[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              h[c] = tf32_rn_dev(v[c]);
              l[c] = isfinite(h[c]) ? tf32_rn_dev(v[c] - h[c]) : 0.0f;
            }
            *(float4*)(xp + di) = make_float4(h[0], h[1], h[2], h[3]);
            *(float4*)(xlo + di) = make_float4(l[0], l[1], l[2], l[3]);
          } else {
            *(uint4*)(xp + di) = *(const uint4*)v;
          }
        } else {
          *(uint2*)(xp + di) = *(const uint2*)v;
        }
      }
    }
    if (ready) __threadfence();  // this thread's copies visible at device scope
    __syncthreads();
    if (ready && threadIdx.x < nb) {  // publish: block (q, ci) of every copy is written
      const int bb = b0 + threadIdx.x, q = bb / cin;  // (overlap mode: group-major order)
      __threadfence();
      atomicAdd(ready + q, 1u);
    }
  }
}

// x[C_in][B][H][W] -> xp3[3][C_in][B][H + 1][wp]: xp3[dx][..][r][c] = x[..][r - 1][c + dx - 2],
// zero outside the image (the layout conv3x3_tma_kernel reads through TMA).  Pure data movement:
// a CTA stages `kPadPlanes` whole input planes in shared memory (16-byte loads when aligned),
// then writes every (plane, copy) output of (H + 1) wp contiguous elements with 16-byte stores
// (wp % V == 0: a vector never leaves its row).  (Round 1 used one thread per padded row with a
// 72-element register row: scalar loads strided by a row per thread.)
template <typename T>
__global__ void __launch_bounds__(256) pad_conv_input(const T* __restrict__ x, T* __restrict__ xp, int64_t planes,
                                                      int H, int W, int wp, int kPadPlanes) {
  constexpr int V = 16 / sizeof(T);
  extern __shared__ __align__(16) uint8_t pad_smem[];
  T* sp = (T*)pad_smem;  // [kPadPlanes][H][W]
  const int HW = H * W, nv = (H + 1) * wp / V;
  const int64_t rows = planes * (H + 1);
  for (int64_t p0 = (int64_t)blockIdx.x * kPadPlanes; p0 < planes; p0 += (int64_t)gridDim.x * kPadPlanes) {
    const int np = (int)min((int64_t)kPadPlanes, planes - p0);
    stage_contig<T>(sp, x + p0 * HW, np * HW, np * HW);
    __syncthreads();
    const float rnv = 1.0f / nv, rwp = 1.0f / wp;
    for (int i = threadIdx.x; i < 3 * np * nv; i += blockDim.x) {
      const int t = div_rcp(i, nv, rnv), e0 = (i - t * nv) * V;
      const int k = div_rcp(t, 3, 1.0f / 3.0f), dx = t - 3 * k;
      const int r = div_rcp(e0, wp, rwp), c0 = e0 - r * wp, y = r - 1;
      const T* sb = sp + (size_t)k * HW + (size_t)y * W;
      alignas(16) T v[V];
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int xx = c0 + c + dx - 2;
        v[c] = (y >= 0 && xx >= 0 && xx < W) ? sb[xx] : T(0);
      }
      *(uint4*)(xp + ((int64_t)dx * rows + (p0 + k) * (H + 1)) * wp + e0) = *(const uint4*)v;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ tensor-core sub-blocks
// the dense-enough 16 x 16 tiles of W (plan.h tc_*) as a dense contraction on
// the tensor cores.  CTA = (row block, 128 columns of N), 4 warps x 32 columns; per tile of
// the row block (k-block ascending): X rows 16 cb .. 16 cb + 15 of the CTA's columns are
// staged in shared memory (272-byte row pitch: conflict-free ldmatrix), each warp loads its
// A fragment (16 bytes per lane, pre-packed by the inspector) and issues 4 mma.m16n8k16
// (fp16 x fp16, fp32 accumulate) with B fragments from ldmatrix.x2.trans.  The fp32 result
// overwrites the workspace rows of the row block; the CUDA-core kernel adds them to its
// accumulators before the single rounding (sparse part + dense part, then epilogue).
struct TcArgs {
  const uint16_t* A;
  const int32_t *rb, *tile_begin, *cb;
  const uint8_t* X;
  float* ws;
  int64_t ldx, ldws, N;
  int32_t K, vec_x;
};

// COLS = columns of N per CTA (4 warps x COLS / 4): 512 for large N, 128 for small N
template <int COLS>
__global__ void __launch_bounds__(128) spmm_tc_kernel(const TcArgs a) {
  constexpr int kTcCols = COLS, JW = COLS / 32;  // n8 tiles per warp
  constexpr int kTcPitch = kTcCols + 8;  // smem row pitch in halves (conflict-free ldmatrix)
  extern __shared__ __align__(128) uint16_t xs[];  // [2][16][kTcPitch]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i = blockIdx.x;
  const int64_t n0 = (int64_t)blockIdx.y * kTcCols;
  float acc[JW][4];
#pragma unroll
  for (int j = 0; j < JW; ++j)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[j][c] = 0.0f;
  const int t0 = a.tile_begin[i], t1 = a.tile_begin[i + 1];
  // stage X[k0 .. k0 + 16][n0 .. n0 + COLS) into buffer `buf`: 16 rows x COLS / 8 chunks
  auto stage = [&](int t, int buf) {
    const int k0 = a.cb[t] * 16;
    uint16_t* dst = xs + buf * 16 * kTcPitch;
    for (int q = tid; q < 16 * (kTcCols / 8); q += 128) {
      const int r = q / (kTcCols / 8), ch = q % (kTcCols / 8);
      const int64_t k = k0 + r, n = n0 + ch * 8;
      uint16_t* d = dst + r * kTcPitch + ch * 8;
      const uint16_t* src = (const uint16_t*)a.X + k * a.ldx + n;
      if (k < a.K && a.vec_x && n + 8 <= a.N) {
        cp_async16(smem_u32(d), src, 16);
      } else {
        uint16_t h[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) h[e] = (k < a.K && n + e < a.N) ? src[e] : (uint16_t)0;
        *(uint4*)d = *(const uint4*)h;
      }
    }
    cp_async_commit();
  };
  if (t0 < t1) stage(t0, 0);
  for (int t = t0; t < t1; ++t) {
    const int buf = (t - t0) & 1;
    if (t + 1 < t1) {
      stage(t + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint4 af = *((const uint4*)a.A + (int64_t)t * 32 + lane);
    const uint16_t* xb = xs + buf * 16 * kTcPitch;
#pragma unroll
    for (int j = 0; j < JW; ++j) {
      // lanes 0-7: K rows 0-7, lanes 8-15: rows 8-15, at column (COLS / 4) warp + 8 j
      const uint32_t addr = smem_u32(xb + (lane & 15) * kTcPitch + warp * (COLS / 4) + j * 8);
      uint32_t b0, b1;
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                   : "=r"(b0), "=r"(b1)
                   : "r"(addr));
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
          "{%8, %9}, {%0, %1, %2, %3};"
          : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
          : "r"(af.x), "r"(af.y), "r"(af.z), "r"(af.w), "r"(b0), "r"(b1));
    }
    __syncthreads();
  }
  // D fragment: lane (g, t): rows g and g + 8, columns 2 t, 2 t + 1 of each 16 x 8 tile
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int j = 0; j < JW; ++j) {
    const int64_t n = n0 + warp * (COLS / 4) + j * 8 + 2 * tq;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float* wp = a.ws + (int64_t)(i * 16 + g + 8 * h) * a.ldws + n;
      if (n + 1 < a.N) {
        *(float2*)wp = make_float2(acc[j][2 * h], acc[j][2 * h + 1]);
      } else if (n < a.N) {
        wp[0] = acc[j][2 * h];
      }
    }
  }
}

// ------------------------------------------------------------------ dispatch
using SpmmFn = void (*)(const __grid_constant__ CUtensorMap, const SpmmArgs);
using ConvFn = void (*)(const ConvArgs);

template <bool F16, bool BF = false>
static SpmmFn pick_spmm(int R, int GK, bool tm) {
  if (BF) {  // bf16: CUDA-core kernel, shared-memory X source only
    if (tm) return nullptr;
#define SRT_B(RR, GG) \
  if (R == RR && GK == GG) return spmm_kernel<RR, GG, true, false, true>;
#define SRT_BR(RR) SRT_B(RR, 1) SRT_B(RR, 2) SRT_B(RR, 4) SRT_B(RR, 8)
    SRT_BR(1) SRT_BR(2) SRT_BR(4) SRT_BR(8)
#undef SRT_BR
#undef SRT_B
    return nullptr;
  }
  if (tm) {  // TMEM X source: split_k = 1 only
    if (GK != 1) return nullptr;
    if (R == 1) return spmm_kernel<1, 1, F16, true>;
    if (R == 2) return spmm_kernel<2, 1, F16, true>;
    if (R == 4) return spmm_kernel<4, 1, F16, true>;
    if (R == 8) return spmm_kernel<8, 1, F16, true>;
    return nullptr;
  }
#define SRT_S(RR, GG) \
  if (R == RR && GK == GG) return spmm_kernel<RR, GG, F16, false>;
#define SRT_SR(RR) SRT_S(RR, 1) SRT_S(RR, 2) SRT_S(RR, 4) SRT_S(RR, 8)
  SRT_SR(1) SRT_SR(2) SRT_SR(4) SRT_SR(8)
  if constexpr (!F16) { SRT_SR(16) }
#undef SRT_SR
#undef SRT_S
  return nullptr;
}

template <bool F16>
static ConvFn pick_conv_vec(int R) {
  if (R == 1) return conv3x3_vec_kernel<1, F16>;
  if (R == 2) return conv3x3_vec_kernel<2, F16>;
  if (R == 4) return conv3x3_vec_kernel<4, F16>;
  if (R == 8) return conv3x3_vec_kernel<8, F16>;
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

static PFN_cuTensorMapEncodeIm2col_v12000 tensor_map_encoder_im2col() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeIm2col_v12000)p;
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
  if (e != cudaSuccess) {
    cudaFreeAsync(*Xp, (cudaStream_t)stream);
    *Xp = nullptr;
    return cuda_fail(e, "repack launch", err);
  }
  return SPARSE_OK;
}

// Tiled transpose out[c][r] = in[r][c] (rows x cols, leading dims in elements), 32 x 32 tiles
// through shared memory (padded: conflict-free), element size 2 or 4 bytes.  Pure data movement
// for the token-major entry point sparse_linear.
template <typename T>
__global__ void transpose_2d(const T* __restrict__ in, int64_t ldi, T* __restrict__ out, int64_t ldo,
                             int64_t rows, int64_t cols) {
  __shared__ T tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * ldi + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * ldo + r] = tile[threadIdx.x][i];
  }
}

// CNHW -> NHWC for the im2col conv on the tcgen05 block executor: out[p][c] = in[c][p] (P = B H W
// pixels).  A CTA moves 32 channels x 128 pixels through shared memory: 16-byte loads along the
// pixels of each channel row, 16-byte stores along the 32 channels of each pixel (128-byte
// segments).  SPLIT (fp32 plans, 3xTF32): out = TF32 RN of x, out_lo = TF32 RN of the remainder
// (0 for non-finite x).  Pure data movement (+ the operand split).
template <typename T, bool SPLIT>
__global__ void __launch_bounds__(256) nhwc_pack(const T* __restrict__ in, T* __restrict__ out, T* __restrict__ out_lo,
                                                 int64_t C, int64_t P) {
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
  __shared__ T tile[32][128 + V];
  const int64_t p0 = (int64_t)blockIdx.x * 128, c0 = (int64_t)blockIdx.y * 32;
  const bool vec_in = (P % V) == 0 && p0 + 128 <= P && ((uintptr_t)in % 16) == 0;
  // loads: warp w takes channel rows w, w + 8, ...; lane l the pixels l V .. l V + V - 1
  for (int i = threadIdx.x >> 5; i < 32; i += 8) {
    const int64_t c = c0 + i;
    for (int e0 = (threadIdx.x & 31) * V; e0 < 128; e0 += 32 * V) {
      if (vec_in && c < C) {
        const uint4 v = __ldg((const uint4*)(in + c * P + p0 + e0));
        const T* t = (const T*)&v;
#pragma unroll
        for (int k = 0; k < V; ++k) tile[i][e0 + k] = t[k];
      } else {
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const int64_t px = p0 + e0 + k;
          tile[i][e0 + k] = (c < C && px < P) ? in[c * P + px] : T(0);
        }
      }
    }
  }
  __syncthreads();
  // stores: 32 / V threads per pixel (one 16-byte vector of channels each)
  constexpr int TPP = 32 / V;
  const bool vec_out = (C % V) == 0 && c0 + 32 <= C;
  for (int j = threadIdx.x / TPP; j < 128; j += 256 / TPP) {
    const int64_t px = p0 + j;
    if (px >= P) break;
    const int cv = (threadIdx.x % TPP) * V;
    alignas(16) T h[V], l[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const T v = tile[cv + k][j];
      if constexpr (SPLIT) {
        h[k] = tf32_rn_dev(v);
        l[k] = isfinite(h[k]) ? tf32_rn_dev(v - h[k]) : 0.0f;
      } else {
        h[k] = v;
      }
    }
    if (vec_out) {
      *(uint4*)(out + px * C + c0 + cv) = *(const uint4*)h;
      if constexpr (SPLIT) *(uint4*)(out_lo + px * C + c0 + cv) = *(const uint4*)l;
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if (c0 + cv + k >= C) break;
        out[px * C + c0 + cv + k] = h[k];
        if constexpr (SPLIT) out_lo[px * C + c0 + cv + k] = l[k];
      }
    }
  }
}

int launch_transpose(int device, int S, const void* in, int64_t ldi, void* out, int64_t ldo, int64_t rows,
                     int64_t cols, void* stream, std::string& err) {
  DeviceGuard dg(device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  for (int64_t rb = 0; rb < rows; rb += 32 * 65535) {  // grid.y limit
    const int64_t rr = std::min<int64_t>(rows - rb, 32 * 65535);
    const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rr + 31) / 32)), block(32, 8);
    if (S == 2)
      transpose_2d<uint16_t><<<grid, block, 0, (cudaStream_t)stream>>>((const uint16_t*)in + rb * ldi, ldi,
                                                                       (uint16_t*)out + rb, ldo, rr, cols);
    else
      transpose_2d<float><<<grid, block, 0, (cudaStream_t)stream>>>((const float*)in + rb * ldi, ldi,
                                                                    (float*)out + rb, ldo, rr, cols);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "transpose launch", err);
  return SPARSE_OK;
}

// Sampled pixels of a strided 1x1 convolution: xs[k][(b ho + oy) wo + ox] = x[k][b][oy s][ox s].
// Pure data movement (one thread per output element, consecutive threads -> consecutive ox).
template <typename T>
__global__ void stride_gather(const T* __restrict__ x, T* __restrict__ xs, int64_t planes, int h, int w, int s,
                              int ho, int wo) {
  const int64_t per = (int64_t)ho * wo, tot = planes * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pl = i / per;
    const int r = (int)(i - pl * per), oy = r / wo, ox = r - oy * wo;
    xs[i] = __ldg(x + (pl * h + (int64_t)oy * s) * w + (int64_t)ox * s);
  }
}

int launch_stride_gather(int device, int S, const void* x, int64_t K, int64_t B, int h, int w, int s, void* xs,
                         void* stream, std::string& err) {
  DeviceGuard dg(device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  const int ho = (h + s - 1) / s, wo = (w + s - 1) / s;
  const int64_t tot = K * B * ho * wo;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 148 * 32));
  if (S == 2)
    stride_gather<uint16_t><<<grid, 256, 0, (cudaStream_t)stream>>>((const uint16_t*)x, (uint16_t*)xs, K * B, h, w,
                                                                    s, ho, wo);
  else
    stride_gather<float><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)x, (float*)xs, K * B, h, w, s, ho, wo);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "stride gather launch", err);
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
  {
    // The executors take stream-ordered scratch (X repack, conv input copies, tensor-core
    // workspace) with cudaMallocAsync.  With the default release threshold (0) the device pool
    // hands its memory back to the driver at every synchronisation, so the next call pays a
    // real allocation; keep it instead (the pool then grows to the largest scratch used).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, p.device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  const size_t nrow = p.row_id.size() * 4, noff = p.blk_off.size() * 8, nblob = p.blob.size();
  const size_t o_off = 0, o_row = (noff + 255) & ~size_t(255),
               o_blob = (o_row + nrow + 255) & ~size_t(255);
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  const size_t o_tca = al(o_blob + nblob), o_tcrb = al(o_tca + p.tc_a.size() * 2),
               o_tctb = al(o_tcrb + p.tc_rb.size() * 4), o_tccb = al(o_tctb + p.tc_tile_begin.size() * 4),
               o_wsr = al(o_tccb + p.tc_cb.size() * 4);
  const size_t o_tcpo = al(o_wsr + p.ws_row.size() * 4), o_tcps = al(o_tcpo + p.tcp_step_off.size() * 4);
  const size_t total = o_tcps + p.tcp_steps.size();
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
      (e = cudaMemcpy(b + o_blob, p.blob.data(), nblob, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (p.tc_ntiles > 0 &&
       ((e = cudaMemcpy(b + o_tca, p.tc_a.data(), p.tc_a.size() * 2, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(b + o_tcrb, p.tc_rb.data(), p.tc_rb.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(b + o_tctb, p.tc_tile_begin.data(), p.tc_tile_begin.size() * 4,
                        cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(b + o_tccb, p.tc_cb.data(), p.tc_cb.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(b + o_wsr, p.ws_row.data(), p.ws_row.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess))) {
    cudaFree(mem);
    return cuda_fail(e, "cudaMemcpy(plan)", err);
  }
  if ((p.executor == 3 || p.executor == 4) &&
      ((e = cudaMemcpy(b + o_tcpo, p.tcp_step_off.data(), p.tcp_step_off.size() * 4, cudaMemcpyHostToDevice)) !=
           cudaSuccess ||
       (e = cudaMemcpy(b + o_tcps, p.tcp_steps.data(), p.tcp_steps.size(), cudaMemcpyHostToDevice)) != cudaSuccess)) {
    cudaFree(mem);
    return cuda_fail(e, "cudaMemcpy(tensor-core panels)", err);
  }
  // A cudaMemcpy from pageable memory may return before the DMA has landed; it is ordered
  // only with the legacy default stream.  Executors may run on any (non-blocking) stream,
  // so the plan must be complete in device memory when create returns.
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
    cudaFree(mem);
    return cuda_fail(e, "cudaDeviceSynchronize(plan upload)", err);
  }
  p.d_mem = mem;
  p.d_blk_off = (const int64_t*)(b + o_off);
  p.d_row_id = (const int32_t*)(b + o_row);
  p.d_blob = b + o_blob;
  if (p.tc_ntiles > 0) {
    p.d_tc_a = (const uint16_t*)(b + o_tca);
    p.d_tc_rb = (const int32_t*)(b + o_tcrb);
    p.d_tc_tile_begin = (const int32_t*)(b + o_tctb);
    p.d_tc_cb = (const int32_t*)(b + o_tccb);
    p.d_ws_row = (const int32_t*)(b + o_wsr);
  }
  if (p.executor == 3 || p.executor == 4) {
    p.d_tcp_step_off = (const int32_t*)(b + o_tcpo);
    p.d_tcp_steps = b + o_tcps;
  }
  return SPARSE_OK;
}

void free_plan_device(Plan& p) {
  if (p.d_mem) {
    DeviceGuard dg(p.device);
    cudaFree(p.d_mem);
    p.d_mem = nullptr;
  }
}

// ------------------------------------------------------------------ condensed-panel tensor cores
// SURVEY NEXT #1 (executor = 3, fp16 SpMM): per 16-row panel and 64-row K chunk, the union of
// the panel's nonzero columns is multiplied as a dense block on the tensor cores,
// mma.sync m16n8k16 (fp16 x fp16, fp32 accumulate): A = W[16 rows x 16 union slots] (packed
// by the inspector in fragment order), B = the union's X rows, GATHERED by ldmatrix.x4.trans
// with one row address per lane from the staged chunk.  The chunk is two 128-byte-swizzled
// TMA boxes (64 K rows x 64 columns each), so the 8 rows of one ldmatrix matrix, chosen
// with distinct k mod 8 by the inspector, hit distinct banks.  CTA = kTcpPanels warps (8: two
// CTAs per SM; measured faster than 16 warps in one CTA) = 8 panels x 128 columns; every warp
// keeps 16 rows x 128 columns of fp32 accumulators; the chunk's A fragments and slot rows
// arrive with the X boxes (bulk copy); mbarrier ring refilled by the last releasing warp.
struct TcpArgs {
  const int32_t* step_off;
  const uint8_t* steps;
  uint8_t* Y;
  int64_t ldy, N;
  int32_t M, nchunks, npanels, stages, stage_bytes;
  int32_t cy;  // CTAs per cluster along N sharing (multicasting) the panels' A steps
  const uint8_t* bias;
  float beta;
  int32_t relu;
};

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
template <bool BF = false>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  if (BF)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
                 "{%8, %9}, {%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                 "{%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// NB = 64-column boxes per CTA (N tile = 64 NB): 2 for large N (A fragments reused over 16
// n8 tiles), 1 below (twice the CTAs; measured 1.4x faster at N = 1568 / 392).  Loading the
// next step's B fragments ahead of this step's mma.sync (software pipelining) was measured
// 1.2-1.6x slower (register pressure at 2 CTAs per SM).
#ifndef SRT_TCP_CY
#define SRT_TCP_CY 1
#endif
template <int NB, bool BF = false>
__global__ void __launch_bounds__(32 * kTcpPanels, kTcpPanels >= 16 ? 1 : 2) spmm_tcp_kernel(const __grid_constant__ CUtensorMap tmap, const TcpArgs a) {
  constexpr int NTT = 8 * NB;       // n8 tiles per warp
  constexpr int XST = NB * kTcpKc * 128;  // X part of a stage
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;
  const int q = blockIdx.x * nwarps + warp;  // this warp's panel
  const int64_t n0 = (int64_t)blockIdx.y * (64 * NB);
  uint8_t* sbase = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);  // 128B swizzle: 1 KB aligned
  const uint32_t full0 = smem_u32(sbase + (size_t)a.stages * a.stage_bytes);
  uint32_t* ctr = (uint32_t*)(sbase + (size_t)a.stages * a.stage_bytes + 8 * kMaxStages);
  const int G = blockIdx.x;
  const int32_t* offs = a.step_off + (int64_t)G * a.nchunks * (kTcpPanels + 1);
  // cy > 1 (-DSRT_TCP_CY=2/4, exact-tested): the cy CTAs of a cluster (consecutive N tiles,
  // same panel group) receive every chunk's A steps through ONE multicast bulk copy issued by
  // rank 0, which refills a slot once all cy CTAs released it (cluster-empty barrier in rank 0,
  // one remote arrive per CTA).  Cuts the A-step L2 traffic by cy but measured 1.4-1.7x slower
  // (the cluster-wide release lockstep), as the X multicast of spmm_kernel; off by default.
  constexpr int cy = SRT_TCP_CY;  // compile-time: the multicast code vanishes for cy == 1
  const uint32_t crank = cy > 1 ? cluster_rank() : 0u;
  const uint32_t cempty0 = full0 + 8 * kMaxStages + 64;  // after ctr[8]
  if (tid < kMaxStages) ctr[tid] = 0u;
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(full0 + 8 * s, 1);
    for (int s = 0; cy > 1 && s < a.stages; ++s) mbar_init(cempty0 + 8 * s, (uint32_t)cy);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (cy > 1) cluster_sync_all();  // every CTA's barriers exist before multicasts arrive
  auto nbytes = [&](int c) -> uint32_t {
    const int o0 = __ldg(offs + c * (kTcpPanels + 1)), o1 = __ldg(offs + c * (kTcpPanels + 1) + kTcpPanels);
    return (uint32_t)(o1 - o0);  // byte offsets
  };
  auto load_a = [&](int c) {  // the group's steps of chunk c -> slot (multicast when cy > 1)
    const int slot = c % a.stages;
    const uint32_t nb = nbytes(c);
    if (!nb) return;
    const int o0 = __ldg(offs + c * (kTcpPanels + 1));
    const uint32_t dst = smem_u32(sbase + (size_t)slot * a.stage_bytes + XST), fb = full0 + 8 * slot;
    const uint8_t* src = a.steps + o0;
    if (cy > 1)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
          " [%0], [%1], %2, [%3], %4;" ::"r"(dst), "l"(src), "r"(nb), "r"(fb), "h"((uint16_t)((1u << cy) - 1u))
          : "memory");
    else
      bulk_load(dst, src, nb, fb);
  };
  auto refill = [&](int c) {  // lane 0 of one warp: X chunk (NB TMA boxes) (+ A steps if cy == 1)
    const int slot = c % a.stages;
    uint8_t* st = sbase + (size_t)slot * a.stage_bytes;
    const uint32_t fb = full0 + 8 * slot;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(fb, (uint32_t)XST + nbytes(c));
#pragma unroll
    for (int bx = 0; bx < NB; ++bx)
      tma_load_2d(smem_u32(st + bx * (kTcpKc * 128)), &tmap, (int)n0 + 64 * bx, c * kTcpKc, fb);
    if (cy == 1) load_a(c);
  };
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tid == 0) {
    for (int c = 0; c < min(a.stages, a.nchunks); ++c) refill(c);
    if (cy > 1 && crank == 0)
      for (int c = 0; c < min(a.stages, a.nchunks); ++c) load_a(c);
  }

  float acc[NTT][4];
#pragma unroll
  for (int t = 0; t < NTT; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[t][i] = 0.0f;
  const bool active = q < a.npanels;
  // lane's role in ldmatrix.x4.trans: slot (lane & 15) of the step, n8 tile 2 j + (lane >> 4)
  const int lslot = lane & 15, lhi = lane >> 4;
  auto load_b = [&](uint32_t st, int kr, uint32_t (&bf)[NTT / 2][4]) {
    const uint32_t rowa = st + (uint32_t)kr * 128u;
    const uint32_t sw = (uint32_t)(kr & 7);
#pragma unroll
    for (int j = 0; j < NTT / 2; ++j) {
      const int tile = 2 * j + lhi;
      const uint32_t box = (uint32_t)(tile >> 3), ch = (uint32_t)(tile & 7);
      ldsm_x4_t(rowa + box * (kTcpKc * 128) + ((ch ^ sw) << 4), bf[j][0], bf[j][1], bf[j][2], bf[j][3]);
    }
  };
  uint32_t ph = 0;
  for (int c = 0; c < a.nchunks; ++c) {
    const int slot = c % a.stages;
    mbar_wait(full0 + 8 * slot, ph);
    const uint32_t st = smem_u32(sbase + (size_t)slot * a.stage_bytes);
    if (active) {
      const int* oc = offs + c * (kTcpPanels + 1);
      const int o0 = __ldg(oc), s0 = __ldg(oc + warp), s1 = __ldg(oc + warp + 1);
      const uint8_t* sp = sbase + (size_t)slot * a.stage_bytes + XST + (s0 - o0);
      const uint8_t* se = sp + (s1 - s0);
#if SRT_TCP_PACK
      // packed steps (-DSRT_TCP_PACK=1, exact-tested): each lane rebuilds its 8 fragment halves
      // from its mask and the lane-major nonzero values (~31 of 256 per step): 3.3x fewer plan
      // bytes to stream from L2, but the decode chain (header -> values -> mma) measured
      // 1.4-1.6x slower than the dense fragment; off by default
#pragma unroll 1
      while (sp < se) {
        const int kr = (int)sp[lslot];
        const uint32_t m = sp[16 + lane];
        const uint16_t* vals = (const uint16_t*)(sp + 96) + sp[48 + lane];
        const uint32_t rec = *(const uint16_t*)(sp + 80);
        uint32_t bcur[NTT / 2][4];
        load_b(st, kr, bcur);
        uint32_t hv[8];
        int k = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const bool on = (m >> i) & 1u;
          hv[i] = on ? (uint32_t)vals[k] : 0u;
          k += on ? 1 : 0;
        }
        const uint4 av = make_uint4(hv[0] | (hv[1] << 16), hv[2] | (hv[3] << 16), hv[4] | (hv[5] << 16),
                                    hv[6] | (hv[7] << 16));
#pragma unroll
        for (int j = 0; j < NTT / 2; ++j) {
          mma16816<BF>(acc[2 * j], av, bcur[j][0], bcur[j][1]);
          mma16816<BF>(acc[2 * j + 1], av, bcur[j][2], bcur[j][3]);
        }
        sp += rec;
      }
#else
      uint4 av = sp < se ? *(const uint4*)(sp + lane * 16) : make_uint4(0, 0, 0, 0);
      int kr = sp < se ? (int)sp[512 + lslot] : 0;
#pragma unroll 1
      for (; sp < se; sp += kTcpStepBytes) {
        // prefetch the next step's A fragment and slot row (shared memory)
        uint4 an = av;
        int kn = kr;
        if (sp + kTcpStepBytes < se) {
          an = *(const uint4*)(sp + kTcpStepBytes + lane * 16);
          kn = (int)sp[kTcpStepBytes + 512 + lslot];
        }
        uint32_t bcur[NTT / 2][4];
        load_b(st, kr, bcur);
#pragma unroll
        for (int j = 0; j < NTT / 2; ++j) {
          mma16816<BF>(acc[2 * j], av, bcur[j][0], bcur[j][1]);
          mma16816<BF>(acc[2 * j + 1], av, bcur[j][2], bcur[j][3]);
        }
        av = an;
        kr = kn;
      }
#endif
    }
    __syncwarp();
    uint32_t old = 0;
    if (lane == 0)
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(ctr + slot)) : "memory");
    old = __shfl_sync(0xffffffffu, old, 0);
    if ((old + 1u) % (uint32_t)nwarps == 0u && c + a.stages < a.nchunks && lane == 0) {
      refill(c + a.stages);
      if (cy > 1) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(map_rank(cempty0 + 8 * slot, 0u))
                     : "memory");
        if (crank == 0) {
          mbar_wait(cempty0 + 8 * slot, (uint32_t)((c / a.stages) & 1));
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
          load_a(c + a.stages);
        }
      }
    }
    if (slot == a.stages - 1) ph ^= 1u;
  }
  if (cy > 1) cluster_sync_all();  // no CTA leaves while multicasts / remote arrives may target it
  if (!active) return;
  // epilogue: c0, c1 -> (row g, columns 2t, 2t + 1 of tile), c2, c3 -> row g + 8
  const int g = lane >> 2, t = lane & 3;
  const bool epi = a.bias != nullptr || a.beta != 0.0f || a.relu;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int row = 16 * q + g + 8 * h;
    if (row >= a.M) continue;
    uint16_t* yr = (uint16_t*)a.Y + (int64_t)row * a.ldy;
#pragma unroll
    for (int tile = 0; tile < NTT; ++tile) {
      const int64_t col = n0 + tile * 8 + 2 * t;
      float v0 = acc[tile][2 * h], v1 = acc[tile][2 * h + 1];
      if (epi) {
        if (col < a.N) v0 = epilogue_one<true, BF>(v0, a.bias, row, a.beta, (const uint8_t*)(yr + col), a.relu);
        if (col + 1 < a.N) v1 = epilogue_one<true, BF>(v1, a.bias, row, a.beta, (const uint8_t*)(yr + col + 1), a.relu);
      }
      if (col + 1 < a.N && ((((uintptr_t)(yr + col)) & 3) == 0)) {
        *(uint32_t*)(yr + col) = (uint32_t)to16<BF>(v0) | ((uint32_t)to16<BF>(v1) << 16);
      } else {
        if (col < a.N) yr[col] = to16<BF>(v0);
        if (col + 1 < a.N) yr[col + 1] = to16<BF>(v1);
      }
    }
  }
}

static int launch_tcp(const Plan& p, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy, void* stream,
                      std::string& err, const Epilogue& ep) {
  auto encode = tensor_map_encoder();
  if (!encode || ((uintptr_t)X % 16) || ((ldx * 2) % 16)) {
    err = "tensor-core panels need a TMA-aligned X (16-byte base and row stride)";
    return SPARSE_EINTERNAL;
  }
  DeviceGuard dg(p.device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  const int warps = kTcpPanels;
  const int NB = N >= 4096 ? 2 : 1;
  const bool bf = p.dtype == SPARSE_BF16;
  auto kfn = NB == 2 ? (bf ? spmm_tcp_kernel<2, true> : spmm_tcp_kernel<2, false>)
                     : (bf ? spmm_tcp_kernel<1, true> : spmm_tcp_kernel<1, false>);
  const int stage_bytes = (NB * kTcpKc * 128 + p.tcp_max_blk + 1023) & ~1023;  // X boxes stay 1 KB aligned
  // 16 panels per CTA: one CTA per SM (126 registers x 512 threads); 8: two CTAs per SM
  const int budget = kTcpPanels >= 16 ? 227 * 1024 : 113 * 1024;
  const int stages = std::min(kMaxStages, (budget - 1024 - 256) / stage_bytes);
  if (stages < 2) {
    err = "tensor-core panels: a chunk's steps do not fit two pipeline stages";
    return SPARSE_EUNSUPPORTED;
  }
  const int smem = stages * stage_bytes + 1024 + 256;
  const int cy = SRT_TCP_CY;
  cudaError_t e = ensure_smem_attr(kfn, smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof tmap);
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)p.K};
  cuuint64_t strides[1] = {(cuuint64_t)(ldx * 2)};
  cuuint32_t box[2] = {64u, (cuuint32_t)kTcpKc};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)X, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "tensor-core panels: cuTensorMapEncodeTiled failed";
    return SPARSE_EINTERNAL;
  }
  TcpArgs a;
  a.step_off = p.d_tcp_step_off;
  a.steps = p.d_tcp_steps;
  a.Y = (uint8_t*)Y;
  a.ldy = ldy;
  a.N = N;
  a.M = p.M;
  a.nchunks = p.tcp_nchunks;
  a.npanels = p.tcp_npanels;
  a.stages = stages;
  a.stage_bytes = stage_bytes;
  a.cy = cy;
  a.bias = (const uint8_t*)ep.bias;
  a.beta = ep.beta;
  a.relu = ep.relu;
  const int64_t ntn = ((N + 64 * NB - 1) / (64 * NB) + cy - 1) / cy * cy;  // whole clusters
  if (ntn > 65535) {
    err = "tensor-core panels: N too large for one launch";
    return SPARSE_EUNSUPPORTED;
  }
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3((unsigned)((p.tcp_npanels + warps - 1) / warps), (unsigned)ntn, 1);  // x = group G
  cfg.blockDim = dim3((unsigned)(warps * 32), 1, 1);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = (unsigned)cy;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, kfn, tmap, a);
  if (e != cudaSuccess) return cuda_fail(e, "tensor-core panel launch", err);
  return SPARSE_OK;
}

// ------------------------------------------------------------------ tcgen05 blocks (executor 4)
// SURVEY NEXT #1 on Blackwell's 5th-generation tensor cores: W's nonzero 128 x 64 blocks (stored
// dense, pre-swizzled by the inspector) times X on tcgen05.mma, fp32 accumulators in TMEM.
// Tile = 128 rows of W x 256 columns of X; a persistent CTA walks tiles (row block fastest, so
// concurrently running CTAs share the X tile in L2).  Warp roles (the canonical sm_100 GEMM
// shape): warp 0 = producer (per nonzero block of the tile's row block: one bulk copy of the
// 16 KB W block + four 128-byte-swizzled TMA boxes of X (64 k rows x 64 columns each) into a
// ring stage), warp 1 = MMA issuer (one elected lane: 4 x tcgen05.mma M128 N256 K16 per stage,
// tcgen05.commit releases the stage), warps 2-5 = epilogue (tcgen05.ld of their 32 TMEM lanes =
// 32 rows, fp32 -> 16-bit, fused bias / beta / ReLU, stores).  Two TMEM accumulators (2 x 256
// columns) let the epilogue of a tile overlap the MMAs of the next.  Summation order: k-block
// ascending, the tensor core's order inside a K16 step (within tolerance; exact on integer data).
constexpr int kTcgMetaMax = 2048;  // block-list entries kept in shared memory
struct TcgArgs {
  const uint8_t* blocks;     // [entries][cs][A bytes] pre-swizzled W blocks (fp32: [W_hi | W_lo])
  const int32_t* meta;       // [ngroups + 1] prefix, then k-block indices
  int32_t nblk;              // union entries of all groups (k-block list length)
  uint8_t* Y;
  int64_t ldy, N;            // conv: N = the span of the interleaved copies (positions incl. halo)
  int32_t M, ngroups, cs, stages;
  int32_t dbg;               // diagnostics only (SRT_TCG_DBG): 1 = skip the Y stores, 2 = skip the MMAs
  const uint8_t* bias;
  float beta;
  int32_t relu;
  uint32_t idesc;
  // conv (implicit im2col over the interleaved copies): pitch P = g W, group stride Sg =
  // (H + 2) P, 64-channel blocks per tap ncb, batch Bt, output plane B H W
  int32_t P, g, Sg, H, W, ncb, Bt;
  int64_t plane;
  // split tail (sp > 1): the first `rounds` x clusters tiles run whole; the remaining `ntail`
  // tiles are each cut into sp column slices of np = 256 / sp columns (whole X boxes), one per
  // cluster, each over the full k-block list with an N = np instruction descriptor (idesc_p).
  // No partial sums: a slice is the same per-column dot products, just fewer columns.
  int32_t rounds, sp, ntail, np;
  uint32_t idesc_p;
  // CTA pair (cs == 2): rank 0 issues tcgen05.mma.cta_group::2 (M = 256) over both CTAs' W
  // blocks and X halves
  int32_t pair;
  // conv through im2col TMA (i2c = 1): X is NHWC (plane = B H W pixels, N = plane, ldy = plane),
  // B is K-major (pixel rows of 128-byte channel groups); each CTA loads i2c_pix pixels per tile
  int32_t i2c, i2c_pix;
  // tile width (columns of Y per tile; 0 = 256): the im2col conv picks it so that the tiles fill
  // the persistent clusters' rounds (C5: 196 tiles of 256 on 74 pairs = 2.65 rounds; 210 of 240)
  int32_t bn;
  // column stride of Y in elements (0 = 1): the NHWC conv writes Y[pixel][channel] (ldy = 1,
  // ycs = M) - consecutive lanes (rows = output channels) store consecutive addresses
  int64_t ycs;
  // K slices per tile (ks > 1): work item = (tile, slice), a slice's k-block range is
  // [j0 + L s / ks, j0 + L (s + 1) / ks); its fp32 partial goes to ws[s][column][row] (rows
  // contiguous: lanes store consecutive addresses) and tcg_ksum adds the slices in order
  int32_t ks;
  float* ws;
  // tail K slices (tks > 1, chosen at launch): the `ntail` tiles left after `rounds` full rounds
  // are each cut into tks K slices, one per otherwise idle cluster; slice partials go to
  // tws[(slice ntail + tail tile) BNT + column][group row] and tcg_tailsum adds them in order
  int32_t tks;
  float* tws;
};

// work item i of cluster cl: tile t and column slice (-1 = the whole tile)
__device__ __forceinline__ bool tcg_work(const TcgArgs& a, int64_t cl, int64_t ncl, int64_t i, int64_t ntiles,
                                         int64_t& t, int& slice, int& tk) {
  slice = -1;
  tk = -1;
  if (a.tks > 1 && i >= a.rounds) {  // tail K slices
    if (i > a.rounds || cl >= (int64_t)a.ntail * a.tks) return false;
    t = (int64_t)a.rounds * ncl + cl / a.tks;
    tk = (int)(cl % a.tks);
    return true;
  }
  if (a.ks > 1) {  // (tile, K slice) items; t carries the slice in its low bits: see tcg_kslice
    t = cl + i * ncl;
    return t < ntiles * a.ks;
  }
  if (a.sp <= 1 || i < a.rounds) {
    t = cl + i * ncl;
    return t < ntiles;
  }
  if (i == a.rounds && cl < (int64_t)a.ntail * a.sp) {
    t = (int64_t)a.rounds * ncl + cl / a.sp;
    slice = (int)(cl % a.sp);
    return true;
  }
  return false;
}

// K-sliced items (ks > 1): item -> tile (returned) and slice ksl
__device__ __forceinline__ int64_t tcg_item(const TcgArgs& a, int64_t item, int& ksl) {
  if (a.ks <= 1) {
    ksl = 0;
    return item;
  }
  const int64_t t = item / a.ks;
  ksl = (int)(item - t * a.ks);
  return t;
}
// the slice's part [j0, j1) of the group's k-block entries (plan K slices, or a tail K slice)
__device__ __forceinline__ void tcg_krange(const TcgArgs& a, int ksl, int tk, int& j0, int& j1) {
  const int n = tk >= 0 ? a.tks : a.ks, k = tk >= 0 ? tk : ksl;
  if (n <= 1) return;
  const int L = j1 - j0, jb = j0;
  j0 = jb + (int)((int64_t)L * k / n);
  j1 = jb + (int)((int64_t)L * (k + 1) / n);
}

// shared-memory matrix descriptor: start, leading / stride byte offsets, version 1 (bit 46),
// layout type (bits 61-63): 2 = 128-byte swizzle (16-byte chunks, 8-row atoms), 1 = 128-byte
// swizzle of 32-byte chunks (4-row atoms; the only layout for MN-major TF32 operands)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                                    uint32_t layout = 2u) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
template <bool TF>
__device__ __forceinline__ void umma(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t en,
                                     bool pair = false) {
  if (pair) {  // CTA pair: M = 256 over both CTAs' A and B halves, D in both CTAs' TMEM
    if (TF)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
          "l"(da), "l"(db), "r"(idesc), "r"(en)
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
          "l"(da), "l"(db), "r"(idesc), "r"(en)
          : "memory");
    return;
  }
  if (TF)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(en)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(en)
        : "memory");
}
// arrive on the mbarrier at offset `bar` of every CTA in `mask` once this thread's MMAs are done
__device__ __forceinline__ void tm_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          bar),
      "h"(mask)
      : "memory");
}
// CTA pair: arrive on the mbarrier at offset `bar` of both CTAs once the pair's MMAs are done
__device__ __forceinline__ void tm_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          bar),
      "h"((uint16_t)3)
      : "memory");
}
// tcgen05.ld 32x32b.x32: this warp's 32 TMEM lanes x 32 consecutive columns (no wait)
__device__ __forceinline__ void tm_ld32(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(ta));
}
__device__ __forceinline__ void tm_ld16(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(ta));
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar, uint16_t mask, bool mc) {
  if (mc)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "h"(mask)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

// CTA pair: TMA load into this CTA's shared memory whose completion is signalled on the
// mbarrier `bar` of the pair's rank 0 (shared::cluster address) - the 2-SM load form
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// im2col TMA (NHWC input, 3x3 pad 1): `pixels` consecutive output pixels (the map's
// pixelsPerColumn) from the one at (b, y, x), tap (dy, dx), channels c .. c + channelsPerPixel -
// 1: smem row i = the channels of input pixel (y + dy - 1, x + dx - 1) of output pixel i (zero
// outside the image) - the K-major B operand of the implicit GEMM, no im2col matrix in memory
__device__ __forceinline__ void tma_im2col(uint32_t dst, const CUtensorMap* map, int c, int x, int y, int b,
                                           uint16_t dx, uint16_t dy, uint32_t bar, uint16_t mask, int mode) {
  if (mode == 1)  // multicast to the cluster
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8}, %9;" ::"r"(dst),
        "l"((uint64_t)map), "r"(c), "r"(x - 1), "r"(y - 1), "r"(b), "r"(bar), "h"(dx), "h"(dy), "h"(mask)
        : "memory");
  else if (mode == 2)  // CTA pair: completes on rank 0's barrier
    asm volatile(
        "cp.async.bulk.tensor.4d.im2col.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(dst),
        "l"((uint64_t)map), "r"(c), "r"(x - 1), "r"(y - 1), "r"(b), "r"(bar), "h"(dx), "h"(dy)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(dst),
        "l"((uint64_t)map), "r"(c), "r"(x - 1), "r"(y - 1), "r"(b), "r"(bar), "h"(dx), "h"(dy)
        : "memory");
}

// conv epilogue: the NT epilogue threads (tid 0 .. NT - 1) decode the tile's 256 span positions
// once (named barrier among the epilogue warps only): s -> group q, row r, column (image j, x)
// -> the CNHW offset of the output pixel, -1 for halo rows, padding images and past the span
template <int NT>
__device__ __forceinline__ void tcg_conv_table(int32_t* otab, int64_t n0, const TcgArgs& a, int tid) {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");  // the previous tile's readers are done
  for (int c = tid; c < 256; c += NT) {
    const int64_t sp = n0 + c;
    const int64_t gq = sp / a.Sg;
    const int rem = (int)(sp - gq * a.Sg), r = rem / a.P, xx = rem - r * a.P, jj = xx / a.W;
    const int64_t b = gq * a.g + jj;
    otab[c] = (sp < a.N && r >= 1 && r <= a.H && b < a.Bt) ? (int32_t)((b * a.H + (r - 1)) * a.W + (xx - jj * a.W)) : -1;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// TF = fp32 plan as 3xTF32.  Per stage (k-block):
//   16-bit: A = one 128 x 64 W block (16 KB), B = 64 k x 256 columns of X as 4 boxes of 64
//           columns (8 KB each); 4 x tcgen05.mma kind::f16 K16
//   TF:     A = [W_hi | W_lo] (2 x 16 KB, 128 x 32 fp32 each), B = [X_hi | X_lo] (2 x 32 KB,
//           8 boxes of 32 k x 32 columns each); per K8 step 3 x tcgen05.mma kind::tf32:
//           W_hi X_hi + W_lo X_hi + W_hi X_lo
// Cluster of cs CTAs = cs consecutive row blocks (one group) on the same N tile: CTA rank r
// loads boxes [r * NBOX / cs, (r + 1) * NBOX / cs) and multicasts them to the whole cluster;
// a stage is refilled only when every CTA of the cluster has consumed it (each CTA's MMA
// commit arrives on the stage's empty barrier in all cs CTAs).
// PAIR (a template parameter: a kernel containing cta_group::2 instructions cannot be launched
// without a cluster) = CTA pairs, see TcgArgs::pair.
template <bool BF, bool CONV = false, bool TF = false, bool PAIR = false>
__global__ void __launch_bounds__(TF ? 320 : 192, 1) spmm_tcg_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          const __grid_constant__ CUtensorMap tmap2,
                                                          const __grid_constant__ CUtensorMap tmapA,
                                                          const TcgArgs a) {
  constexpr int BN = 256, A_HALF = 128 * 128, A_BYTES = TF ? 2 * A_HALF : A_HALF;
  constexpr int NBOX = TF ? 8 : 4, BOX_BYTES = TF ? 32 * 128 : 64 * 128, BOX_COLS = TF ? 32 : 64;
  constexpr int B_HALF = NBOX * BOX_BYTES, B_BYTES = TF ? 2 * B_HALF : B_HALF;
  constexpr int ST_BYTES = A_BYTES + B_BYTES, KSTEP_B = TF ? 1024 : 2048;
  // epilogue warps, and k-blocks per TMEM partial (TF: short truncating chains, see below)
  constexpr int NEPI = TF ? 8 : 4, FLUSH = TF ? 8 : (1 << 30);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);  // SW128: 1 KB atoms
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.stages, CS = a.cs;
  const uint32_t rank = CS > 1 ? cluster_rank() : 0u;
  const uint16_t mask = (uint16_t)((1u << CS) - 1u);
  const int64_t cl = blockIdx.x / CS, ncl = gridDim.x / CS;
  // a CTA of a pair stages its W block and half of the X tile (one operand half = BHE bytes)
  constexpr bool pair = PAIR;
  const int BHE = pair ? B_HALF / 2 : B_HALF, STB = A_BYTES + (TF ? 2 : 1) * BHE;
  uint64_t* bars = (uint64_t*)(smem + (size_t)S * STB);
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * S;
  const uint32_t tfull0 = empty0 + 8 * S, tempty0 = tfull0 + 16;
  uint32_t* tslot = (uint32_t*)(bars + 2 * S + 4);
  const int BNT = a.bn > 0 ? a.bn : BN;  // tile width (the TMEM accumulators stay BN apart)
  const int64_t nnb = (a.N + BNT - 1) / BNT;
  const int64_t ntiles = (int64_t)a.ngroups * nnb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      // pair: only rank 0's full barriers are used (both CTAs' loads complete on them)
      mbar_init(full0 + 8 * s, 1);
      // one MMA commit per CTA of the cluster (pair: rank 0's one commit reaches both)
      mbar_init(empty0 + 8 * s, pair ? 1u : (uint32_t)CS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, pair ? 2 * NEPI : NEPI);  // one arrive per epilogue warp (of the pair)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: two 128 x 256 fp32 accumulators (pair: allocated in both CTAs at once)
    if (pair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tm_fence_before();
  __syncthreads();
  if (CS > 1) cluster_sync_all();  // peers multicast into this CTA's stages and barriers
  tm_fence_after();
  const uint32_t tbase = *tslot;
  // the block lists, copied once into shared memory (dependent global loads on the producer's
  // issue path were the kernel's top stall)
  const int nmeta = a.ngroups + 1 + a.nblk;
  const int32_t* meta = a.meta;
  if (nmeta <= kTcgMetaMax) {
    int32_t* sm = (int32_t*)((uint8_t*)tslot + 64 + 1024);
    for (int i = threadIdx.x; i < nmeta; i += blockDim.x) sm[i] = __ldg(a.meta + i);
    __syncthreads();
    meta = sm;
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      const int nb = NBOX / CS;  // X boxes per operand this CTA loads (and multicasts)
      const bool mc = CS > 1 && !pair;
      int s = 0;
      uint32_t ph = 0;
      int64_t t;
      int slice, tk;
      for (int64_t it = 0; tcg_work(a, cl, ncl, it, ntiles, t, slice, tk); ++it) {
        int ksl;
        t = tcg_item(a, t, ksl);
        const int gi = (int)(t % a.ngroups);
        const int64_t n0 = (t / a.ngroups) * BNT;
        int j0 = meta[gi], j1 = meta[gi + 1];
        tcg_krange(a, ksl, tk, j0, j1);
        // boxes of this work item: the whole tile (this CTA loads boxes rank nb .. + nb - 1 and
        // multicasts them), or the slice's nbs boxes (box i loaded by rank i % CS) stored from
        // box 0 of the stage.  This thread's loads: stage positions pos0 + i pstep, i < cnt, of
        // tile box position + boff.  (The issue path is kept short: for 16-bit plans a stage's
        // MMAs take ~0.26 us, the single producer thread must issue its loads within that.)
        // A pair: each CTA loads (no multicast) and stages its half of the item's boxes.
        const int nbs = slice < 0 ? NBOX : NBOX / a.sp;
        int pos0, pstep, cnt, boff, nst;
        if (pair) {
          pos0 = 0, pstep = 1, cnt = nbs / 2, boff = (slice < 0 ? 0 : slice * nbs) + (int)rank * (nbs / 2);
          nst = nbs / 2;
        } else {
          pos0 = slice < 0 ? (int)rank * nb : (int)rank, pstep = slice < 0 ? 1 : CS;
          cnt = slice < 0 ? nb : ((int)rank < nbs ? (nbs - 1 - (int)rank) / CS + 1 : 0);
          boff = slice < 0 ? 0 : slice * nbs;
          nst = nbs;
        }
        uint32_t tx = (uint32_t)(A_BYTES + (TF ? 2 : 1) * nst * BOX_BYTES);
        // im2col conv: this CTA's first pixel (a pair / multicast cluster: rank r loads pixels
        // r i2c_pix .. of the tile; a multicast CTA's stage receives the whole tile)
        int ib = 0, iy = 0, ix = 0;
        uint32_t i2c_dst = 0;
        if (CONV && a.i2c) {
          const int64_t p0 = n0 + (CS > 1 ? (int64_t)rank * a.i2c_pix : 0);
          const int64_t hw = (int64_t)a.H * a.W;
          ib = (int)(p0 / hw);
          const int rem = (int)(p0 - (int64_t)ib * hw);
          iy = rem / a.W;
          ix = rem - iy * a.W;
          i2c_dst = (CS > 1 && !pair) ? (uint32_t)rank * (uint32_t)a.i2c_pix * 128u : 0u;
          tx = (uint32_t)(A_BYTES + (TF ? 2 : 1) * (pair ? a.i2c_pix : BNT) * 128);
        }
        for (int j = j0; j < j1; ++j) {
          const int kb = meta[a.ngroups + 1 + j];
          mbar_wait(empty0 + 8 * s, ph ^ 1u);
          uint8_t* st = smem + (size_t)s * STB;
          // pair: both CTAs' loads complete on rank 0's barrier, which expects both CTAs' bytes
          const uint32_t fb = pair ? map_rank(full0 + 8 * s, 0) : full0 + 8 * s;
          if (!pair || rank == 0) mbar_arrive_expect_tx(full0 + 8 * s, pair ? 2 * tx : tx);
          if constexpr (pair)  // the W block through a plain 2-D map of 128-byte rows
            tma_load_2d_pair(smem_u32(st), &tmapA, 0, (int)(((int64_t)j * CS + rank) * (A_BYTES / 128)), fb);
          else
            bulk_load(smem_u32(st), a.blocks + ((size_t)j * CS + rank) * A_BYTES, (uint32_t)A_BYTES, fb);
          uint32_t dst = smem_u32(st + A_BYTES + pos0 * BOX_BYTES);
          if (CONV && a.i2c) {  // k-block (channel block, dx, dy): one im2col box per operand
            const int cb = kb / 9, r9 = kb - cb * 9, dx = r9 / 3, dy = r9 - dx * 3;
            const uint32_t d0 = smem_u32(st + A_BYTES) + i2c_dst;
            const int mode = pair ? 2 : (CS > 1 ? 1 : 0);
            tma_im2col(d0, &tmap, cb * (TF ? 32 : 64), ix, iy, ib, (uint16_t)dx, (uint16_t)dy, fb, mask, mode);
            if (TF) tma_im2col(d0 + BHE, &tmap2, cb * 32, ix, iy, ib, (uint16_t)dx, (uint16_t)dy, fb, mask, mode);
          } else if (CONV) {  // k-block (channel block, dx, dy): copy dx, shifted by (dy - 1) pitches
            const int cb = kb / 9, r9 = kb - cb * 9, dx = r9 / 3, dy = r9 - dx * 3;
            int c0 = (int)n0 + (dy - 1) * a.P + BOX_COLS * (pos0 + boff);
            const int c1 = cb * (TF ? 32 : 64);
            for (int i = 0; i < cnt; ++i, dst += pstep * BOX_BYTES, c0 += pstep * BOX_COLS) {
              if constexpr (pair) {
                tma_load_3d_pair(dst, &tmap, c0, c1, dx, fb);
                if (TF) tma_load_3d_pair(dst + BHE, &tmap2, c0, c1, dx, fb);
              } else {
                tma_load_3d(dst, &tmap, c0, c1, dx, fb, mask, mc);
                if (TF) tma_load_3d(dst + BHE, &tmap2, c0, c1, dx, fb, mask, mc);  // X_lo copies
              }
            }
          } else {
            int c0 = (int)n0 + BOX_COLS * (pos0 + boff);
            const int c1 = kb * (TF ? 32 : 64);
            for (int i = 0; i < cnt; ++i, dst += pstep * BOX_BYTES, c0 += pstep * BOX_COLS) {
              if constexpr (pair) {
                tma_load_2d_pair(dst, &tmap, c0, c1, fb);
                if (TF) tma_load_2d_pair(dst + BHE, &tmap2, c0, c1, fb);
                continue;
              }
              if (mc) tma_load_2d_mc(dst, &tmap, c0, c1, fb, mask);
              else tma_load_2d(dst, &tmap, c0, c1, fb);
              if (TF) {
                if (mc) tma_load_2d_mc(dst + BHE, &tmap2, c0, c1, fb, mask);
                else tma_load_2d(dst + BHE, &tmap2, c0, c1, fb);
              }
            }
          }
          if (++s == S) s = 0, ph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one lane)
    // A tile's k-blocks run in chunks of FLUSH k-blocks, each into a fresh TMEM partial
    // (alternating between the two 256-column buffers); 16-bit plans: one chunk per tile
    if (lane == 0 && (!pair || rank == 0)) {  // (pair: rank 0 issues the pair's MMAs)
      int s = 0, acc = 0;
      uint32_t ph = 0, aph[2] = {0u, 0u};
      int64_t t;
      int slice, tk;
      for (int64_t it = 0; tcg_work(a, cl, ncl, it, ntiles, t, slice, tk); ++it) {
        int ksl;
        t = tcg_item(a, t, ksl);
        const int gi = (int)(t % a.ngroups);
        int j0 = meta[gi], j1 = meta[gi + 1];
        tcg_krange(a, ksl, tk, j0, j1);
        const uint32_t idesc = slice < 0 ? a.idesc : a.idesc_p;
        int j = j0;
        do {
          const int jc = j, je = min(j1, j + FLUSH);
          // the epilogue (pair: of both CTAs) drained this buffer
          if (pair) mbar_wait_cluster(tempty0 + 8 * acc, aph[acc] ^ 1u);
          else mbar_wait(tempty0 + 8 * acc, aph[acc] ^ 1u);
          tm_fence_after();
          const uint32_t d = tbase + (uint32_t)(acc * BN);
          for (; j < je; ++j) {
            mbar_wait(full0 + 8 * s, ph);
            tm_fence_after();
            const uint32_t sa = smem_u32(smem + (size_t)s * STB), sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              // A: K-major SW128 (rows of 128 B, 8-row atoms of 1 KB): K step (16 x 16-bit or
              //    8 x tf32) = +32 B
              // B: MN-major (128-byte column groups of BOX_BYTES): 16-bit: 128-byte swizzle,
              //    8-row atoms (SBO 1 KB), K16 step = +2 KB; TF32: 32-byte-chunk swizzle, 4-row
              //    atoms (SBO 512 B), K8 step = +1 KB
              const uint32_t en = (j > jc || k > 0) ? 1u : 0u;
              if (a.dbg & 2) continue;
              constexpr uint32_t B_SBO = TF ? 512u : 1024u, B_LAYOUT = TF ? 1u : 2u;
              const uint64_t da = umma_desc_sw128(sa + 32u * k, 16u, 1024u);
              // im2col conv: B K-major like A (pixel rows of 128 B, K step = +32 B)
              const uint64_t db = (CONV && a.i2c) ? umma_desc_sw128(sb + 32u * k, 16u, 1024u)
                                                  : umma_desc_sw128(sb + (uint32_t)KSTEP_B * k, (uint32_t)BOX_BYTES, B_SBO, B_LAYOUT);
              umma<TF>(d, da, db, idesc, en, pair);
              if (TF) {
                const uint64_t da_lo = umma_desc_sw128(sa + A_HALF + 32u * k, 16u, 1024u);
                const uint64_t db_lo =
                    (CONV && a.i2c) ? umma_desc_sw128(sb + (uint32_t)BHE + 32u * k, 16u, 1024u)
                                    : umma_desc_sw128(sb + (uint32_t)BHE + (uint32_t)KSTEP_B * k, (uint32_t)BOX_BYTES, B_SBO, B_LAYOUT);
                umma<TF>(d, da_lo, db, idesc, 1u, pair);
                umma<TF>(d, da, db_lo, idesc, 1u, pair);
              }
            }
            // the stage is free once these MMAs have read it (in every CTA of the cluster)
            if (pair) tm_commit_pair(empty0 + 8 * s);
            else if (CS > 1) tm_commit_mc(empty0 + 8 * s, mask);
            else tm_commit(empty0 + 8 * s);
            if (++s == S) s = 0, ph ^= 1u;
          }
          // partial complete (also when the group is empty); pair: in both CTAs' TMEM
          if (pair) tm_commit_pair(tfull0 + 8 * acc);
          else tm_commit(tfull0 + 8 * acc);
          aph[acc] ^= 1u;
          acc ^= 1;
        } while (j < j1);
      }
    }
  } else if constexpr (TF) {
    // ---------------- epilogue (3xTF32): 8 warps; warp w reads TMEM lanes 32 (w % 4) .. + 31
    // (rows of the tile) and columns 128 ((w - 2) / 4) .. + 127.  The tensor core's fp32
    // accumulation truncates (measured: error linear in K, 1.1e-5 rel-L2 at K = 3072), so the
    // chain stays short: every FLUSH k-blocks the partial is added into an fp32 master held in
    // registers (round to nearest), in k order - a fixed summation order.
    const int q = warp & 3, hc = ((warp - 2) >> 2) * 128;
    int acc = 0;
    uint32_t aph[2] = {0u, 0u};
    const bool epi = a.bias != nullptr || a.beta != 0.0f || a.relu;
    // per-warp staging buffer (32 rows x 64 B) for coalesced Y stores
    uint8_t* stg = (uint8_t*)tslot + 64 + 1024 + 4 * kTcgMetaMax + (warp - 2) * 2048;
    const int64_t ycs = a.ycs > 0 ? a.ycs : 1;
    const bool coal = ycs == 1 && ((a.ldy * 4) % 16) == 0 && ((uintptr_t)a.Y % 16) == 0;
    int32_t* otab = (int32_t*)((uint8_t*)tslot + 64);  // conv: span position -> output offset
    int64_t tab_n0 = -1;
    int64_t t;
    int slice, tk;
    for (int64_t it = 0; tcg_work(a, cl, ncl, it, ntiles, t, slice, tk); ++it) {
      int ksl;
      t = tcg_item(a, t, ksl);
      const int gi = (int)(t % a.ngroups);
      const int rb = gi * CS + (int)rank;
      const int64_t nt0 = (t / a.ngroups) * BNT;
      // accumulator column c = tile column cbase + c (a slice: the first nacc columns)
      const int cbase = slice < 0 ? 0 : slice * a.np, nacc = slice < 0 ? BNT : a.np;
      const int64_t n0 = nt0 + cbase;
      int kj0 = meta[gi], kj1 = meta[gi + 1];
      tcg_krange(a, ksl, tk, kj0, kj1);
      const int nent = kj1 - kj0;
      if (CONV && !a.i2c && nt0 != tab_n0) {
        tcg_conv_table<32 * NEPI>(otab, nt0, a, threadIdx.x - 64);
        tab_n0 = nt0;
      }
      const int nch = nent > 0 ? (nent + FLUSH - 1) / FLUSH : 1;
      float m[128];
#pragma unroll
      for (int c = 0; c < 128; ++c) m[c] = 0.0f;
      for (int ch = 0; ch < nch; ++ch) {
        mbar_wait(tfull0 + 8 * acc, aph[acc]);
        tm_fence_after();
        if (nent > 0) {
#pragma unroll
          for (int c0 = 0; c0 < 128; c0 += 16) {
            uint32_t v[16];
            tm_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + hc + c0), v);
            tm_wait_ld();
#pragma unroll
            for (int c = 0; c < 16; ++c) m[c0 + c] = __fadd_rn(m[c0 + c], __uint_as_float(v[c]));
          }
        }
        tm_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (pair && rank == 1) mbar_arrive_remote(map_rank(tempty0 + 8 * acc, 0));
          else mbar_arrive(tempty0 + 8 * acc);
        }
        aph[acc] ^= 1u;
        acc ^= 1;
      }
      const int row0 = rb * 128 + q * 32, row = row0 + lane;
      const int ncol = (int)max((int64_t)0, min((int64_t)nacc, a.N - n0));
      if (row0 >= a.M || (a.dbg & 1)) continue;
      if (tk >= 0) {  // tail K slice: the fp32 partial of this CTA's rows, lanes = consecutive rows
        const int R = CS * 128;
        float* wp = a.tws + ((size_t)(tk * a.ntail + (t - (int64_t)a.rounds * ncl)) * BNT + hc) * R +
                    (int)rank * 128 + q * 32 + lane;
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (hc + c < ncol) wp[(size_t)c * R] = m[c];
        continue;
      }
      if (a.ks > 1) {  // K slice: the fp32 partial, column-major (lanes = consecutive rows)
        if (row < a.M) {
          float* wp = a.ws + ((size_t)ksl * a.N + n0 + hc) * a.M + row;
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (hc + c < ncol) wp[(size_t)c * a.M] = m[c];
        }
        continue;
      }
      if (CONV && !a.i2c) {
        // span positions -> CNHW pixels (otab; -1 = halo / padding / past the span)
        if (hc >= nacc) continue;
        if (epi) {
#pragma unroll
          for (int c = 0; c < 128; ++c) {
            const int32_t o = hc + c < nacc ? otab[cbase + hc + c] : -1;
            if (row < a.M && o >= 0)
              m[c] = epilogue_one<false>(m[c], a.bias, row, a.beta, a.Y + ((int64_t)row * a.plane + o) * 4, a.relu);
          }
        }
        // 16 positions of the warp's 32 rows through the staging buffer, then each store
        // instruction writes 16 consecutive span positions of two output rows
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 16) {
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *(float4*)(stg + lane * 64 + ((j ^ (lane & 3)) * 16)) =
                make_float4(m[c0 + 4 * j], m[c0 + 4 * j + 1], m[c0 + 4 * j + 2], m[c0 + 4 * j + 3]);
          __syncwarp();
          const int c = lane & 15;
          const int32_t o = hc + c0 + c < nacc ? otab[cbase + hc + c0 + c] : -1;
          if (o >= 0) {
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
              const int r = 2 * i + (lane >> 4);
              if (row0 + r >= a.M) break;
              const float v = *(const float*)(stg + r * 64 + (((c >> 2) ^ (r & 3)) * 16) + (c & 3) * 4);
              *(float*)(a.Y + ((int64_t)(row0 + r) * a.plane + o) * 4) = v;
            }
          }
        }
        continue;
      }
      if (epi) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (row < a.M && hc + c < ncol)
            m[c] = epilogue_one<false>(m[c], a.bias, row, a.beta, a.Y + ((int64_t)row * a.ldy + (n0 + hc + c) * ycs) * 4, a.relu);
      }
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 16) {
        if (hc + c0 >= ncol) break;
        if (coal && hc + c0 + 16 <= ncol) {
          // 16 fp32 of the row -> staging (16-byte chunks XOR-swizzled by row), then each store
          // instruction writes eight whole 64-byte row segments
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *(float4*)(stg + lane * 64 + ((j ^ (lane & 3)) * 16)) =
                make_float4(m[c0 + 4 * j], m[c0 + 4 * j + 1], m[c0 + 4 * j + 2], m[c0 + 4 * j + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = i * 8 + (lane >> 2), j = lane & 3;
            const float4 d4 = *(const float4*)(stg + r * 64 + ((j ^ (r & 3)) * 16));
            if (row0 + r < a.M) *(float4*)(a.Y + ((int64_t)(row0 + r) * a.ldy + n0 + hc + c0) * 4 + j * 16) = d4;
          }
        } else if (row < a.M) {
          float* yp = (float*)(a.Y + ((int64_t)row * a.ldy + (n0 + hc + c0) * ycs) * 4);
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (hc + c0 + c < ncol) yp[c * ycs] = m[c0 + c];
        }
      }
    }
  } else {
    // ---------------- epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 = rows of the tile
    const int q = warp & 3;
    int acc = 0;
    uint32_t aph[2] = {0u, 0u};
    const bool epi = a.bias != nullptr || a.beta != 0.0f || a.relu;
    int32_t* otab = (int32_t*)((uint8_t*)tslot + 64);  // conv: span position -> output offset
    int64_t tab_n0 = -1;
    // per-warp staging buffer (32 rows x 128 B) for coalesced Y stores
    uint8_t* stg = (uint8_t*)tslot + 64 + 1024 + 4 * kTcgMetaMax + (warp - 2) * 4096;
    const int64_t ycs = a.ycs > 0 ? a.ycs : 1;
    const bool coal = ycs == 1 && a.beta == 0.0f && ((a.ldy * 2) % 16) == 0 && ((uintptr_t)a.Y % 16) == 0;
    int64_t t;
    int slice, tk;
    for (int64_t it = 0; tcg_work(a, cl, ncl, it, ntiles, t, slice, tk); ++it) {
      int ksl;
      t = tcg_item(a, t, ksl);
      const int gi = (int)(t % a.ngroups);
      const int rb = gi * CS + (int)rank;
      const int64_t nt0 = (t / a.ngroups) * BNT;
      // accumulator column c = tile column cbase + c (a slice: the first nacc columns)
      const int cbase = slice < 0 ? 0 : slice * a.np, nacc = slice < 0 ? BNT : a.np;
      const int64_t n0 = nt0 + cbase;
      int kj0 = meta[gi], kj1 = meta[gi + 1];
      tcg_krange(a, ksl, tk, kj0, kj1);
      const bool has = kj1 > kj0;
      if (CONV && !a.i2c && nt0 != tab_n0) {
        tcg_conv_table<128>(otab, nt0, a, threadIdx.x - 64);
        tab_n0 = nt0;
      }
      const int32_t* ot = otab + cbase;
      mbar_wait(tfull0 + 8 * acc, aph[acc]);
      tm_fence_after();
      const int row0 = rb * 128 + q * 32, row = row0 + lane;
      const int ncol = (int)min((int64_t)nacc, a.N - n0);
      if (tk >= 0 || a.ks > 1) {
        // K slice (plan K slices or a tail K slice): the tile's fp32 partial, column-major (lanes
        // = consecutive rows).  A separate loop: the plain store loop below stays as lean as it
        // was (these branches inside it cost short-K 16-bit tiles ~15 %, measured)
#pragma unroll 1
        for (int c0 = 0; c0 < nacc; c0 += 32) {
          uint32_t v[32];
          tm_ld32(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), v);
          tm_wait_ld();
          if (c0 >= ncol || row0 >= a.M) continue;
          float* wp;
          size_t cst;
          if (tk >= 0) {
            cst = (size_t)CS * 128;
            wp = a.tws + ((size_t)(tk * a.ntail + (t - (int64_t)a.rounds * ncl)) * BNT + c0) * cst +
                 (int)rank * 128 + q * 32 + lane;
          } else {
            if (row >= a.M) continue;
            cst = (size_t)a.M;
            wp = a.ws + ((size_t)ksl * a.N + n0 + c0) * a.M + row;
          }
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c0 + c < ncol) wp[c * cst] = has ? __uint_as_float(v[c]) : 0.0f;
        }
        tm_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (pair && rank == 1) mbar_arrive_remote(map_rank(tempty0 + 8 * acc, 0));
          else mbar_arrive(tempty0 + 8 * acc);
        }
        aph[acc] ^= 1u;
        acc ^= 1;
        continue;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < nacc; c0 += 64) {
        uint32_t v[64];
        const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0);
        tm_ld32(ta, v);
        tm_ld32(ta + 32, v + 32);
        tm_wait_ld();
        if (CONV && !a.i2c) {
          if (a.beta != 0.0f) {  // beta * Y_old: element-wise (the fp32 sum needs Y_old)
            if (row >= a.M) continue;
#pragma unroll
            for (int c = 0; c < 64; ++c) {  // (unrolled: v stays in registers)
              const int32_t o = ot[c0 + c];
              if (o < 0) continue;
              uint8_t* yp = a.Y + ((int64_t)row * a.plane + o) * 2;
              const float f = epilogue_one<true, BF>(has ? __uint_as_float(v[c]) : 0.0f, a.bias, row, a.beta, yp, a.relu);
              *(uint16_t*)yp = to16<BF>(f);
            }
            continue;
          }
          // rows' values through the staging buffer, then one output row per store instruction
          // (the lanes write 32 consecutive span positions: contiguous runs of the CNHW plane)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t w4[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float f0 = has ? __uint_as_float(v[32 * h + 8 * j + 2 * e]) : 0.0f;
                float f1 = has ? __uint_as_float(v[32 * h + 8 * j + 2 * e + 1]) : 0.0f;
                if (epi) {
                  f0 = epilogue_one<true, BF>(f0, a.bias, row, 0.0f, nullptr, a.relu);
                  f1 = epilogue_one<true, BF>(f1, a.bias, row, 0.0f, nullptr, a.relu);
                }
                w4[e] = (uint32_t)to16<BF>(f0) | ((uint32_t)to16<BF>(f1) << 16);
              }
              *(uint4*)(stg + lane * 64 + ((j ^ (lane & 3)) * 16)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            }
            __syncwarp();
            const int32_t o = ot[c0 + 32 * h + lane];
            if (o >= 0) {
              const int j = lane >> 3;
              for (int r = 0; r < 32 && row0 + r < a.M; ++r) {
                const uint16_t hv = *(const uint16_t*)(stg + r * 64 + ((j ^ (r & 3)) * 16) + (lane & 7) * 2);
                *(uint16_t*)(a.Y + ((int64_t)(row0 + r) * a.plane + o) * 2) = hv;
              }
            }
          }
          continue;
        }
        if (row0 >= a.M || c0 >= ncol) continue;
        if (coal && c0 + 64 <= ncol) {
          // 16-bit row of 64 values -> staging (16-byte chunks XOR-swizzled by row), then each
          // store instruction writes four whole 128-byte row segments (coalesced)
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float f0 = has ? __uint_as_float(v[8 * j + 2 * e]) : 0.0f;
              float f1 = has ? __uint_as_float(v[8 * j + 2 * e + 1]) : 0.0f;
              if (epi) {
                f0 = epilogue_one<true, BF>(f0, a.bias, row, 0.0f, nullptr, a.relu);
                f1 = epilogue_one<true, BF>(f1, a.bias, row, 0.0f, nullptr, a.relu);
              }
              w4[e] = (uint32_t)to16<BF>(f0) | ((uint32_t)to16<BF>(f1) << 16);
            }
            *(uint4*)(stg + lane * 128 + ((j ^ (lane & 7)) * 16)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + (lane >> 3), j = lane & 7;
            const uint4 d4 = *(const uint4*)(stg + r * 128 + ((j ^ (r & 7)) * 16));
            if (row0 + r < a.M) *(uint4*)(a.Y + ((int64_t)(row0 + r) * a.ldy + n0 + c0) * 2 + j * 16) = d4;
          }
          continue;
        }
        if (row >= a.M) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = c0 + 32 * h;
          if (cc >= ncol) break;
          uint8_t* yp = a.Y + ((int64_t)row * a.ldy + (n0 + cc) * ycs) * 2;
          alignas(16) uint16_t hv[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            float f = has ? __uint_as_float(v[32 * h + c]) : 0.0f;
            if (epi && cc + c < ncol) f = epilogue_one<true, BF>(f, a.bias, row, a.beta, yp + c * ycs * 2, a.relu);
            hv[c] = to16<BF>(f);
          }
          // (compile-time indices into hv: a runtime-bounded loop put hv in local memory, which
          // made the channels-last fp16 conv 68 -> 156 us)
          if (ycs != 1) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (cc + c < ncol) ((uint16_t*)yp)[c * ycs] = hv[c];
          } else if (cc + 32 <= ncol && ((uintptr_t)yp % 16) == 0) {
#pragma unroll
            for (int c = 0; c < 32; c += 8) *(uint4*)(yp + c * 2) = *(const uint4*)(hv + c);
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (cc + c < ncol) ((uint16_t*)yp)[c] = hv[c];
          }
        }
      }
      tm_fence_before();
      __syncwarp();
      if (lane == 0) {
          if (pair && rank == 1) mbar_arrive_remote(map_rank(tempty0 + 8 * acc, 0));
          else mbar_arrive(tempty0 + 8 * acc);
        }
      aph[acc] ^= 1u;
      acc ^= 1;
    }
  }
  tm_fence_before();
  __syncthreads();
  if (CS > 1) cluster_sync_all();  // no peer may still arrive on / multicast into this CTA
  if (warp == 1) {
    if (pair) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

// 3xTF32 operand split of X (fp32 plans on the tcgen05 block executor): X = X_hi + X_lo with
// X_hi = TF32 RN of X and X_lo = TF32 RN of the (exact) remainder, written to two K x ldp
// scratch matrices (ldp a multiple of 4: 16-byte TMA row strides).  Non-finite X: X_lo = 0.
__global__ void __launch_bounds__(256) split_tf32(const float* __restrict__ X, int64_t ldx, float* __restrict__ hi,
                                                  float* __restrict__ lo, int64_t ldp, int64_t K, int64_t N) {
  const int64_t n4 = (N + 3) / 4, total = K * n4;
  const bool vec = ((uintptr_t)X % 16) == 0 && (ldx % 4) == 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / n4, n = (i - k * n4) * 4;
    float x[4];
    if (vec && n + 4 <= N) {
      const float4 v = __ldg((const float4*)(X + k * ldx + n));
      x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) x[c] = n + c < N ? X[k * ldx + n + c] : 0.0f;
    }
    float h[4], l[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      h[c] = tf32_rn_dev(x[c]);
      l[c] = isfinite(h[c]) ? tf32_rn_dev(x[c] - h[c]) : 0.0f;
    }
    *(float4*)(hi + k * ldp + n) = make_float4(h[0], h[1], h[2], h[3]);
    *(float4*)(lo + k * ldp + n) = make_float4(l[0], l[1], l[2], l[3]);
  }
}

// Tail K slices: Y tile = epilogue(sum over slices s = 0 .. tks - 1, in order, of the slices'
// partials) for the ntail tail tiles (tile rounds * ncl + tt: group t % ngroups, N tile t /
// ngroups); 32 x 32 blocks through shared memory.  Y element (row, col) at row ldy + col ycs.
template <int S, bool BF>
__global__ void __launch_bounds__(256) tcg_tailsum(const float* __restrict__ tws, int tks, int ntail, int bnt, int R,
                                                   int64_t tile0, int ngroups, int64_t M, int64_t N,
                                                   uint8_t* __restrict__ Y, int64_t ldy, int64_t ycs,
                                                   const uint8_t* __restrict__ bias, float beta, int relu) {
  __shared__ float tile[32][33];
  const int tt = blockIdx.z;
  const int64_t t = tile0 + tt;
  const int64_t row0 = (t % ngroups) * R + (int64_t)blockIdx.x * 32, col0 = (t / ngroups) * bnt + (int64_t)blockIdx.y * 32;
  const int cl0 = blockIdx.y * 32, rl0 = blockIdx.x * 32;  // within the tile
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int j = ty; j < 32; j += 8) {
    const int cl = cl0 + j;
    float v = 0.0f;
    if (cl < bnt && row0 + tx < M && col0 + j < N) {
      const size_t off = (size_t)cl * R + rl0 + tx;
      v = __ldg(tws + (size_t)tt * bnt * R + off);
      for (int sx = 1; sx < tks; ++sx) v = __fadd_rn(v, __ldg(tws + ((size_t)sx * ntail + tt) * bnt * R + off));
    }
    tile[j][tx] = v;
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const int64_t r = row0 + j, c = col0 + tx;
    if (r >= M || c >= N || cl0 + tx >= bnt) continue;
    uint8_t* yp = Y + (r * ldy + c * ycs) * S;
    const float f = epilogue_one<S == 2, BF>(tile[tx][j], bias, (int)r, beta, yp, relu);
    if constexpr (S == 2) *(uint16_t*)yp = to16<BF>(f);
    else *(float*)yp = f;
  }
}

// tail K slices per tail tile: the idle clusters of the last round share the tail tiles' k-blocks
// (at least 2 k-blocks per slice on average, at most 16 slices)
static int tcg_tail_slices(int64_t ncl, int64_t ntail, int64_t nblk, int64_t ngroups) {
  if (ntail <= 0) return 1;
  const int64_t per = nblk / std::max<int64_t>(1, ngroups);
  const int64_t t = std::min(std::min(ncl / ntail, (int64_t)16), per / 2);
  return t >= 2 ? (int)t : 1;
}

// grid of a persistent cluster launch: whole clusters, at most as many as can be co-resident
template <typename Fn>
static unsigned tcg_grid(Fn fn, cudaLaunchConfig_t cfg, int cs, int64_t ntiles, int sms) {
  int64_t ncl = std::max<int64_t>(1, sms / cs);
  if (cs > 1) {
    int maxc = 0;
    if (cudaOccupancyMaxActiveClusters(&maxc, fn, &cfg) == cudaSuccess && maxc > 0) ncl = std::min<int64_t>(ncl, maxc);
    else cudaGetLastError();
  }
  ncl = std::max<int64_t>(1, std::min<int64_t>(ncl, ntiles));
  return (unsigned)(ncl * cs);
}

static int tcg_launch(const Plan& p, const void* fn_, const CUtensorMap& tmap, const CUtensorMap& tmap2,
                      TcgArgs a, int64_t ntiles, void* stream, std::string& err, const char* what,
                      int threads = 192) {
  const bool tf = p.dtype == SPARSE_F32;
  using TFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcgArgs);
  TFn fn = (TFn)fn_;
  cudaError_t e = ensure_smem_attr(fn, p.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
  const int cs = a.cs;
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.blockDim = dim3((unsigned)threads, 1, 1);
  cfg.dynamicSmemBytes = (size_t)p.smem_bytes;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = (unsigned)cs;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cs > 1 ? 2 : 1;
  cfg.gridDim = dim3((unsigned)cs, 1, 1);
  const int64_t items = a.ks > 1 ? ntiles * a.ks : ntiles;  // (tile, K slice) work items
  cfg.gridDim = dim3(tcg_grid(fn, cfg, cs, items, sms), 1, 1);
  // tail K slices for fp32 (3xTF32: long tiles; measured counter-productive for 16-bit tiles,
  // whose partial-sum pass costs more than the idle clusters save): with fewer tiles than
  // co-resident clusters the grid is sized for the slices, not the tiles
  const bool copies_conv = a.plane > 0 && !a.i2c;  // (its epilogue maps span positions)
  int tks = 1;
  if (tf && a.ks <= 1 && !copies_conv) {
    const int64_t ncl_max = tcg_grid(fn, cfg, cs, INT64_MAX / 4, sms) / cs;
    const int64_t tail = ntiles % ncl_max;
    tks = tcg_tail_slices(ncl_max, tail, a.nblk, a.ngroups);
    // worth it only when the idle time it saves, (1 - 1/tks) of a tile (~1 us per fp32 k-block,
    // measured), exceeds the partial-sum pass (~15 us): C5 at batch 32 - 128 yes (72 k-blocks),
    // BERT 3072 x 768 no (24 k-blocks: 264 -> 272 us with it)
    const int64_t per = a.nblk / std::max<int64_t>(1, a.ngroups);
    if (tks > 1 && per * (tks - 1) / tks < 15) tks = 1;
    if (const char* ev = std::getenv("SRT_TCG_TAIL_KS"))
      if (std::atoi(ev) == 0) tks = 1;
    if (tks > 1 && ntiles < ncl_max) cfg.gridDim = dim3((unsigned)(std::min(ncl_max, ntiles * tks) * cs), 1, 1);
  }
  // split tail: when the tiles do not fill the last round of the persistent clusters (C5 conv:
  // 224 tiles on 74 clusters = 3 rounds + 2 tiles), each last-round tile is cut into sp column
  // slices of whole X boxes (a power of two: 16-bit <= 4, fp32 <= 8), one per otherwise idle
  // cluster; a slice streams the tile's whole W block list with an N = 256 / sp MMA.
  // SRT_TCG_SPLIT_TAIL=0 disables it (A/B); n > 0 caps sp.
  const int64_t ncl = cfg.gridDim.x / cs;
  int cap = (a.i2c || a.ks > 1) ? 1 : (tf ? 8 : 4) / (a.pair ? 2 : 1);  // a slice is >= 1 X box (pair: per CTA)
  if (const char* st = std::getenv("SRT_TCG_SPLIT_TAIL")) cap = std::min(cap, std::max(1, std::atoi(st)));
  a.rounds = (int32_t)(ntiles / ncl);
  a.ntail = (int32_t)(ntiles % ncl);
  a.sp = 1;
  // tail K slices (preferred): the tail tiles' k-blocks spread over the idle clusters, partial
  // sums added in order by tcg_tailsum (SRT_TCG_TAIL_KS=0 disables)
  a.tks = tks > 1 && a.ntail > 0 ? tks : 1;
  if (a.tks > 1 && a.rounds == 0) a.tks = std::max<int>(1, (int)std::min<int64_t>(a.tks, ncl / a.ntail));
  if (a.ntail > 0 && a.tks <= 1)
    while (a.sp * 2 <= cap && (int64_t)a.sp * 2 * a.ntail <= ncl) a.sp *= 2;
  a.np = 256 / a.sp;
  a.idesc_p = (a.idesc & ~(0x3Fu << 17)) | ((uint32_t)(a.np >> 3) << 17);
  const int bnt = a.bn > 0 ? a.bn : 256, R = cs * 128;
  void* tws = nullptr;
  if (a.tks > 1) {
    e = cudaMallocAsync(&tws, (size_t)a.tks * a.ntail * bnt * R * 4, (cudaStream_t)stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cuda_fail(e, "cudaMallocAsync(tail K-slice partials)", err);
    }
    a.tws = (float*)tws;
  }
  struct FreeT {
    void* b;
    void* st;
    ~FreeT() {
      if (b) cudaFreeAsync(b, (cudaStream_t)st);
    }
  } ft{tws, stream};
  // CTA pairs: the W blocks through a 2-D map of 128-byte rows (the 2-SM TMA form signals the
  // pair's rank-0 barrier; the 1-D bulk copy has no such form)
  CUtensorMap tmapA;
  std::memset(&tmapA, 0, sizeof tmapA);
  if (a.pair) {
    auto encode = tensor_map_encoder();
    const int ab = tf ? 32768 : 16384;
    cuuint64_t dims[2] = {32, (cuuint64_t)p.tcp_nsteps * cs * (ab / 128)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32u, (cuuint32_t)(ab / 128)};
    cuuint32_t estr[2] = {1, 1};
    if (!encode || encode(&tmapA, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint8_t*>(p.d_tcp_steps), dims, strides,
                          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      err = "tcgen05 pair: cuTensorMapEncodeTiled (W blocks) failed";
      return SPARSE_EINTERNAL;
    }
  }
  e = cudaLaunchKernelEx(&cfg, fn, tmap, tmap2, tmapA, a);
  if (e != cudaSuccess) return cuda_fail(e, what, err);
  if (a.tks > 1) {
    const int S = tf ? 4 : 2;
    const dim3 grid((unsigned)(R / 32), (unsigned)((bnt + 31) / 32), (unsigned)a.ntail);
    const int64_t tile0 = (int64_t)a.rounds * ncl, ycs = a.ycs > 0 ? a.ycs : 1;
    if (S == 4)
      tcg_tailsum<4, false><<<grid, 256, 0, (cudaStream_t)stream>>>(a.tws, a.tks, a.ntail, bnt, R, tile0, a.ngroups, a.M,
                                                                    a.N, a.Y, a.ldy, ycs, a.bias, a.beta, a.relu);
    else if (p.dtype == SPARSE_BF16)
      tcg_tailsum<2, true><<<grid, 256, 0, (cudaStream_t)stream>>>(a.tws, a.tks, a.ntail, bnt, R, tile0, a.ngroups, a.M,
                                                                   a.N, a.Y, a.ldy, ycs, a.bias, a.beta, a.relu);
    else
      tcg_tailsum<2, false><<<grid, 256, 0, (cudaStream_t)stream>>>(a.tws, a.tks, a.ntail, bnt, R, tile0, a.ngroups, a.M,
                                                                    a.N, a.Y, a.ldy, ycs, a.bias, a.beta, a.relu);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "tail K-slice sum launch", err);
  }
  return SPARSE_OK;
}

// K-sliced tcgen05 tiles: Y = epilogue(sum over slices s = 0 .. ks - 1, in order, of ws[s]); ws is
// column-major per slice ([s][column][row]).  32 x 32 tiles through shared memory: reads along
// the rows, writes along the columns.  fp32 sums, one rounding to the output type.
template <int S, bool BF>
__global__ void __launch_bounds__(256) tcg_ksum(const float* __restrict__ ws, int ks, int64_t M, int64_t N,
                                                uint8_t* __restrict__ Y, int64_t ldy, const uint8_t* __restrict__ bias,
                                                float beta, int relu) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int j = ty; j < 32; j += 8) {
    const int64_t c = c0 + j, r = r0 + tx;
    float v = 0.0f;
    if (c < N && r < M) {
      v = __ldg(ws + c * M + r);
      for (int sx = 1; sx < ks; ++sx) v = __fadd_rn(v, __ldg(ws + ((int64_t)sx * N + c) * M + r));
    }
    tile[j][tx] = v;
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const int64_t r = r0 + j, c = c0 + tx;
    if (r >= M || c >= N) continue;
    uint8_t* yp = Y + (r * ldy + c) * S;
    const float f = epilogue_one<S == 2, BF>(tile[tx][j], bias, (int)r, beta, yp, relu);
    if constexpr (S == 2) *(uint16_t*)yp = to16<BF>(f);
    else *(float*)yp = f;
  }
}

static int launch_tcg(const Plan& p, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy, void* stream,
                      std::string& err, const Epilogue& ep) {
  const bool bf = p.dtype == SPARSE_BF16, tf = p.dtype == SPARSE_F32;
  auto encode = tensor_map_encoder();
  if (!encode) {
    err = "internal: no tensor-map encoder";
    return SPARSE_EINTERNAL;
  }
  DeviceGuard dg(p.device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  const void* Xa = X;
  const void* Xb = nullptr;
  int64_t lda = ldx;
  void* scratch = nullptr;
  bool pooled = false;  // scratch from cudaMallocAsync (3xTF32 split) vs the repack helper
  if (tf) {
    // X_hi / X_lo for the 3xTF32 products, stream ordered
    lda = (N + 3) / 4 * 4;
    const size_t bytes = (size_t)p.K * (size_t)lda * 4;
    cudaError_t e = cudaMallocAsync(&scratch, 2 * bytes, (cudaStream_t)stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cuda_fail(e, "cudaMallocAsync(3xTF32 split)", err);
    }
    pooled = true;
    Xa = scratch;
    Xb = (const uint8_t*)scratch + bytes;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
    const int64_t work = (int64_t)p.K * ((N + 3) / 4);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)sms * 16));
    split_tf32<<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)X, ldx, (float*)scratch, (float*)Xb, lda,
                                                        p.K, N);
    if ((e = cudaGetLastError()) != cudaSuccess) {
      cudaFreeAsync(scratch, (cudaStream_t)stream);
      return cuda_fail(e, "3xTF32 split launch", err);
    }
  } else if (((uintptr_t)X % 16) != 0 || ((ldx * 2) % 16) != 0) {
    const int rc = launch_repack(p.device, p.K, N, 2, X, ldx, &scratch, &lda, stream, err);
    if (rc != SPARSE_OK) return rc;
    Xa = scratch;
  }
  struct Free {
    void* b;
    void* st;
    int dev;
    bool pooled;
    ~Free() {
      if (b && pooled) cudaFreeAsync(b, (cudaStream_t)st);
      else if (b) free_repack(dev, b, st);
    }
  } fr{scratch, stream, p.device, pooled};
  const int es = tf ? 4 : 2;
  CUtensorMap tmap, tmap2;
  std::memset(&tmap, 0, sizeof tmap);
  std::memset(&tmap2, 0, sizeof tmap2);
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)p.K};
  cuuint64_t strides[1] = {(cuuint64_t)(lda * es)};
  cuuint32_t box[2] = {tf ? 32u : 64u, tf ? 32u : 64u};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = tf ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                               : bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  // MN-major TF32 operands take the 32-byte-chunk 128-byte swizzle (UMMA layout type 1)
  const CUtensorMapSwizzle swz = tf ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = encode(&tmap, dt, 2, const_cast<void*>(Xa), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS && tf)
    r = encode(&tmap2, dt, 2, const_cast<void*>(Xb), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "tcgen05 blocks: cuTensorMapEncodeTiled failed";
    return SPARSE_EINTERNAL;
  }
  TcgArgs a;
  std::memset(&a, 0, sizeof a);
  a.blocks = p.d_tcp_steps;
  a.meta = p.d_tcp_step_off;
  a.nblk = (int32_t)p.tcp_nsteps;
  a.Y = (uint8_t*)Y;
  a.ldy = ldy;
  a.N = N;
  a.M = p.M;
  a.ngroups = p.tcg_ngroups;
  a.cs = p.tcg_cs;
  a.stages = p.stages;
  if (const char* dbg = std::getenv("SRT_TCG_DBG")) a.dbg = std::atoi(dbg);
  a.bias = (const uint8_t*)ep.bias;
  a.beta = ep.beta;
  a.relu = ep.relu;
  // instruction descriptor: D fp32, A / B fp16 (0), bf16 (1) or tf32 (2), A K-major, B MN-major,
  // N = 256, M = 128
  const uint32_t fmt = tf ? 2u : bf ? 1u : 0u;
  a.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 16) | ((256u >> 3) << 17) |
            (((p.tcg_pair ? 256u : 128u) >> 4) << 24);
  a.pair = p.tcg_pair;
  const int64_t ntiles = (int64_t)p.tcg_ngroups * ((N + 255) / 256);
  const bool pr = p.tcg_pair != 0;
  const void* fn = tf ? (pr ? (const void*)spmm_tcg_kernel<false, false, true, true>
                            : (const void*)spmm_tcg_kernel<false, false, true, false>)
                 : bf ? (pr ? (const void*)spmm_tcg_kernel<true, false, false, true>
                            : (const void*)spmm_tcg_kernel<true, false, false, false>)
                      : (pr ? (const void*)spmm_tcg_kernel<false, false, false, true>
                            : (const void*)spmm_tcg_kernel<false, false, false, false>);
  if (p.tcg_ks <= 1)
    return tcg_launch(p, fn, tmap, tmap2, a, ntiles, stream, err, "tcgen05 block launch", tf ? 320 : 192);
  // K slices: fp32 partials in a stream-ordered workspace, then tcg_ksum (ordered sum + epilogue)
  if ((N + 31) / 32 > 65535 || (p.M + 31) / 32 > INT32_MAX) {
    err = "tcgen05 K slices: N too large for the slice sum (use k_split = 1)";
    return SPARSE_EUNSUPPORTED;
  }
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, (size_t)p.tcg_ks * (size_t)N * (size_t)p.M * 4, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(e, "cudaMallocAsync(K-slice partials)", err);
  }
  struct FreeWs {
    void* b;
    void* st;
    ~FreeWs() { cudaFreeAsync(b, (cudaStream_t)st); }
  } fw{ws, stream};
  a.ks = p.tcg_ks;
  a.ws = (float*)ws;
  a.bias = nullptr, a.beta = 0.0f, a.relu = 0;
  int rc = tcg_launch(p, fn, tmap, tmap2, a, ntiles, stream, err, "tcgen05 block launch (K slices)", tf ? 320 : 192);
  if (rc != SPARSE_OK) return rc;
  const dim3 grid((unsigned)((p.M + 31) / 32), (unsigned)((N + 31) / 32));
  if (tf)
    tcg_ksum<4, false><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)ws, p.tcg_ks, p.M, N, (uint8_t*)Y, ldy,
                                                               (const uint8_t*)ep.bias, ep.beta, ep.relu);
  else if (bf)
    tcg_ksum<2, true><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)ws, p.tcg_ks, p.M, N, (uint8_t*)Y, ldy,
                                                              (const uint8_t*)ep.bias, ep.beta, ep.relu);
  else
    tcg_ksum<2, false><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)ws, p.tcg_ks, p.M, N, (uint8_t*)Y, ldy,
                                                               (const uint8_t*)ep.bias, ep.beta, ep.relu);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "K-slice sum launch", err);
  return SPARSE_OK;
}

// Conv on the tcgen05 block executor (conv_kernel 5): the interleaved copies pre-pass (pitch a
// multiple of 8 elements), then spmm_tcg_kernel<CONV> over the span of the copies.
// Conv on the tcgen05 block executor through im2col TMA: the input is packed once CNHW -> NHWC
// (fp32: split into TF32 halves), then every k-block (64 / 32 channels, tap) of every tile is ONE
// im2col box per operand: 256 (pair: 128 per CTA) consecutive output pixels x the channel group,
// the zero padding of P:215 done by the TMA engine (pixels outside the image read as zero).  No
// shifted copies, no halo positions; the output tile is 256 consecutive pixels of the CNHW
// plane, stored like an SpMM tile (ldy = plane).
static int launch_conv_i2c(const Plan& p, int64_t batch, const void* x, void* y, void* stream, std::string& err,
                           const Epilogue& ep, bool nhwc = false) {
  const bool bf = p.dtype == SPARSE_BF16, tf = p.dtype == SPARSE_F32;
  const int S = tf ? 4 : 2, BK = tf ? 32 : 64;
  auto encode = tensor_map_encoder_im2col();
  if (!encode) {
    err = "internal: no im2col tensor-map encoder";
    return SPARSE_EINTERNAL;
  }
  const int64_t plane = batch * (int64_t)p.h * p.w;
  DeviceGuard dg(p.device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  void* xn = nullptr;  // NHWC input (fp32: X_hi, then X_lo)
  const void* xn_user = nullptr;  // 16-bit NHWC input: read in place
  const size_t nb = (size_t)plane * p.c_in * S;
  cudaError_t e = cudaMallocAsync(&xn, (nhwc && !tf) ? 16 : (tf ? 2 * nb : nb), (cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(e, "cudaMallocAsync(conv NHWC)", err);
  }
  struct Free {
    void* b;
    void* st;
    ~Free() { cudaFreeAsync(b, (cudaStream_t)st); }
  } fr{xn, stream};
  if (nhwc) {  // the input is NHWC already: 16-bit needs nothing, fp32 only the TF32 split
    if (tf) {
      const int64_t work = plane * ((p.c_in + 3) / 4);
      const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)148 * 16));
      split_tf32<<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)x, p.c_in, (float*)xn,
                                                          (float*)((uint8_t*)xn + nb), p.c_in, plane, p.c_in);
      if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "3xTF32 split launch", err);
    } else {
      xn_user = x;
    }
  } else {
    const dim3 grid((unsigned)((plane + 127) / 128), (unsigned)((p.c_in + 31) / 32));
    if (tf)
      nhwc_pack<float, true><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)x, (float*)xn,
                                                                     (float*)((uint8_t*)xn + nb), p.c_in, plane);
    else
      nhwc_pack<uint16_t, false><<<grid, 256, 0, (cudaStream_t)stream>>>((const uint16_t*)x, (uint16_t*)xn, nullptr,
                                                                         p.c_in, plane);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "NHWC pack launch", err);
  }
  // tile width: fp32 (3xTF32) fills the rounds of the persistent clusters (cost ~ rounds, the
  // tail counted as K slices where it leaves >= 2 clusters per tile, x the operand bytes of a
  // k-block; C5: 240 -> 229 to 218 us); 16-bit plans keep 256 (240 measured 68 -> 73 us).
  // SRT_CONV_BN overrides; a multiple of 16 (M = 256)
  const int cs = p.tcg_cs;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
  int bn = 256;
  {
    const int64_t ncl = std::max(1, sms / cs);
    int64_t best = INT64_MAX;
    for (int w = 256; w >= (tf ? 128 : 256); w -= 16) {
      if ((w / cs) % 8) continue;  // a CTA's pixel rows: whole 8-row (1 KB) swizzle atoms
      const int64_t tiles = (int64_t)p.tcg_ngroups * ((plane + w - 1) / w);
      // rounds of whole tiles, the tail as K slices when it leaves >= 2 clusters per tile
      const int64_t full = tiles / ncl, tail = tiles % ncl;
      const int tks = tcg_tail_slices(ncl, tail, p.tcp_nsteps, p.tcg_ngroups);
      const int64_t r100 = full * 100 + (tail ? (tks > 1 ? 100 / tks + 15 : 100) : 0);
      // a k-block's time ~ the operand bytes into the SM (measured bound, DESIGN 5d): the W
      // block(s) + this CTA's pixel rows of 128 bytes per operand
      const int64_t ops = tf ? 2 : 1, abytes = 16384 * ops, bbytes = (int64_t)(p.tcg_pair ? w / 2 : w) * 128 * ops;
      const int64_t cost = r100 * (abytes + bbytes);
      if (cost < best) best = cost, bn = w;
    }
    if (const char* ev = std::getenv("SRT_CONV_BN")) {
      const int v = std::atoi(ev);
      if (v >= 16 * cs && v <= 256 && v % 16 == 0 && (v / cs) % 8 == 0) bn = v;
    }
  }
  const int pix = bn / cs;
  CUtensorMap tmap, tmap2;
  std::memset(&tmap, 0, sizeof tmap);
  std::memset(&tmap2, 0, sizeof tmap2);
  cuuint64_t dims[4] = {(cuuint64_t)p.c_in, (cuuint64_t)p.w, (cuuint64_t)p.h, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)p.c_in * S, (cuuint64_t)p.c_in * S * p.w, (cuuint64_t)p.c_in * S * p.w * p.h};
  const int lower[2] = {-1, -1}, upper[2] = {-1, -1};  // 3 x 3, padding 1, stride 1 (W, H)
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUtensorMapDataType dt = tf ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                               : bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUresult r = encode(&tmap, dt, 4, xn_user ? const_cast<void*>(xn_user) : xn, dims, strides, lower, upper,
                      (cuuint32_t)BK, (cuuint32_t)pix, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS && tf)
    r = encode(&tmap2, dt, 4, (uint8_t*)xn + nb, dims, strides, lower, upper, (cuuint32_t)BK, (cuuint32_t)pix, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "conv (tcgen05, im2col): cuTensorMapEncodeIm2col failed";
    return SPARSE_EINTERNAL;
  }
  TcgArgs a;
  std::memset(&a, 0, sizeof a);
  a.blocks = p.d_tcp_steps;
  a.meta = p.d_tcp_step_off;
  a.nblk = (int32_t)p.tcp_nsteps;
  a.Y = (uint8_t*)y;
  a.ldy = nhwc ? 1 : plane;  // CNHW: Y[channel][pixel]; NHWC: Y[pixel][channel]
  a.ycs = nhwc ? p.M : 1;
  a.N = plane;
  a.M = p.M;
  a.ngroups = p.tcg_ngroups;
  a.cs = cs;
  a.stages = p.stages;
  if (const char* dbg = std::getenv("SRT_TCG_DBG")) a.dbg = std::atoi(dbg);
  a.bias = (const uint8_t*)ep.bias;
  a.beta = ep.beta;
  a.relu = ep.relu;
  // D fp32, A / B fp16 (0), bf16 (1) or tf32 (2), both K-major, N = 256, M = 128 (pair: 256)
  const uint32_t fmt = tf ? 2u : bf ? 1u : 0u;
  a.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (((uint32_t)bn >> 3) << 17) |
            (((p.tcg_pair ? 256u : 128u) >> 4) << 24);
  a.pair = p.tcg_pair;
  a.i2c = 1;
  a.i2c_pix = pix;
  a.bn = bn;
  a.H = p.h;
  a.W = p.w;
  a.Bt = (int32_t)batch;
  a.plane = plane;
  const int64_t ntiles = (int64_t)p.tcg_ngroups * ((plane + bn - 1) / bn);
  const bool pr = p.tcg_pair != 0;
  const void* fn = tf ? (pr ? (const void*)spmm_tcg_kernel<false, true, true, true>
                            : (const void*)spmm_tcg_kernel<false, true, true, false>)
                 : bf ? (pr ? (const void*)spmm_tcg_kernel<true, true, false, true>
                            : (const void*)spmm_tcg_kernel<true, true, false, false>)
                      : (pr ? (const void*)spmm_tcg_kernel<false, true, false, true>
                            : (const void*)spmm_tcg_kernel<false, true, false, false>);
  return tcg_launch(p, fn, tmap, tmap2, a, ntiles, stream, err, "conv3x3 (tcgen05, im2col) launch", tf ? 320 : 192);
}

static int launch_conv_tcg(const Plan& p, int64_t batch, const void* x, void* y, void* stream, std::string& err,
                           const Epilogue& ep) {
  const bool bf = p.dtype == SPARSE_BF16, tf = p.dtype == SPARSE_F32;
  const int S = tf ? 4 : 2;
  {  // im2col TMA (default; SRT_CONV_IM2COL=0 selects the interleaved dx-shifted copies)
    const char* ev = std::getenv("SRT_CONV_IM2COL");
    const bool rows16 = ((int64_t)p.c_in * S) % 16 == 0;  // TMA: 16-byte pixel strides
    if ((!ev || std::atoi(ev) != 0) && rows16 && batch * (int64_t)p.h * p.w < INT32_MAX)
      return launch_conv_i2c(p, batch, x, y, stream, err, ep);
  }
  auto encode = tensor_map_encoder();
  if (!encode) {
    err = "internal: no tensor-map encoder";
    return SPARSE_EINTERNAL;
  }
  const int g = p.tcg_g, P = g * p.w, Sg = (p.h + 2) * P;
  const int64_t ngroups = (batch + g - 1) / g, span = ngroups * Sg;
  if (span > INT32_MAX - 4096 || batch > INT32_MAX / 2) {
    err = "conv (tcgen05): batch too large for one launch";
    return SPARSE_EUNSUPPORTED;
  }
  DeviceGuard dg(p.device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  void* xp = nullptr;  // the copies (3xTF32: the X_hi copies, then the X_lo copies)
  const size_t cbytes = (size_t)3 * p.c_in * span * S;
  cudaError_t e = cudaMallocAsync(&xp, tf ? 2 * cbytes : cbytes, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(e, "cudaMallocAsync(conv copies)", err);
  }
  struct Free {
    void* b;
    void* st;
    ~Free() { cudaFreeAsync(b, (cudaStream_t)st); }
  } fr{xp, stream};
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
  {
    const int blk = g * p.h * p.w;
    const int pp = (int)std::max<int64_t>(1, std::min<int64_t>(16, (96 * 1024) / ((int64_t)blk * S)));
    const size_t psm = (size_t)pp * blk * S;
    const int64_t nblk = (int64_t)p.c_in * ngroups;
    const unsigned pg = (unsigned)std::min<int64_t>((nblk + pp - 1) / pp, (int64_t)sms * 8);
    if (tf) {
      if ((e = ensure_smem_attr(il_pad_input<float>, (int)psm)) != cudaSuccess)
        return cuda_fail(e, "cudaFuncSetAttribute(il pad)", err);
      il_pad_input<float><<<pg, 256, psm, (cudaStream_t)stream>>>((const float*)x, (float*)xp, p.c_in, (int)batch,
                                                                  p.h, p.w, g, (int)ngroups, Sg, pp, nullptr,
                                                                  (float*)((uint8_t*)xp + cbytes));
    } else {
      if ((e = ensure_smem_attr(il_pad_input<uint16_t>, (int)psm)) != cudaSuccess)
        return cuda_fail(e, "cudaFuncSetAttribute(il pad)", err);
      il_pad_input<uint16_t><<<pg, 256, psm, (cudaStream_t)stream>>>((const uint16_t*)x, (uint16_t*)xp, p.c_in,
                                                                     (int)batch, p.h, p.w, g, (int)ngroups, Sg,
                                                                     pp, nullptr);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "il pad launch", err);
  }
  CUtensorMap tmap, tmap2;
  std::memset(&tmap, 0, sizeof tmap);
  std::memset(&tmap2, 0, sizeof tmap2);
  cuuint64_t dims[3] = {(cuuint64_t)span, (cuuint64_t)p.c_in, 3};
  cuuint64_t strides[2] = {(cuuint64_t)(span * S), (cuuint64_t)(span * S * p.c_in)};
  // 16-bit: 64 positions x 64 channels, 128-byte swizzle; 3xTF32: 32 x 32 fp32, 32-byte-chunk
  // 128-byte swizzle (the MN-major TF32 operand layout, as the SpMM form)
  cuuint32_t box[3] = {tf ? 32u : 64u, tf ? 32u : 64u, 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapDataType dt = tf ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                               : bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const CUtensorMapSwizzle swz = tf ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = encode(&tmap, dt, 3, xp, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS && tf)
    r = encode(&tmap2, dt, 3, (uint8_t*)xp + cbytes, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "conv (tcgen05): cuTensorMapEncodeTiled failed";
    return SPARSE_EINTERNAL;
  }
  TcgArgs a;
  std::memset(&a, 0, sizeof a);
  a.blocks = p.d_tcp_steps;
  a.meta = p.d_tcp_step_off;
  a.nblk = (int32_t)p.tcp_nsteps;
  a.Y = (uint8_t*)y;
  a.ldy = 0;
  a.N = span;
  a.M = p.M;
  a.ngroups = p.tcg_ngroups;
  a.cs = p.tcg_cs;
  a.stages = p.stages;
  if (const char* dbg = std::getenv("SRT_TCG_DBG")) a.dbg = std::atoi(dbg);
  a.bias = (const uint8_t*)ep.bias;
  a.beta = ep.beta;
  a.relu = ep.relu;
  const uint32_t fmt = tf ? 2u : bf ? 1u : 0u;
  a.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 16) | ((256u >> 3) << 17) |
            (((p.tcg_pair ? 256u : 128u) >> 4) << 24);
  a.pair = p.tcg_pair;
  a.P = P;
  a.g = g;
  a.Sg = Sg;
  a.H = p.h;
  a.W = p.w;
  a.ncb = p.tcg_ncb;
  a.Bt = (int32_t)batch;
  a.plane = batch * (int64_t)p.h * p.w;
  const int64_t ntiles = (int64_t)p.tcg_ngroups * ((span + 255) / 256);
  const bool pr = p.tcg_pair != 0;
  const void* fn = tf ? (pr ? (const void*)spmm_tcg_kernel<false, true, true, true>
                            : (const void*)spmm_tcg_kernel<false, true, true, false>)
                 : bf ? (pr ? (const void*)spmm_tcg_kernel<true, true, false, true>
                            : (const void*)spmm_tcg_kernel<true, true, false, false>)
                      : (pr ? (const void*)spmm_tcg_kernel<false, true, false, true>
                            : (const void*)spmm_tcg_kernel<false, true, false, false>);
  return tcg_launch(p, fn, tmap, tmap2, a, ntiles, stream, err, "conv3x3 (tcgen05) launch", tf ? 320 : 192);
}

int launch_spmm(const Plan& p, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy,
                void* stream, std::string& err, const Epilogue& ep) {
  if (p.executor == 3) return launch_tcp(p, N, X, ldx, Y, ldy, stream, err, ep);
  if (p.executor == 4) return launch_tcg(p, N, X, ldx, Y, ldy, stream, err, ep);
  const bool f16 = p.dtype != SPARSE_F32;  // 16-bit X / Y (fp16 or bf16: TMA copies the bits)
  const int S = f16 ? 2 : 4;
  SpmmFn fn = p.dtype == SPARSE_BF16 ? pick_spmm<true, true>(p.R, p.gk, p.tm)
            : f16 ? pick_spmm<true>(p.R, p.gk, p.tm) : pick_spmm<false>(p.R, p.gk, p.tm);
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
  a.blk_bytes = p.max_blk_bytes;
  a.bar_off = p.smem_bytes - 256;
  a.bias = (const uint8_t*)ep.bias;
  a.beta = ep.beta;
  a.relu = ep.relu;
  const int smem = p.smem_bytes;
  const bool vec_x = ((uintptr_t)X % 16 == 0) && ((ldx * S) % 16 == 0);
  a.vec_y = ((uintptr_t)Y % 16 == 0) && ((ldy * S) % 16 == 0);
  a.npanels = p.npanels;
  auto encode = tensor_map_encoder();
  const int threads = p.warps * 32;
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
  a.tcws = nullptr;
  a.ws_row = nullptr;
  a.ldws = 0;
  float* tcws = nullptr;
  if (p.tc_ntiles > 0) {
    // dense 16 x 16 tiles on the tensor cores -> fp32 workspace (stream ordered)
    const int64_t ldws = (N + 3) / 4 * 4;  // float2 stores stay 8-byte aligned
    e = cudaMallocAsync((void**)&tcws, (size_t)p.tc_nrb * 16 * ldws * 4, (cudaStream_t)stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cuda_fail(e, "cudaMallocAsync(tensor-core workspace)", err);
    }
    TcArgs t;
    t.A = p.d_tc_a;
    t.rb = p.d_tc_rb;
    t.tile_begin = p.d_tc_tile_begin;
    t.cb = p.d_tc_cb;
    t.X = (const uint8_t*)X;
    t.ws = tcws;
    t.ldx = ldx;
    t.ldws = ldws;
    t.N = N;
    t.K = p.K;
    t.vec_x = vec_x ? 1 : 0;
    const int cols = N >= 2048 ? 512 : 128;
    auto tc_fn = cols == 512 ? spmm_tc_kernel<512> : spmm_tc_kernel<128>;
    const int64_t nblk = (N + cols - 1) / cols;
    const size_t tc_smem = 2 * 16 * (cols + 8) * 2;
    e = ensure_smem_attr(tc_fn, (int)tc_smem);
    if (e != cudaSuccess) {
      cudaFreeAsync(tcws, (cudaStream_t)stream);
      return cuda_fail(e, "cudaFuncSetAttribute(tensor-core kernel)", err);
    }
    for (int64_t b0 = 0; b0 < nblk; b0 += 65535) {
      const int64_t nb = std::min<int64_t>(65535, nblk - b0);
      t.X = (const uint8_t*)X + b0 * cols * S;
      t.ws = tcws + b0 * cols;
      t.N = N - b0 * cols;
      tc_fn<<<dim3((unsigned)p.tc_nrb, (unsigned)nb), 128, tc_smem, (cudaStream_t)stream>>>(t);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFreeAsync(tcws, (cudaStream_t)stream);
      return cuda_fail(e, "tensor-core sub-block launch", err);
    }
    a.tcws = tcws;
    a.ws_row = p.d_ws_row;
    a.ldws = ldws;
  }
  struct WsFree {
    float* w;
    void* st;
    ~WsFree() {
      if (w) cudaFreeAsync(w, (cudaStream_t)st);
    }
  } ws_free{tcws, stream};
  if (p.ps == 1) {
    // plan in kernel parameters (constant bank): X through TMA only
    a.X = (const uint8_t*)X;
    a.Y = (uint8_t*)Y;
    a.N = N;
    a.cm = 1;
    CUtensorMap tmap;
    make_map(tmap);
    if (!a.use_tma) {
      err = "plan_source = 1 needs the TMA path (16-byte aligned X)";
      return SPARSE_EINTERNAL;
    }
    using PFn = void (*)(const CUtensorMap, const SpmmArgs, const ParamPlan);
    PFn pf = nullptr;
    const bool bf = p.dtype == SPARSE_BF16;
#define SRT_PP(RR) \
    if (p.R == RR) pf = bf ? spmm_param_kernel<RR, true, true> : f16 ? spmm_param_kernel<RR, true> : spmm_param_kernel<RR, false>;
    SRT_PP(1) SRT_PP(2) SRT_PP(4) SRT_PP(8)
#undef SRT_PP
    if (!pf || p.blob.size() > sizeof(ParamPlan)) {
      err = "internal: no parameter-plan kernel instance / plan too large";
      return SPARSE_EINTERNAL;
    }
    if ((e = ensure_smem_attr(pf, smem)) != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
    static thread_local ParamPlan pp;  // 30 KB: not on the host stack
    std::memcpy(&pp, p.blob.data(), p.blob.size());
    const int64_t ntiles = (int64_t)p.npanels * ntn;
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pf, threads, smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    cudaGetLastError();
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sms * per_sm)), 1, 1);
    cfg.blockDim = dim3((unsigned)threads, 1, 1);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, pf, tmap, a, pp);
    if (e != cudaSuccess) return cuda_fail(e, "spmm (parameter plan) launch", err);
    return SPARSE_OK;
  }
  if (p.ks == 1) {
    // persistent: one wave of CTAs (clusters of cm CTAs when X is multicast), each walking
    // tiles (panel group, N tile) cluster_id + j * clusters
    a.X = (const uint8_t*)X;
    a.Y = (uint8_t*)Y;
    a.N = N;
    a.cm = p.cm;
    CUtensorMap tmap;
    make_map(tmap);
    if (!a.use_tma && p.cm > 1) {
      err = "internal: x_multicast needs the TMA path (16-byte aligned X)";
      return SPARSE_EINTERNAL;
    }
    const int64_t ntiles = (int64_t)(p.npanels / p.cm) * ntn;
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.blockDim = dim3((unsigned)threads, 1, 1);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)p.cm;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see kernel)
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (p.grid_cache <= 0) {  // resident clusters (CTAs) in one wave; cached per plan
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
      int per_sm = 1;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
      if (e != cudaSuccess || per_sm < 1) per_sm = 1;
      int64_t clusters = (int64_t)sms * per_sm / p.cm;
      if (p.cm > 1) {
        int nc = 0;
        cfg.gridDim = dim3((unsigned)(p.cm * clusters), 1, 1);
        if (cudaOccupancyMaxActiveClusters(&nc, (const void*)fn, &cfg) == cudaSuccess && nc > 0)
          clusters = nc;
        cudaGetLastError();
      }
      p.grid_cache = (int32_t)std::max<int64_t>(1, clusters);
    }
    const int64_t clusters = std::max<int64_t>(1, std::min<int64_t>(ntiles, p.grid_cache));
    cfg.gridDim = dim3((unsigned)(clusters * p.cm), 1, 1);
    e = cudaLaunchKernelEx(&cfg, fn, tmap, a);
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
    a.tcws = tcws ? tcws + c0 : nullptr;
    CUtensorMap tmap;
    make_map(tmap);
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    a.cm = 1;
    cfg.gridDim = dim3((unsigned)(p.npanels * p.ks), (unsigned)nt, 1);
    cfg.blockDim = dim3((unsigned)threads, 1, 1);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)p.ks;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, fn, tmap, a);
    if (e != cudaSuccess) return cuda_fail(e, "spmm launch", err);
  }
  return SPARSE_OK;
}

// Interleaved conv (conv3x3_il_kernel): the copies pre-pass into a stream-ordered scratch, then
// one persistent wave (programmatic dependent launch after the pre-pass).
static int launch_conv_il(const Plan& p, int64_t batch, const void* x, void* y, void* stream,
                          std::string& err, const Epilogue& ep) {
  const bool f16 = p.dtype != SPARSE_F32, bf = p.dtype == SPARSE_BF16;
  const int S = f16 ? 2 : 4;
  using IlFn = void (*)(const CUtensorMap, const IlArgs);
  IlFn fn = nullptr;
#define SRT_I(RR) \
  if (p.R == RR) fn = bf ? conv3x3_il_kernel<RR, true, true> : f16 ? conv3x3_il_kernel<RR, true> : conv3x3_il_kernel<RR, false>;
  SRT_I(1) SRT_I(2) SRT_I(4) SRT_I(8)
#undef SRT_I
  auto encode = tensor_map_encoder();
  if (!fn || !encode) {
    err = "internal: no interleaved conv kernel instance / tensor-map encoder";
    return SPARSE_EINTERNAL;
  }
  if (batch > INT32_MAX / 2) {
    err = "batch too large";
    return SPARSE_EUNSUPPORTED;
  }
  const int g = p.il_g, P = g * p.w, Sg = (p.h + 2) * P;
  const int64_t ngroups = (batch + g - 1) / g, span = ngroups * Sg;
  if (span > INT32_MAX - 4096) {
    err = "interleaved conv: batch too large for one launch";
    return SPARSE_EUNSUPPORTED;
  }
  DeviceGuard dg(p.device);
  if (dg.st != cudaSuccess) return cuda_fail(dg.st, "cudaSetDevice", err);
  cudaError_t e = ensure_smem_attr(fn, p.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
  // scratch: the three copies, then one ready counter per image group (overlap mode)
  const size_t copies_bytes = ((size_t)(3 * p.c_in * span * S) + 255) / 256 * 256;
  void* xp = nullptr;
  e = cudaMallocAsync(&xp, copies_bytes + (size_t)ngroups * 4, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(e, "cudaMallocAsync(conv copies)", err);
  }
  struct Free {
    void* b;
    void* st;
    ~Free() { cudaFreeAsync(b, (cudaStream_t)st); }
  } fr{xp, stream};
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
  uint32_t* ready = nullptr;
  {
    // Overlap (opt-in, SPARSERT_CONV_OVERLAP=1): the pre-pass runs as one persistent CTA per SM
    // next to the conv kernel's CTA (programmatic dependent launch; per-group ready counters)
    // when both fit in one SM's shared memory.  Measured slower on C5 (one
    // pre-pass CTA per SM needs ~250 us and competes with the conv kernel), so the default is
    // the sequential form: the pre-pass alone at full width, then the conv kernel.
    const int blk = g * p.h * p.w;
    const char* ov = getenv("SPARSERT_CONV_OVERLAP");
    const int64_t budget = 227 * 1024 - (int64_t)p.smem_bytes - 2048;
    int pp = (int)std::min<int64_t>(16, budget / ((int64_t)blk * S));
    const bool overlap = ov && ov[0] == '1' && pp >= 1;
    if (!overlap) pp = (int)std::max<int64_t>(1, std::min<int64_t>(16, (96 * 1024) / ((int64_t)blk * S)));
    const size_t psm = (size_t)pp * blk * S;
    const int64_t nblk = (int64_t)p.c_in * ngroups;
    const unsigned pg = (unsigned)std::min<int64_t>((nblk + pp - 1) / pp, overlap ? (int64_t)sms : (int64_t)sms * 8);
    if (overlap) {
      ready = (uint32_t*)((uint8_t*)xp + copies_bytes);
      if ((e = cudaMemsetAsync(ready, 0, (size_t)ngroups * 4, (cudaStream_t)stream)) != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync(ready)", err);
    }
    if (f16) {
      if ((e = ensure_smem_attr(il_pad_input<uint16_t>, (int)psm)) != cudaSuccess)
        return cuda_fail(e, "cudaFuncSetAttribute(il pad)", err);
      il_pad_input<uint16_t><<<pg, 256, psm, (cudaStream_t)stream>>>((const uint16_t*)x, (uint16_t*)xp, p.c_in,
                                                                     (int)batch, p.h, p.w, g, (int)ngroups, Sg, pp,
                                                                     ready);
    } else {
      if ((e = ensure_smem_attr(il_pad_input<float>, (int)psm)) != cudaSuccess)
        return cuda_fail(e, "cudaFuncSetAttribute(il pad)", err);
      il_pad_input<float><<<pg, 256, psm, (cudaStream_t)stream>>>((const float*)x, (float*)xp, p.c_in, (int)batch,
                                                                  p.h, p.w, g, (int)ngroups, Sg, pp, ready);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "il pad launch", err);
  }
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof tmap);
  cuuint64_t dims[3] = {(cuuint64_t)span, (cuuint64_t)p.c_in, 3};
  cuuint64_t strides[2] = {(cuuint64_t)(span * S), (cuuint64_t)(span * S * p.c_in)};
  cuuint32_t box[3] = {(cuuint32_t)p.il_lc, (cuuint32_t)p.cc, 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(&tmap, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, xp, dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "interleaved conv: cuTensorMapEncodeTiled failed";
    return SPARSE_EINTERNAL;
  }
  IlArgs a;
  a.blob = p.d_blob;
  a.blk_off = p.d_blk_off;
  a.row_id = p.d_row_id;
  a.y = (uint8_t*)y;
  a.npos = ngroups * p.h * P;
  a.plane = batch * (int64_t)p.h * p.w;
  a.H = p.h;
  a.W = p.w;
  a.P = P;
  a.g = g;
  a.Bt = (int32_t)batch;
  a.Sg = Sg;
  a.cc = p.cc;
  a.nchunks = p.nchunks;
  a.Mp = p.Mp;
  a.npanels = p.npanels;
  a.stages = p.stages;
  a.stage_bytes = p.il_stage_bytes;
  a.lc = p.il_lc;
  a.cs = p.conv_cs;
  a.blk_at = p.il_blk_at;
  a.hdr_bytes = p.hdr_bytes;
  a.bar_off = p.smem_bytes - 256;
  a.bias = (const uint8_t*)ep.bias;
  a.beta = ep.beta;
  a.relu = ep.relu;
  a.ready = ready;
  a.ready_target = (uint32_t)p.c_in;
  a.ngroups = (int32_t)ngroups;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, p.warps * 32, p.smem_bytes) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  cudaGetLastError();
  const int64_t ntot = (int64_t)p.npanels * ((a.npos + 127) / 128);
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ntot, (int64_t)sms * per_sm)), 1, 1);
  cfg.blockDim = dim3((unsigned)(p.warps * 32), 1, 1);
  cfg.dynamicSmemBytes = (size_t)p.smem_bytes;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, fn, tmap, a);
  if (e != cudaSuccess) return cuda_fail(e, "conv3x3 (interleaved) launch", err);
  return SPARSE_OK;
}

// Channels-last conv directly on the tcgen05 block executor's im2col path: x NHWC is what the
// im2col TMA reads (16-bit: in place; fp32: split into TF32 halves), y NHWC is written by the
// epilogue with column stride M.  SPARSE_EUNSUPPORTED when the plan is not eligible (the caller
// then transposes around launch_conv3x3).
int launch_conv3x3_nhwc(const Plan& p, int64_t batch, const void* x, void* y, void* stream, std::string& err) {
  const int S = p.dtype == SPARSE_F32 ? 4 : 2;
  const char* ev = std::getenv("SRT_CONV_IM2COL");
  if (p.executor != 4 || (ev && std::atoi(ev) == 0) || ((int64_t)p.c_in * S) % 16 != 0 || ((uintptr_t)x % 16) != 0 ||
      batch * (int64_t)p.h * p.w >= INT32_MAX)
    return SPARSE_EUNSUPPORTED;
  Epilogue ep;
  return launch_conv_i2c(p, batch, x, y, stream, err, ep, true);
}

int launch_conv3x3(const Plan& p, int64_t batch, const void* x, void* y, void* stream,
                   std::string& err, const Epilogue& ep) {
  const bool f16 = p.dtype != SPARSE_F32;  // 16-bit data (bf16 plans always take the TMA-fed kernel)
  ConvFn fn = p.conv_vec ? (f16 ? pick_conv_vec<true>(p.R) : pick_conv_vec<false>(p.R))
                        : (f16 ? pick_conv<true>(p.R, p.C) : pick_conv<false>(p.R, p.C));
  if (p.executor == 4) return launch_conv_tcg(p, batch, x, y, stream, err, ep);
  if (p.conv_vec == 4) return launch_conv_il(p, batch, x, y, stream, err, ep);
  if (!fn && p.conv_vec != 2) {
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
  a.bands = p.conv_vec ? (p.h + p.conv_rb - 1) / p.conv_rb : p.h / p.conv_rb;
  a.cs = p.conv_cs;
  a.bias = (const uint8_t*)ep.bias;
  a.beta = ep.beta;
  a.relu = ep.relu;
  a.npanels = p.npanels;
  a.stages = p.stages;
  if (p.conv_vec == 2) {
    a.stage_bytes = (a.stage_bytes + 127) & ~127;  // TMA destinations 128-byte aligned (inspector)
    // TMA-fed kernel: width-pad the input into a stream-ordered scratch, then one persistent
    // wave of CTAs (programmatic dependent launch after the pad kernel)
    using TmaFn = void (*)(const CUtensorMap, const ConvArgs);
    TmaFn tf = nullptr;
    const bool bf = p.dtype == SPARSE_BF16;
#define SRT_T(RR) \
    if (p.R == RR) tf = bf ? conv3x3_tma_kernel<RR, true, true> : f16 ? conv3x3_tma_kernel<RR, true> : conv3x3_tma_kernel<RR, false>;
    SRT_T(1) SRT_T(2) SRT_T(4) SRT_T(8)
#undef SRT_T
    auto encode = tensor_map_encoder();
    if (!tf || !encode) {
      err = "internal: no TMA conv kernel instance / tensor-map encoder";
      return SPARSE_EINTERNAL;
    }
    if ((e = ensure_smem_attr(tf, p.smem_bytes)) != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
    const int S = f16 ? 2 : 4;
    const int64_t planes = (int64_t)p.c_in * batch, rows = planes * (p.h + 1);
    void* xp = nullptr;
    e = cudaMallocAsync(&xp, (size_t)(3 * rows * p.conv_wp * S), (cudaStream_t)stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cuda_fail(e, "cudaMallocAsync(conv pad)", err);
    }
    const int kPadPlanes = (int)std::max<int64_t>(1, std::min<int64_t>(8, (160 * 1024) / ((int64_t)p.h * p.w * S)));
    const unsigned pg = (unsigned)std::min<int64_t>((planes + kPadPlanes - 1) / kPadPlanes, 148 * 8);
    const size_t psm = (size_t)kPadPlanes * p.h * p.w * S;
    if (f16) {
      if ((e = ensure_smem_attr(pad_conv_input<uint16_t>, (int)psm)) != cudaSuccess)
        return cuda_fail(e, "cudaFuncSetAttribute(pad)", err);
      pad_conv_input<uint16_t><<<pg, 256, psm, (cudaStream_t)stream>>>((const uint16_t*)x, (uint16_t*)xp, planes,
                                                                       p.h, p.w, p.conv_wp, kPadPlanes);
    } else {
      if ((e = ensure_smem_attr(pad_conv_input<float>, (int)psm)) != cudaSuccess)
        return cuda_fail(e, "cudaFuncSetAttribute(pad)", err);
      pad_conv_input<float><<<pg, 256, psm, (cudaStream_t)stream>>>((const float*)x, (float*)xp, planes, p.h, p.w,
                                                                    p.conv_wp, kPadPlanes);
    }
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof tmap);
    cuuint64_t dims[5] = {(cuuint64_t)p.conv_wp, (cuuint64_t)(p.h + 1), (cuuint64_t)batch, (cuuint64_t)p.c_in, 3};
    cuuint64_t strides[4] = {(cuuint64_t)p.conv_wp * S, (cuuint64_t)p.conv_wp * S * (p.h + 1),
                             (cuuint64_t)p.conv_wp * S * (p.h + 1) * batch,
                             (cuuint64_t)p.conv_wp * S * (p.h + 1) * batch * p.c_in};
    cuuint32_t box[5] = {(cuuint32_t)p.conv_wp, (cuuint32_t)(p.conv_rb + 2), 1u, (cuuint32_t)p.cc, 1u};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(&tmap, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, xp, dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      cudaFreeAsync(xp, (cudaStream_t)stream);
      err = "conv: cuTensorMapEncodeTiled failed for the padded input";
      return SPARSE_EINTERNAL;
    }
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tf, p.warps * 32, p.smem_bytes) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    cudaGetLastError();
    const int64_t ntot = (int64_t)p.npanels * batch * a.bands;
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ntot, (int64_t)sms * per_sm)), 1, 1);
    cfg.blockDim = dim3((unsigned)(p.warps * 32), 1, 1);
    cfg.dynamicSmemBytes = (size_t)p.smem_bytes;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, tf, tmap, a);
    cudaFreeAsync(xp, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "conv3x3 (TMA) launch", err);
    return SPARSE_OK;
  }
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
