// Offline autotuner (Sec. 3.7 "Autotuning"): "we perform
// exhaustive grid search over a list of hand picked choices for each SpMM problem
// according to a couple of simple heuristics ... This typically resulted in less
// than 100 parameter combinations for each problem."
//
// Here: sparse_plan_create(..., opts.tune = 1) times every candidate tile
// configuration (and the JIT executor when its per-panel code is small) on the
// plan's device with synthetic X of the hinted size, and keeps the fastest.  The
// candidate grid stays under 100 entries.  Timing: 2 warm-up launches, then the
// median of 5 single launches, each after a 256 MiB memset that evicts the L2 and a 256 MiB
// read that leaves it clean (cold inputs, as bench.py measures), CUDA events on a private
// stream.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sparsert.h"
#include "plan.h"

namespace srt {

namespace {

constexpr int64_t kJitMaxPanelCode = 24 * 1024;
constexpr size_t kFlushBytes = 256u << 20;

__global__ void fill_uniform(uint8_t* p, int64_t n, int f16, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    const float v = (float)(h & 0xffffff) * (2.0f / 16777216.0f) - 1.0f;
    if (f16)
      reinterpret_cast<__half*>(p)[i] = __float2half_rn(v);
    else
      reinterpret_cast<float*>(p)[i] = v;
  }
}

// reads a buffer (so that L2 holds clean lines: no write-back of the memset flush is
// charged to the timed launch)
__global__ void read_sink(const uint4* p, int64_t n, uint32_t* sink) {
  uint32_t a = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = p[i];
    a ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (a == 0x9e3779b9u) *sink = a;
}

void release(Plan& p) {
  jit_unload(p);
  free_plan_device(p);
}

}  // namespace

int tune_plan(Plan& best, int32_t M, int32_t K, int64_t nnz, const int32_t* row_ptr,
              const int32_t* col_idx, const float* values, int32_t dtype, const BuildOpts& base,
              int device, std::string& err) {
  if (base.n_hint <= 0) {
    err = "tune = 1 needs n_hint > 0 (N for SpMM, batch for conv)";
    return SPARSE_EINVAL;
  }
  const bool f16 = dtype == SPARSE_F16;
  const int S = dtype != SPARSE_F32 ? 2 : 4;
  // candidate grid (hand-picked): warps per CTA, rows per warp, pipeline depth,
  // cluster K-split, split-K groups (small N); plus the JIT executor
  std::vector<BuildOpts> cands;
  if (base.kind == SPARSE_SPMM) {
    // consumer warps x rows per warp (panel height), K chunk, pipeline depth (stages < 0:
    // the inspector fills a shared-memory budget, -1 = one CTA per SM, -2 = two), cluster
    // K-split (N <= 4096), split-K groups (N <= 512)
    const int C = S == 2 ? 8 : 4;
    const int64_t N = base.n_hint;
    const bool small = N <= 512, medium = N <= 4096;
    for (int w : {8, 16})
      for (int R : {2, 4, 8})
        for (int kc : {32, 64, 128})
          for (int st : {-1, -2})
            for (int ks : {1, 2, 4, 8})
              for (int gk : {1, 2, 4}) {
                const int nch = (K + kc - 1) / kc;
                if (ks > nch || (ks > 1 && !medium) || (ks == 8 && !small)) continue;
                // split-K groups: small N (narrow tiles), and gk = 2 for the HBM-streaming
                // layers (K <= 256: twice the N tiles -> a finer last wave on 148 SMs)
                if (gk > 1 && !small && !(gk == 2 && K <= 256 && ks == 1 && st == -1)) continue;
                if (gk == 2 && N <= 256) continue;  // N <= 256: G_k in {1, 4}
                if (gk == 4 && N > 256) continue;
                if (R == 8 && (small || R * C > 64)) continue;
                if (kc == 32 && medium) continue;
                if (st == -2 && small) continue;
                if (kc > 32 && K <= kc / 2) continue;
                BuildOpts o = base;
                o.warps = w;
                o.rows_per_warp = R;
                o.k_chunk = kc;
                o.stages = st;
                o.k_split = ks;
                o.split_k = gk;
                o.executor = 0;
                cands.push_back(o);
                // small plans: the same tiles with the plan in kernel parameters (constant
                // cache, plan_source = 1; build_plan rejects plans over 30 KB)
                const int64_t est = nnz * (S == 2 ? 4 : 8);
                if (ks == 1 && gk == 1 && st == -1 && kc > 32 && est < 24 * 1024) {
                  o.ps = 1;
                  o.tc_min_pct = 0;
                  cands.push_back(o);
                }
              }
    if (f16) {  // tensor-core sub-blocks on / off (when the matrix has dense 16x16 tiles)
      for (int tc : {50, 0}) {
        BuildOpts o = base;
        o.warps = 16;
        o.rows_per_warp = 4;
        o.k_chunk = 128;
        o.tc_min_pct = tc;
        o.executor = 0;
        cands.push_back(o);
      }
    }
    BuildOpts j = base;
    j.executor = 1;
    cands.push_back(j);
    // tensor cores: condensed panels on mma.sync (16-bit), and W's nonzero
    // 128-row blocks on tcgen05 (TMEM accumulators; fp32 as 3xTF32), alone or in clusters of
    // 2 / 4 row blocks sharing each X tile by TMA multicast
    BuildOpts t = base;
    if (S == 2) {
      t.executor = 3;
      cands.push_back(t);
    }
    for (int cs : {1, 2, 4}) {
      if (cs > 1 && (M + 127) / 128 < cs) continue;
      t.executor = 4;
      t.cm = cs;
      cands.push_back(t);
    }
    if ((M + 127) / 128 >= 2) {  // CTA pairs (cta_group::2, M = 256)
      t.cm = 2;
      t.pair = 1;
      cands.push_back(t);
      t.pair = 0;
    }
    // few tiles for 148 SMs (small N): K slices per tile, reduced in order by a second kernel
    {
      const int64_t tiles = (int64_t)((M + 127) / 128) * ((base.n_hint + 255) / 256);
      const int bk = S == 2 ? 64 : 32, nkb = (K + bk - 1) / bk;
      for (int ks : {2, 4, 8, 16}) {
        if (tiles * ks > 2 * 148 || nkb < 2 * ks) continue;
        t.cm = (M + 127) / 128 >= 2 ? 2 : 1;
        t.pair = t.cm == 2;
        t.k_split = ks;
        cands.push_back(t);
      }
      t.k_split = base.k_split;
      t.pair = 0;
    }
  } else {
    // vectorised kernels (16-byte loads of consecutive positions; TMA-fed = 2, register-
    // staged = 1) and the position-strided one (0); cc = channels per chunk (0: inspector)
    for (int vec : {2, 4, 1, 0})
      for (int R : {2, 4, 8})
        for (int w : {8, 16})
          for (int cc : {0, 8, 16, 24, 32}) {
            if (!vec && w == 16) continue;  // the position-strided kernel runs <= 8 warps
            if (vec == 4 ? (R == 2 || w != 16 || cc < 16) : vec == 2 ? cc == 8 : (cc == 0 || cc == 24)) continue;
            BuildOpts o = base;
            o.rows_per_warp = R;
            o.warps = w;
            o.k_chunk = cc;
            o.conv_vec = vec;
            cands.push_back(o);
          }
    {  // implicit im2col on the tcgen05 block executor (conv_kernel 5; fp32 as 3xTF32)
      for (int cs : {1, 2, 3}) {  // 3 = a CTA pair
        if (cs > 1 && (M + 127) / 128 < 2) continue;
        BuildOpts o = base;
        o.conv_vec = 2;
        o.executor = 4;
        o.cm = cs == 3 ? 2 : cs;
        o.pair = cs == 3;
        cands.push_back(o);
      }
    }
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return SPARSE_ECUDA;
  }
  int64_t xe, ye, N = base.n_hint;
  // at run time unaligned X is repacked to a 16-byte row stride first, so time that layout
  const int64_t per16 = 16 / S;
  const int64_t ldt = (N + per16 - 1) / per16 * per16;
  if (base.kind == SPARSE_SPMM) {
    xe = (int64_t)K * ldt;
    ye = (int64_t)M * ldt;
  } else {
    xe = (int64_t)base.c_in * N * base.h * base.w;
    ye = (int64_t)M * N * base.h * base.w;
  }
  uint8_t *X = nullptr, *Y = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  if (cudaMalloc(&X, (size_t)xe * S + 16) != cudaSuccess ||
      cudaMalloc(&Y, (size_t)ye * S + 16) != cudaSuccess) {
    cudaFree(X);
    cudaGetLastError();
    err = "tune: cannot allocate the synthetic X / Y";
    return SPARSE_ENOMEM;
  }
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEventCreate(&ev[0]);
  cudaEventCreate(&ev[1]);
  fill_uniform<<<1024, 256, 0, st>>>(X, xe, S == 2 ? 1 : 0, 12345u);
  void* flush = nullptr;
  if (cudaMalloc(&flush, 2 * kFlushBytes) != cudaSuccess) {
    cudaGetLastError();
    flush = nullptr;  // warm-L2 timing only
  }
  float best_ms = 1e30f;
  const bool debug = getenv("SPARSERT_TUNE_DEBUG") != nullptr;
  bool have = false;
  std::string last_err;
  for (const BuildOpts& o : cands) {
    Plan p;
    std::string e2;
    int rc = build_plan(p, M, K, nnz, row_ptr, col_idx, values, dtype, o, e2);
    if (rc != SPARSE_OK) continue;
    if (p.executor == 1) {
      // JIT only where each panel's straight-line code stays instruction-cache sized
      // (the instruction-fetch limit of P:379, measured on B200: DESIGN.md)
      if (jit_panel_code_bytes(p) > kJitMaxPanelCode) continue;
      if (jit_compile(p, e2) != SPARSE_OK) continue;
    }
    p.device = device;
    if (upload_plan(p, e2) != SPARSE_OK) continue;
    if (p.executor == 1 && jit_load(p, e2) != SPARSE_OK) {
      release(p);
      continue;
    }
    auto run = [&]() -> int {
      if (base.kind == SPARSE_SPMM) {
        if (p.executor == 1 && jit_can_launch(p, X, ldt)) return jit_launch(p, N, X, ldt, Y, ldt, st, e2);
        return launch_spmm(p, N, X, ldt, Y, ldt, st, e2);
      }
      return launch_conv3x3(p, N, X, Y, st, e2);
    };
    // every timed launch starts with a cold L2 (a 256 MiB memset evicts it), as in bench.py:
    // the HBM-honest condition a layer meets when its input was produced long before
    bool ok = run() == SPARSE_OK && run() == SPARSE_OK;
    std::vector<float> ms;
    for (int r = 0; ok && r < 5; ++r) {
      if (flush) {  // write 256 MiB (evicts the L2), then read another 256 MiB (cleans it)
        cudaMemsetAsync(flush, r, kFlushBytes, st);
        read_sink<<<1184, 256, 0, st>>>((const uint4*)((uint8_t*)flush + kFlushBytes),
                                        (int64_t)(kFlushBytes / 16), (uint32_t*)flush);
      }
      cudaEventRecord(ev[0], st);
      ok = run() == SPARSE_OK;
      cudaEventRecord(ev[1], st);
      if (cudaEventSynchronize(ev[1]) != cudaSuccess) ok = false;
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[0], ev[1]);
      ms.push_back(t);
    }
    if (!ok) {
      if (debug)
        fprintf(stderr, "[tune] exec=%d warps=%d R=%d kc=%d ks=%d gk=%d stages=%d: FAILED %s / %s\n",
                p.executor, p.warps, p.R, p.kc, p.ks, p.gk, p.stages, e2.c_str(),
                cudaGetErrorString(cudaGetLastError()));
      last_err = e2;
      cudaGetLastError();
      release(p);
      continue;
    }
    std::sort(ms.begin(), ms.end());
    const float med = ms[ms.size() / 2];
    if (debug)
      fprintf(stderr, "[tune] exec=%d warps=%d R=%d kc=%d ks=%d gk=%d stages=%d: %.2f us\n",
              p.executor, p.warps, p.R, p.kc, p.ks, p.gk, p.stages, med * 1000.0f);
    if (med < best_ms) {
      if (have) release(best);
      best = std::move(p);
      // `p` no longer owns the device state
      p.d_mem = nullptr;
      for (auto& jm : p.jit) jm.mod = jm.fn = nullptr;
      best_ms = med;
      have = true;
    } else {
      release(p);
    }
  }
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  cudaStreamDestroy(st);
  cudaFree(flush);
  cudaFree(X);
  cudaFree(Y);
  if (!have) {
    err = "tune: no candidate ran" + (last_err.empty() ? std::string() : ": " + last_err);
    return SPARSE_EINTERNAL;
  }
  best.tuned_us = best_ms * 1000.0;
  return SPARSE_OK;
}

}  // namespace srt
