// C ABI (include/sparsert.h): argument validation, error reporting and plan
// ownership around the inspector (inspector.cpp) and executors (kernels.cu).
// No exception crosses this boundary; nothing here computes on the CPU.
#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include "../../include/sparsert.h"
#include "plan.h"

#include <cuda_runtime.h>

struct sparse_plan_s {
  srt::Plan p;
  bool host_only = false;
};

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int ok() {
  g_err.clear();
  return SPARSE_OK;
}
}  // namespace

extern "C" {

void sparse_plan_opts_init(sparse_plan_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->kind = SPARSE_SPMM;
  o->device = -1;
}

int sparse_plan_create(sparse_plan_t* out, int32_t M, int32_t K, int64_t nnz,
                       const int32_t* row_ptr, const int32_t* col_idx, const float* values,
                       int32_t dtype, const sparse_plan_opts* opts) {
  if (!out) return fail(SPARSE_EINVAL, "out is NULL");
  *out = nullptr;
  sparse_plan_opts d;
  sparse_plan_opts_init(&d);
  const sparse_plan_opts& o = opts ? *opts : d;
  if (o.tune != 0 && o.tune != 1) return fail(SPARSE_EINVAL, "tune must be 0 or 1");
  srt::BuildOpts bo;
  bo.kind = o.kind;
  bo.c_in = o.c_in;
  bo.h = o.h;
  bo.w = o.w;
  bo.n_hint = o.n_hint;
  bo.drop_zeros = o.drop_zeros;
  bo.warps = o.warps;
  bo.rows_per_warp = o.rows_per_warp;
  bo.k_chunk = o.k_chunk;
  bo.split_k = o.split_k;
  bo.k_split = o.k_split;
  bo.stages = o.stages;
  bo.executor = o.executor;
  bo.jit_rows = o.jit_rows;
  bo.jit_warps = o.jit_warps;
  bo.cm = o.x_multicast;
  bo.tm = o.x_source;
  if (o.cta_pair != 0 && o.cta_pair != 1) return fail(SPARSE_EINVAL, "cta_pair must be 0 or 1");
  bo.pair = o.cta_pair;
  if (o.conv_kernel < 0 || o.conv_kernel > 5)
    return fail(SPARSE_EINVAL,
                "conv_kernel must be 0 (auto), 1 (position-strided), 2 (TMA-fed), 3 (register-staged), "
                "4 (interleaved) or 5 (tcgen05 blocks)");
  // (conv_kernel 5 runs on the tcgen05 block executor; its CUDA-core plan is the default TMA-fed one)
  bo.conv_vec = o.conv_kernel == 1 ? 0 : o.conv_kernel == 3 ? 1 : o.conv_kernel == 4 ? 4 : 2;
  if (o.kind == SPARSE_CONV3X3 && o.conv_kernel == 5) bo.executor = 4;
  if (o.row_order != 0 && o.row_order != 1)
    return fail(SPARSE_EINVAL, "row_order must be 0 (load balanced) or 1 (natural)");
  bo.row_order = o.row_order;
  if (o.tc_min_density < -1 || o.tc_min_density > 100)
    return fail(SPARSE_EINVAL, "tc_min_density must be -1 (off), 0 (default) or 1..100");
  bo.tc_min_pct = o.tc_min_density == 0 ? 50 : (o.tc_min_density < 0 ? 0 : o.tc_min_density);
  bo.ps = o.plan_source;
  if (o.stages < 0 || o.stages > srt::kMaxStages)
    return fail(SPARSE_EUNSUPPORTED, "stages must be in [0, 8]");
  sparse_plan_s* h = nullptr;
  try {
    h = new sparse_plan_s();
  } catch (const std::bad_alloc&) {
    return fail(SPARSE_ENOMEM, "host allocation failed");
  }
  std::string err;
  int rc;
  if (o.tune == 1) {
    if (o.device == SPARSE_DEVICE_HOST_ONLY) {
      delete h;
      return fail(SPARSE_EINVAL, "tune = 1 needs a device");
    }
    int dev = o.device, prev_dev = -1;
    if (cudaGetDevice(&prev_dev) != cudaSuccess) {
      delete h;
      return fail(SPARSE_ECUDA, "no CUDA device");
    }
    if (dev < 0) dev = prev_dev;
    try {
      rc = srt::tune_plan(h->p, M, K, nnz, row_ptr, col_idx, values, dtype, bo, dev, err);
      cudaSetDevice(prev_dev);  // the tuner selects `dev`; the caller's current device is kept
    } catch (const std::bad_alloc&) {
      rc = SPARSE_ENOMEM;
      err = "host allocation failed in tuner";
    }
    if (rc != SPARSE_OK) {
      delete h;
      return fail(rc, err);
    }
    *out = h;
    return ok();
  }
  const bool auto_exec = bo.executor == 2;
  // auto: try the JIT executor first, except where it cannot apply (bf16 values, the TMEM X
  // source, conv plans), which go straight to the plan-driven kernel
  if (auto_exec) bo.executor = (dtype == SPARSE_BF16 || bo.tm || bo.ps || bo.kind != SPARSE_SPMM) ? 0 : 1;
  try {
    rc = srt::build_plan(h->p, M, K, nnz, row_ptr, col_idx, values, dtype, bo, err);
    if (auto_exec && bo.executor == 1 &&
        (rc == SPARSE_EUNSUPPORTED ||
         (rc == SPARSE_OK && h->p.executor == 1 && srt::jit_panel_code_bytes(h->p) > 24 * 1024))) {
      // auto: the JIT executor only where each panel's code fits the instruction cache
      bo.executor = 0;
      rc = srt::build_plan(h->p, M, K, nnz, row_ptr, col_idx, values, dtype, bo, err);
    }
  } catch (const std::bad_alloc&) {
    rc = SPARSE_ENOMEM;
    err = "host allocation failed in inspector";
  } catch (...) {
    rc = SPARSE_EINTERNAL;
    err = "unexpected exception in inspector";
  }
  if (rc == SPARSE_OK && h->p.executor == 1) rc = srt::jit_compile(h->p, err);
  if (rc != SPARSE_OK) {
    delete h;
    return fail(rc, err);
  }
  if (o.device == SPARSE_DEVICE_HOST_ONLY) {
    h->host_only = true;
    h->p.device = SPARSE_DEVICE_HOST_ONLY;
  } else {
    if (o.device < -1) {
      delete h;
      return fail(SPARSE_EINVAL, "device must be >= -1 or SPARSE_DEVICE_HOST_ONLY");
    }
    h->p.device = o.device;
    rc = srt::upload_plan(h->p, err);
    if (rc == SPARSE_OK && h->p.executor == 1) rc = srt::jit_load(h->p, err);
    if (rc != SPARSE_OK) {
      srt::jit_unload(h->p);
      srt::free_plan_device(h->p);
      delete h;
      return fail(rc, err);
    }
  }
  *out = h;
  return ok();
}

static int spmm_impl(sparse_plan_t plan, int64_t N, const void* X, int64_t ldx, void* Y,
                     int64_t ldy, const sparse_epilogue* e, sparse_stream_t stream) {
  if (!plan) return fail(SPARSE_EINVAL, "plan is NULL");
  if (plan->p.kind != SPARSE_SPMM) return fail(SPARSE_EINVAL, "sparse_spmm on a conv plan");
  if (plan->host_only) return fail(SPARSE_EINVAL, "host-only plan cannot compute");
  if (N < 0) return fail(SPARSE_EINVAL, "N < 0");
  if (N == 0) return ok();
  if (!X || !Y) return fail(SPARSE_EINVAL, "X or Y is NULL");
  if (ldx < N || ldy < N) return fail(SPARSE_EINVAL, "ldx and ldy must be >= N");
  srt::Epilogue ep;
  if (e) {
    if (e->relu != 0 && e->relu != 1) return fail(SPARSE_EINVAL, "epilogue relu must be 0 or 1");
    ep.beta = e->beta;
    ep.bias = e->bias;
    ep.relu = e->relu;
  }
  std::string err;
  const srt::Plan& p = plan->p;
  const int S = p.dtype != SPARSE_F32 ? 2 : 4;
  const void* Xa = X;
  int64_t lda = ldx;
  void* scratch = nullptr;
  if (((uintptr_t)X % 16) != 0 || ((ldx * S) % 16) != 0) {
    // TMA needs a 16-byte aligned base and row stride: repack on the device (never on the
    // host); if no scratch can be had, the kernels' element-wise staging path is used
    if (srt::launch_repack(p.device, p.K, N, S, X, ldx, &scratch, &lda, stream, err) == SPARSE_OK) {
      Xa = scratch;
    } else {
      lda = ldx;
      scratch = nullptr;
    }
  }
  const int rc = ep.trivial() && srt::jit_can_launch(p, Xa, lda)
                     ? srt::jit_launch(p, N, Xa, lda, Y, ldy, stream, err)
                     : srt::launch_spmm(p, N, Xa, lda, Y, ldy, stream, err, ep);
  if (scratch) srt::free_repack(p.device, scratch, stream);
  return rc == SPARSE_OK ? ok() : fail(rc, err);
}

int sparse_spmm(sparse_plan_t plan, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy,
                sparse_stream_t stream) {
  return spmm_impl(plan, N, X, ldx, Y, ldy, nullptr, stream);
}

int sparse_spmm_ex(sparse_plan_t plan, int64_t N, const void* X, int64_t ldx, void* Y,
                   int64_t ldy, const sparse_epilogue* ep, sparse_stream_t stream) {
  return spmm_impl(plan, N, X, ldx, Y, ldy, ep, stream);
}

int sparse_linear(sparse_plan_t plan, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy,
                  sparse_stream_t stream) {
  if (!plan) return fail(SPARSE_EINVAL, "plan is NULL");
  if (plan->p.kind != SPARSE_SPMM) return fail(SPARSE_EINVAL, "sparse_linear on a conv plan");
  if (plan->host_only) return fail(SPARSE_EINVAL, "host-only plan cannot compute");
  if (N < 0) return fail(SPARSE_EINVAL, "N < 0");
  if (N == 0) return ok();
  if (!X || !Y) return fail(SPARSE_EINVAL, "X or Y is NULL");
  const srt::Plan& p = plan->p;
  if (ldx < p.K || ldy < p.M) return fail(SPARSE_EINVAL, "ldx must be >= K and ldy >= M");
  const int S = p.dtype != SPARSE_F32 ? 2 : 4;
  const int64_t ldt = (N + 15) / 16 * 16;  // 16-byte aligned rows for the TMA paths (S <= 4)
  void* Xt = nullptr;
  void* Yt = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  int prev_dev = -1;
  if (cudaGetDevice(&prev_dev) != cudaSuccess) return fail(SPARSE_ECUDA, "cudaGetDevice failed");
  struct Restore {  // the scratch lives on the plan's device; restore the caller's device
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{prev_dev};
  if (p.device >= 0 && p.device != prev_dev && cudaSetDevice(p.device) != cudaSuccess)
    return fail(SPARSE_ECUDA, "cudaSetDevice(plan device) failed");
  if (cudaMallocAsync(&Xt, (size_t)(p.K * ldt * S), st) != cudaSuccess ||
      cudaMallocAsync(&Yt, (size_t)(p.M * ldt * S), st) != cudaSuccess) {
    cudaGetLastError();
    if (Xt) cudaFreeAsync(Xt, st);
    return fail(SPARSE_ENOMEM, "sparse_linear: cannot allocate the transposed scratch");
  }
  std::string err;
  int rc = srt::launch_transpose(p.device, S, X, ldx, Xt, ldt, N, p.K, stream, err);  // Xt = X^T (K x N)
  if (rc == SPARSE_OK) {
    const int r2 = sparse_spmm(plan, N, Xt, ldt, Yt, ldt, stream);
    if (r2 != SPARSE_OK) {
      cudaFreeAsync(Xt, st);
      cudaFreeAsync(Yt, st);
      return r2;  // sparse_spmm set the error detail
    }
    rc = srt::launch_transpose(p.device, S, Yt, ldt, Y, ldy, p.M, N, stream, err);  // Y = Yt^T (N x M)
  }
  cudaFreeAsync(Xt, st);
  cudaFreeAsync(Yt, st);
  return rc == SPARSE_OK ? ok() : fail(rc, err);
}

static int conv_impl(sparse_plan_t plan, int64_t batch, const void* x, void* y,
                     const sparse_epilogue* e, sparse_stream_t stream) {
  if (!plan) return fail(SPARSE_EINVAL, "plan is NULL");
  if (plan->p.kind != SPARSE_CONV3X3) return fail(SPARSE_EINVAL, "sparse_conv3x3 on an SpMM plan");
  if (plan->host_only) return fail(SPARSE_EINVAL, "host-only plan cannot compute");
  if (batch < 0) return fail(SPARSE_EINVAL, "batch < 0");
  if (batch == 0) return ok();
  if (!x || !y) return fail(SPARSE_EINVAL, "x or y is NULL");
  srt::Epilogue ep;
  if (e) {
    if (e->relu != 0 && e->relu != 1) return fail(SPARSE_EINVAL, "epilogue relu must be 0 or 1");
    ep.beta = e->beta;
    ep.bias = e->bias;
    ep.relu = e->relu;
  }
  std::string err;
  const int rc = srt::launch_conv3x3(plan->p, batch, x, y, stream, err, ep);
  return rc == SPARSE_OK ? ok() : fail(rc, err);
}

int sparse_conv3x3(sparse_plan_t plan, int64_t batch, const void* x, void* y,
                   sparse_stream_t stream) {
  return conv_impl(plan, batch, x, y, nullptr, stream);
}

int sparse_conv3x3_ex(sparse_plan_t plan, int64_t batch, const void* x, void* y,
                      const sparse_epilogue* ep, sparse_stream_t stream) {
  return conv_impl(plan, batch, x, y, ep, stream);
}

namespace {
// stream-ordered device scratch on the plan's device (caller's device restored on return)
struct Scratch {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  int prev = -1;
  bool ok = false;
  Scratch(int dev, size_t bytes, sparse_stream_t stream) : st((cudaStream_t)stream) {
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    if (dev >= 0 && dev != prev && cudaSetDevice(dev) != cudaSuccess) return;
    ok = cudaMallocAsync(&p, bytes ? bytes : 16, st) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      p = nullptr;
    }
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

int sparse_conv1x1(sparse_plan_t plan, int64_t batch, int32_t h, int32_t w, int32_t stride, const void* x,
                   void* y, sparse_stream_t stream) {
  if (!plan) return fail(SPARSE_EINVAL, "plan is NULL");
  if (plan->p.kind != SPARSE_SPMM) return fail(SPARSE_EINVAL, "sparse_conv1x1 needs an SpMM plan (W = C_out x C_in)");
  if (plan->host_only) return fail(SPARSE_EINVAL, "host-only plan cannot compute");
  if (batch < 0 || h < 1 || w < 1 || stride < 1) return fail(SPARSE_EINVAL, "batch >= 0, h, w, stride >= 1 required");
  if (batch == 0) return ok();
  if (!x || !y) return fail(SPARSE_EINVAL, "x or y is NULL");
  const srt::Plan& p = plan->p;
  const int S = p.dtype != SPARSE_F32 ? 2 : 4;
  const int64_t ho = (h + stride - 1) / stride, wo = (w + stride - 1) / stride, N = batch * ho * wo;
  if (stride == 1) return sparse_spmm(plan, N, x, N, y, N, stream);
  Scratch xs(p.device, (size_t)(p.K * N * S), stream);
  if (!xs.ok) return fail(SPARSE_ENOMEM, "sparse_conv1x1: cannot allocate the gather scratch");
  std::string err;
  const int rc = srt::launch_stride_gather(p.device, S, x, p.K, batch, h, w, stride, xs.p, stream, err);
  if (rc != SPARSE_OK) return fail(rc, err);
  return sparse_spmm(plan, N, xs.p, N, y, N, stream);  // sets the error detail itself
}

int sparse_conv3x3_nhwc(sparse_plan_t plan, int64_t batch, const void* x, void* y, sparse_stream_t stream) {
  if (!plan) return fail(SPARSE_EINVAL, "plan is NULL");
  if (plan->p.kind != SPARSE_CONV3X3) return fail(SPARSE_EINVAL, "sparse_conv3x3_nhwc on an SpMM plan");
  if (plan->host_only) return fail(SPARSE_EINVAL, "host-only plan cannot compute");
  if (batch < 0) return fail(SPARSE_EINVAL, "batch < 0");
  if (batch == 0) return ok();
  if (!x || !y) return fail(SPARSE_EINVAL, "x or y is NULL");
  const srt::Plan& p = plan->p;
  const int S = p.dtype != SPARSE_F32 ? 2 : 4;
  const int64_t N = batch * (int64_t)p.h * p.w;
  {  // tcgen05 block executor: the im2col TMA reads NHWC and the epilogue writes NHWC directly
    std::string err;
    const int rc = srt::launch_conv3x3_nhwc(p, batch, x, y, stream, err);
    if (rc == SPARSE_OK) return ok();
    if (rc != SPARSE_EUNSUPPORTED) return fail(rc, err);
  }
  Scratch xt(p.device, (size_t)(p.c_in * N * S), stream), yt(p.device, (size_t)(p.M * N * S), stream);
  if (!xt.ok || !yt.ok) return fail(SPARSE_ENOMEM, "sparse_conv3x3_nhwc: cannot allocate the CNHW scratch");
  std::string err;
  int rc = srt::launch_transpose(p.device, S, x, p.c_in, xt.p, N, N, p.c_in, stream, err);  // [N][C] -> [C][N]
  if (rc != SPARSE_OK) return fail(rc, err);
  const int r2 = sparse_conv3x3(plan, batch, xt.p, yt.p, stream);
  if (r2 != SPARSE_OK) return r2;
  rc = srt::launch_transpose(p.device, S, yt.p, N, y, p.M, p.M, N, stream, err);  // [M][N] -> [N][M]
  return rc == SPARSE_OK ? ok() : fail(rc, err);
}

int plan_destroy(sparse_plan_t plan) {
  if (!plan) return ok();
  srt::jit_unload(plan->p);
  srt::free_plan_device(plan->p);
  delete plan;
  return ok();
}

int sparse_plan_destroy(sparse_plan_t plan) { return plan_destroy(plan); }

int sparse_plan_info(sparse_plan_t plan, sparse_plan_info_t* out) {
  if (!plan || !out) return fail(SPARSE_EINVAL, "plan or out is NULL");
  const srt::Plan& p = plan->p;
  std::memset(out, 0, sizeof *out);
  out->nnz = p.nnz;
  out->plan_bytes = p.plan_bytes;
  out->M = p.M;
  out->K = p.K;
  out->dtype = p.dtype;
  out->kind = p.kind;
  out->panels = p.npanels;
  out->warps = p.warps;
  out->rows_per_warp = p.R;
  out->cols_per_lane = p.C;
  out->n_tile = p.n_tile;
  out->k_chunk = p.kind == SPARSE_CONV3X3 ? p.cc : p.kc;
  out->chunks = p.nchunks;
  out->split_k = p.gk;
  out->k_split = p.executor == 4 ? p.tcg_ks : p.ks;
  out->stages = p.stages;
  out->smem_bytes = p.smem_bytes;
  out->device = p.device;
  out->conv_rows_per_tile = p.conv_rb;
  out->conv_images_per_tile = p.kind == SPARSE_CONV3X3 && p.executor == 4 ? p.tcg_g : p.conv_ipt;
  out->max_panel_nnz = p.max_panel_nnz;
  out->min_panel_nnz = p.min_panel_nnz;
  out->build_ms = p.build_ms;
  out->digest = p.digest;
  out->executor = p.executor;
  out->jit_modules = (int32_t)p.jit.size();
  out->jit_rows = p.jit_mp;
  out->jit_warps = p.jit_warps;
  out->jit_cubin_bytes = p.jit_cubin_bytes;
  out->jit_compile_ms = p.jit_compile_ms;
  out->tuned_us = p.tuned_us;
  out->x_multicast = p.executor == 4 ? p.tcg_cs : p.cm;
  out->cta_pair = p.tcg_pair;
  out->x_source = p.tm;
  out->conv_kernel = p.kind != SPARSE_CONV3X3 ? 0 : p.executor == 4 ? 5 : !p.conv_vec ? 1 : p.conv_vec == 2 ? 2 : p.conv_vec == 4 ? 4 : 3;
  out->row_order = p.row_order;
  out->tc_min_density = p.tc_ntiles > 0 || p.tc_min_pct > 0 ? p.tc_min_pct : 0;
  out->tc_row_blocks = p.tc_nrb;
  out->tc_tiles = p.tc_ntiles;
  out->tc_panel_steps = p.tcp_nsteps;
  out->tc_nnz = p.tc_nnz;
  out->plan_source = p.ps;
  return ok();
}

int sparse_plan_dump(sparse_plan_t plan, int64_t cap, int32_t* row, int32_t* col, float* value,
                     int32_t* panel, int32_t* chunk, int32_t* slot, int32_t* group) {
  if (!plan) return fail(SPARSE_EINVAL, "plan is NULL");
  const srt::Plan& p = plan->p;
  if (cap < p.nnz) return fail(SPARSE_EINVAL, "cap < nnz");
  const bool f16 = p.dtype != SPARSE_F32;  // 16-bit entries (fp16 or bf16 values)
  const bool bf = p.dtype == SPARSE_BF16;
  const int A = p.entry_align;
  int64_t out = 0;
  auto emit = [&](int32_t m, int32_t k, float w, int32_t q, int32_t c, int32_t s, int32_t g) {
    if (out >= cap) return false;
    if (row) row[out] = m;
    if (col) col[out] = k;
    if (value) value[out] = w;
    if (panel) panel[out] = q;
    if (chunk) chunk[out] = c;
    if (slot) slot[out] = s;
    if (group) group[out] = g;
    ++out;
    return true;
  };
  const int64_t rowb = (int64_t)p.n_tile * (f16 ? 2 : 4);
  for (int32_t q = 0; q < p.npanels; ++q) {
    for (int32_t c = 0; c < p.nchunks; ++c) {
      const uint8_t* blk = p.blob.data() + p.blk_off[(size_t)q * p.nchunks + c];
      const uint32_t* shdr = (const uint32_t*)blk;
      const uint8_t* ents = blk + p.hdr_bytes;
      for (int s = 0; s < p.Mp; ++s) {
        const int32_t m = p.row_id[(size_t)q * p.Mp + s];
        if (p.kind == SPARSE_SPMM || p.conv_vec) {
          for (int g = 0; g < p.gk; ++g) {
            const uint32_t h = shdr[s * p.gk + g];
            const int64_t u0 = h & 0xffffu, nu = h >> 16;
            for (int64_t e = u0 * A; e < (u0 + nu) * A; ++e) {
              const uint8_t* rec = ents + e * p.entry_bytes;
              int64_t xoff;
              float w;
              if (f16) {
                uint16_t a, wh;
                std::memcpy(&a, rec, 2);
                std::memcpy(&wh, rec + 2, 2);
                xoff = (int64_t)a * (p.kind == SPARSE_CONV3X3 && p.conv_vec == 4 ? 8 : 16);
                if (bf) {
                  const uint32_t b = (uint32_t)wh << 16;
                  std::memcpy(&w, &b, 4);
                } else {
                  w = srt::f16_to_f32(wh);
                }
              } else {
                uint32_t a;
                std::memcpy(&a, rec, 4);
                std::memcpy(&w, rec + 4, 4);
                xoff = a;
              }
              int64_t kl;
              if (p.kind == SPARSE_SPMM) {
                if (xoff % rowb) return fail(SPARSE_EINTERNAL, "plan entry offset not a row multiple");
                kl = xoff / rowb;
              } else if (p.conv_vec == 4) {  // interleaved conv: el = dx cs + ci lc + dy P
                const int64_t el = xoff / (f16 ? 2 : 4);
                if (el == 3 * (int64_t)p.conv_cs + p.conv_wp) {
                  kl = p.kc;
                } else {
                  const int64_t dx = el / p.conv_cs, rem = el % p.conv_cs;
                  const int64_t ci = rem / p.il_lc, dyP = rem % p.il_lc;
                  if (dx > 2 || ci >= p.cc || dyP % p.conv_wp || dyP / p.conv_wp > 2)
                    return fail(SPARSE_EINTERNAL, "interleaved conv plan entry offset does not decode");
                  kl = ci * 9 + (dyP / p.conv_wp) * 3 + dx;
                }
              } else {  // vectorised conv: elems = dx * cs + ci * sci + dy * wp, or the zero block
                const int64_t el = xoff / (f16 ? 2 : 4);
                if (el == 3 * (int64_t)p.conv_cs) {
                  kl = p.kc;
                } else {
                  const int64_t dx = el / p.conv_cs, rem = el % p.conv_cs;
                  const int64_t ci = rem / p.conv_sci, dy = (rem % p.conv_sci) / p.conv_wp;
                  if (dx > 2 || dy > 2 || (rem % p.conv_sci) % p.conv_wp)
                    return fail(SPARSE_EINTERNAL, "conv plan entry offset does not decode");
                  kl = ci * 9 + dy * 3 + dx;
                }
              }
              if (kl == p.kc) {  // neutral padding entry (zero row, -0 weight)
                if (!(w == 0.0f && std::signbit(w)))
                  return fail(SPARSE_EINTERNAL, "padding entry with a nonzero weight");
                continue;
              }
              if (m < 0) return fail(SPARSE_EINTERNAL, "entry in an empty row slot");
              const int32_t kg = p.kind == SPARSE_SPMM ? (int32_t)(c * p.kc + kl) : (int32_t)(c * p.cc * 9 + kl);
              if (!emit(m, kg, w, q, c, s, g))
                return fail(SPARSE_EINTERNAL, "plan carries more entries than nnz");
            }
          }
          continue;
        }
        const int beg = (int)(shdr[s] & 0xffffu), cnt = (int)(shdr[s] >> 16);
        for (int e = beg; e < beg + cnt; ++e) {
          const uint8_t* rec = ents + (size_t)e * p.entry_bytes;
          float w;
          int32_t off;
          if (f16) {
            int16_t o16;
            uint16_t wh;
            std::memcpy(&o16, rec, 2);
            std::memcpy(&wh, rec + 2, 2);
            off = o16;
            w = srt::f16_to_f32(wh);
          } else {
            std::memcpy(&off, rec, 4);
            std::memcpy(&w, rec + 4, 4);
          }
          // invert off = ci*sci + (dy-1)*wp + (dx-1), |(dy-1)*wp + (dx-1)| <= wp + 1 < sci / 2
          const int base = off + p.conv_wp + 1;  // = ci*sci + dy*wp + dx
          const int ci = base / p.conv_sci;
          const int rem = base - ci * p.conv_sci;
          const int dy = rem / p.conv_wp, dx = rem % p.conv_wp;
          if (!emit(m, (c * p.cc + ci) * 9 + dy * 3 + dx, w, q, c, s, 0))
            return fail(SPARSE_EINTERNAL, "plan carries more entries than nnz");
        }
      }
    }
  }
  // tensor-core sub-blocks: the nonzero slots of every dense tile (panel/chunk/slot = -1,
  // group = tile index)
  for (size_t i = 0; i < p.tc_rb.size(); ++i) {
    for (int32_t t = p.tc_tile_begin[i]; t < p.tc_tile_begin[i + 1]; ++t) {
      for (int lane = 0; lane < 32; ++lane) {
        for (int sl = 0; sl < 8; ++sl) {
          const uint16_t wh = p.tc_a[(size_t)t * 256 + lane * 8 + sl];
          if ((wh & 0x7fffu) == 0) continue;
          const int g = lane / 4, tq = lane % 4;
          const int r = g + 8 * ((sl >> 1) & 1), c = 2 * tq + (sl & 1) + 8 * (sl >> 2);
          if (!emit(p.tc_rb[i] * 16 + r, p.tc_cb[t] * 16 + c, srt::f16_to_f32(wh), -1, -1, -1, t))
            return fail(SPARSE_EINTERNAL, "plan carries more entries than nnz");
        }
      }
    }
  }
  if (out != p.nnz) return fail(SPARSE_EINTERNAL, "plan entry count != nnz");
  return ok();
}

const char* sparse_last_error(void) { return g_err.c_str(); }

const char* sparse_version(void) { return "sparsert-b200 0.1 sm_100a"; }

}  // extern "C"
