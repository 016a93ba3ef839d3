// JIT executor: the paper's code generator (Sec. 3.5) for sm_100a.
//
// "In SparseRT, we unroll the loop from line 9-11 in the code generator for each
// thread group and fill in the corresponding sparse matrix values, A[a,b], which we
// know them at compile time. This leads to the usage of the constant cache for A
// values and usage of registers for the accumulators".  "The SpMM code
// generator is implemented in Python, and generates PTX code"; here it is
// C++ inside the library and the PTX is assembled in-process with the static
// nvPTXCompiler, then loaded with the driver API.
//
// Generated kernel, one module per group of row panels (compiled in parallel):
//   grid (N tiles, panels of the module), block = W consumer warps + 1 producer warp
//   producer lane: TMA 2-D boxes X[kc rows][32*W columns] into a `stages`-deep ring
//   consumer warp w, lane l: owns output column n0 + 32 w + l (Gsy = 32 W threads,
//     the paper's "inner loop fixed to 1") and one fp32 accumulator register
//     per panel row (ACC[M_list, N_list])
//   per chunk, per k of the panel's K union, ascending (Alg. 3):
//     x = X[k][n]                                   (line 200: cache B[b, N_list])
//     a_r = fma(x, w_rk, a_r)  for r in M_nnz(k)   (lines 201-203, w_rk immediate)
//   epilogue: Y[row_id(r)][n] = a_r (row ids are immediates too)
// Every output's summation is k-ascending and sequential, i.e. bit-identical to the
// plan-driven kernels with split_k = k_split = 1.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvPTXCompiler.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sparsert.h"
#include "plan.h"

namespace srt {

namespace {

void appendf(std::string& s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void appendf(std::string& s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  const int n = vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (n < (int)sizeof buf) {
    s.append(buf, (size_t)n);
  } else {
    std::vector<char> big((size_t)n + 1);
    va_start(ap, fmt);
    vsnprintf(big.data(), big.size(), fmt, ap);
    va_end(ap);
    s.append(big.data(), (size_t)n);
  }
}

uint32_t fbits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

struct DriverApi {
  CUresult (*moduleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, CUstream, void**, void**) = nullptr;
  CUresult (*moduleUnload)(CUmodule) = nullptr;
  CUresult (*tensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
  bool ok = false;
};

const DriverApi& driver() {
  static DriverApi d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fp) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fp, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess;
    };
    bool ok = true;
    ok &= get("cuModuleLoadData", (void**)&d.moduleLoadData);
    ok &= get("cuModuleGetFunction", (void**)&d.moduleGetFunction);
    ok &= get("cuFuncSetAttribute", (void**)&d.funcSetAttribute);
    ok &= get("cuLaunchKernel", (void**)&d.launchKernel);
    ok &= get("cuModuleUnload", (void**)&d.moduleUnload);
    ok &= get("cuTensorMapEncodeTiled", (void**)&d.tensorMapEncodeTiled);
    d.ok = ok;
  });
  return d;
}

// Emit one module covering panels [pb, pe).
void emit_module(std::string& s, const Plan& p, int pb, int pe,
                 const std::vector<std::vector<RowEntry>>& rows, int64_t& fmas) {
  const bool f16 = p.dtype == SPARSE_F16;
  const int S = f16 ? 2 : 4;
  const int W = p.jit_warps, NT = 32 * W, Mp = p.jit_mp, kc = p.jit_kc, ST = p.jit_stages;
  const int stage_bytes = kc * NT * S;
  const int bar_off = ST * stage_bytes;
  const int lg_st = ST == 1 ? 0 : ST == 2 ? 1 : 2;
  const int nch = (p.K + kc - 1) / kc;
  s.reserve(s.size() + (1u << 20));
  appendf(s, ".version 8.7\n.target sm_100a\n.address_size 64\n\n");
  appendf(s, ".extern .shared .align 1024 .b8 smem[];\n\n");
  appendf(s,
          ".visible .entry srt_jit(\n  .param .align 64 .b8 p_tmap[128],\n  .param .u64 p_y,\n"
          "  .param .u64 p_ldy,\n  .param .u64 p_n\n)\n.maxntid %d, 1, 1\n{\n",
          (W + 1) * 32);
  appendf(s, "  .reg .pred %%p<8>;\n  .reg .pred %%pw;\n  .reg .pred %%pv;\n  .reg .pred %%pl;\n");
  appendf(s, "  .reg .b32 %%r<40>;\n  .reg .b32 %%xb<%d>;\n  .reg .b64 %%rd<16>;\n", ST);
  appendf(s, "  .reg .f32 %%a<%d>;\n  .reg .f32 %%x<16>;\n  .reg .b16 %%h<17>;\n", Mp);
  // preamble
  appendf(s,
          "  mov.u32 %%r0, %%tid.x;\n  shr.u32 %%r1, %%r0, 5;\n  and.b32 %%r2, %%r0, 31;\n"
          "  mov.u32 %%r3, %%ctaid.x;\n  mov.u32 %%r4, %%ctaid.y;\n  mov.u32 %%r5, smem;\n"
          "  add.u32 %%r6, %%r5, %d;\n  setp.ne.u32 %%p0, %%r0, 0;\n  @%%p0 bra INIT_DONE;\n",
          bar_off);
  for (int st = 0; st < ST; ++st) {
    appendf(s, "  mbarrier.init.shared::cta.b64 [%%r6+%d], 1;\n", 8 * st);
    appendf(s, "  mbarrier.init.shared::cta.b64 [%%r6+%d], %d;\n", 8 * (ST + st), W);
  }
  appendf(s,
          "  fence.mbarrier_init.release.cluster;\n  fence.proxy.async.shared::cta;\n"
          "INIT_DONE:\n  bar.sync 0;\n  mul.wide.u32 %%rd0, %%r3, %d;\n"
          "  setp.eq.u32 %%p1, %%r1, %d;\n  @%%p1 bra PRODUCER;\n",
          NT, W);
  // consumer preamble
  appendf(s,
          "  mad.lo.u32 %%r7, %%r1, 32, %%r2;\n  cvt.u64.u32 %%rd1, %%r7;\n  add.u64 %%rd2, %%rd0, %%rd1;\n"
          "  ld.param.u64 %%rd3, [p_n];\n  setp.lt.u64 %%pv, %%rd2, %%rd3;\n"
          "  ld.param.u64 %%rd4, [p_y];\n  ld.param.u64 %%rd5, [p_ldy];\n"
          "  mad.lo.u64 %%rd6, %%rd2, %d, %%rd4;\n  mad.lo.u32 %%xb0, %%r7, %d, %%r5;\n",
          S, S);
  for (int st = 1; st < ST; ++st) appendf(s, "  add.u32 %%xb%d, %%xb0, %d;\n", st, st * stage_bytes);
  appendf(s, "  setp.eq.u32 %%pl, %%r2, 0;\n");
  // panel dispatch
  if (pe - pb > 1) {
    appendf(s, "  TS: .branchtargets ");
    for (int q = pb; q < pe; ++q) appendf(s, "%sPANEL_%d", q == pb ? "" : ", ", q);
    appendf(s, ";\n  brx.idx.uni %%r4, TS;\n");
  }
  std::vector<std::tuple<int, int, float>> cz;  // (k, slot, w) of one chunk
  for (int q = pb; q < pe; ++q) {
    appendf(s, "PANEL_%d:\n", q);
    for (int r = 0; r < Mp; ++r) appendf(s, "  mov.f32 %%a%d, 0f00000000;\n", r);
    // per-row cursors
    std::vector<size_t> cur(Mp, 0);
    int xi = 0;
    for (int c = 0; c < nch; ++c) {
      const int st = c % ST, par = (c / ST) & 1;
      const int k0 = c * kc, k1 = std::min(p.K, k0 + kc);
      appendf(s, "W_%d_%d:\n  mbarrier.try_wait.parity.shared::cta.b64 %%pw, [%%r6+%d], %d;\n"
                 "  @!%%pw bra W_%d_%d;\n", q, c, 8 * st, par, q, c);
      cz.clear();
      for (int r = 0; r < Mp; ++r) {
        const int32_t m = p.jit_row_id[(size_t)q * Mp + r];
        if (m < 0) continue;
        const auto& rr = rows[m];
        size_t& i = cur[r];
        while (i < rr.size() && rr[i].k < k1) {
          cz.emplace_back(rr[i].k, r, rr[i].w);
          ++i;
        }
      }
      std::sort(cz.begin(), cz.end(), [](const auto& a, const auto& b) {
        return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b)
                                                : std::get<1>(a) < std::get<1>(b);
      });
      size_t e = 0;
      while (e < cz.size()) {
        const int k = std::get<0>(cz[e]);
        const int off = (k - k0) * NT * S;
        const int xr = xi++ & 15;
        if (f16) {
          appendf(s, "  ld.shared.b16 %%h%d, [%%xb%d+%d];\n  cvt.f32.f16 %%x%d, %%h%d;\n", xr, st, off,
                  xr, xr);
        } else {
          appendf(s, "  ld.shared.f32 %%x%d, [%%xb%d+%d];\n", xr, st, off);
        }
        for (; e < cz.size() && std::get<0>(cz[e]) == k; ++e) {
          appendf(s, "  fma.rn.f32 %%a%d, %%x%d, 0f%08X, %%a%d;\n", std::get<1>(cz[e]), xr,
                  fbits(std::get<2>(cz[e])), std::get<1>(cz[e]));
          ++fmas;
        }
      }
      appendf(s, "  bar.warp.sync -1;\n  @%%pl mbarrier.arrive.shared::cta.b64 _, [%%r6+%d];\n",
              8 * (ST + st));
    }
    // epilogue: Y[row][n] = acc (fp16: round once)
    for (int r = 0; r < Mp; ++r) {
      const int32_t m = p.jit_row_id[(size_t)q * Mp + r];
      if (m < 0) continue;
      appendf(s, "  mad.lo.u64 %%rd7, %%rd5, %d, %%rd6;\n", m);
      if (f16) {
        appendf(s, "  cvt.rn.f16.f32 %%h16, %%a%d;\n  @%%pv st.global.b16 [%%rd7], %%h16;\n", r);
      } else {
        appendf(s, "  @%%pv st.global.f32 [%%rd7], %%a%d;\n", r);
      }
    }
    appendf(s, "  bra.uni DONE;\n");
  }
  // producer: lane 0 issues one TMA box per chunk into the ring
  appendf(s,
          "PRODUCER:\n  setp.ne.u32 %%p2, %%r2, 0;\n  @%%p2 bra DONE;\n"
          "  mov.b64 %%rd8, p_tmap;\n  cvta.param.u64 %%rd8, %%rd8;\n  cvt.u32.u64 %%r8, %%rd0;\n"
          "  mov.u32 %%r9, 0;\nPLOOP:\n  setp.ge.u32 %%p3, %%r9, %d;\n  @%%p3 bra DONE;\n"
          "  and.b32 %%r10, %%r9, %d;\n  shr.u32 %%r11, %%r9, %d;\n  shl.b32 %%r12, %%r10, 3;\n"
          "  add.u32 %%r13, %%r6, %%r12;\n  add.u32 %%r14, %%r13, %d;\n"
          "  setp.lt.u32 %%p4, %%r9, %d;\n  @%%p4 bra PNW;\n  sub.u32 %%r15, %%r11, 1;\n"
          "  and.b32 %%r15, %%r15, 1;\nPWAIT:\n"
          "  mbarrier.try_wait.parity.shared::cta.b64 %%p5, [%%r14], %%r15;\n  @!%%p5 bra PWAIT;\n"
          "PNW:\n  mbarrier.arrive.expect_tx.shared::cta.b64 _, [%%r13], %d;\n"
          "  mul.lo.u32 %%r16, %%r9, %d;\n  mad.lo.u32 %%r17, %%r10, %d, %%r5;\n"
          "  cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
          "[%%r17], [%%rd8, {%%r8, %%r16}], [%%r13];\n"
          "  add.u32 %%r9, %%r9, 1;\n  bra.uni PLOOP;\nDONE:\n  ret;\n}\n",
          nch, ST - 1, lg_st, 8 * ST, ST, stage_bytes, kc, stage_bytes);
}

}  // namespace

int jit_generate(Plan& p, const std::vector<std::vector<RowEntry>>& rows, const BuildOpts& o,
                 std::string& err) {
  const bool f16 = p.dtype == SPARSE_F16;
  const int S = f16 ? 2 : 4;
  const int64_t nh = o.n_hint > 0 ? o.n_hint : 4096;
  const int M = p.M;
  // tile selection: largest Mp (fewest re-reads of X from L2) and widest N tile that
  // still gives >= one wave of CTAs on 148 SMs
  int W = 4, Mp = 128;
  bool found = false;
  for (int w : {4, 2, 1}) {
    for (int mp : {128, 96, 64, 48, 32, 16}) {
      const int64_t ctas = ((M + mp - 1) / mp) * ((nh + 32 * w - 1) / (32 * w));
      if (ctas >= 148) {
        W = w;
        Mp = mp;
        found = true;
        break;
      }
    }
    if (found) break;
  }
  if (!found) {
    W = 1;
    Mp = 16;
  }
  Mp = std::min(Mp, (M + 15) / 16 * 16);
  if (o.jit_rows) Mp = o.jit_rows;
  if (o.jit_warps) W = o.jit_warps;
  if (Mp < 1 || Mp > 192 || (W != 1 && W != 2 && W != 4 && W != 8)) {
    err = "jit: rows must be in [1, 192] and warps 1, 2, 4 or 8";
    return SPARSE_EUNSUPPORTED;
  }
  p.jit_mp = Mp;
  p.jit_warps = W;
  p.jit_kc = 32;
  const int nch = (p.K + p.jit_kc - 1) / p.jit_kc;
  p.jit_stages = nch >= 4 ? 4 : nch >= 2 ? 2 : 1;
  p.jit_smem = p.jit_stages * p.jit_kc * 32 * W * S + 16 * p.jit_stages;
  p.jit_npanels = (M + Mp - 1) / Mp;
  // LPT row panels (same rule as the plan-driven inspector)
  std::vector<int32_t> order(M);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return rows[a].size() > rows[b].size(); });
  using PI = std::pair<int64_t, int32_t>;
  std::priority_queue<PI, std::vector<PI>, std::greater<PI>> heap;
  for (int32_t q = 0; q < p.jit_npanels; ++q) heap.push({0, q});
  std::vector<int> fill(p.jit_npanels, 0);
  std::vector<int64_t> pnnz(p.jit_npanels, 0);
  p.jit_row_id.assign((size_t)p.jit_npanels * Mp, -1);
  for (int32_t m : order) {
    PI top = heap.top();
    heap.pop();
    const int q = top.second;
    p.jit_row_id[(size_t)q * Mp + fill[q]++] = m;
    pnnz[q] += (int64_t)rows[m].size();
    if (fill[q] < Mp) heap.push({pnnz[q], q});
  }
  // modules: consecutive panels, ~24K FMAs each (parallel ptxas)
  p.jit.clear();
  int q = 0;
  while (q < p.jit_npanels) {
    Plan::JitModule jm;
    jm.panel_begin = q;
    int64_t acc = 0;
    while (q < p.jit_npanels && (acc == 0 || acc + pnnz[q] <= 24000) && q - jm.panel_begin < 4096) {
      acc += pnnz[q];
      ++q;
    }
    jm.npanels = q - jm.panel_begin;
    p.jit.push_back(std::move(jm));
  }
  for (auto& jm : p.jit) {
    int64_t f = 0;
    emit_module(jm.ptx, p, jm.panel_begin, jm.panel_begin + jm.npanels, rows, f);
    jm.fmas = f;
  }
  p.executor = 1;
  return SPARSE_OK;
}

int jit_compile(Plan& p, std::string& err) {
  const auto t0 = std::chrono::steady_clock::now();
  std::atomic<int> next{0};
  std::mutex emu;
  std::string first_err;
  auto work = [&] {
    for (;;) {
      const int i = next++;
      if (i >= (int)p.jit.size()) return;
      auto& jm = p.jit[i];
      nvPTXCompilerHandle h = nullptr;
      std::string e;
      if (nvPTXCompilerCreate(&h, jm.ptx.size(), jm.ptx.c_str()) != NVPTXCOMPILE_SUCCESS) {
        e = "nvPTXCompilerCreate failed";
      } else {
        const char* opts[] = {"--gpu-name=sm_100a", "-O3"};
        if (nvPTXCompilerCompile(h, 2, opts) != NVPTXCOMPILE_SUCCESS) {
          size_t n = 0;
          nvPTXCompilerGetErrorLogSize(h, &n);
          std::string log(n, '\0');
          if (n) nvPTXCompilerGetErrorLog(h, &log[0]);
          e = "ptx compile failed: " + log.substr(0, 2000);
        } else {
          size_t n = 0;
          nvPTXCompilerGetCompiledProgramSize(h, &n);
          jm.cubin.resize(n);
          nvPTXCompilerGetCompiledProgram(h, jm.cubin.data());
        }
        nvPTXCompilerDestroy(&h);
      }
      if (!e.empty()) {
        std::lock_guard<std::mutex> lk(emu);
        if (first_err.empty()) first_err = e;
      }
    }
  };
  unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
  nt = std::min<unsigned>(nt, (unsigned)p.jit.size());
  std::vector<std::thread> th;
  for (unsigned i = 1; i < nt; ++i) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  p.jit_compile_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (!first_err.empty()) {
    err = first_err;
    return SPARSE_EINTERNAL;
  }
  p.jit_cubin_bytes = 0;
  const char* dump = std::getenv("SPARSERT_JIT_DUMP");  // debugging / profiling aid
  for (size_t i = 0; i < p.jit.size(); ++i) {
    auto& jm = p.jit[i];
    p.jit_cubin_bytes += (int64_t)jm.cubin.size();
    if (dump && *dump) {
      const std::string base = std::string(dump) + "/srt_jit_" + std::to_string(p.digest) + "_" +
                               std::to_string(i);
      if (FILE* f = std::fopen((base + ".ptx").c_str(), "wb")) {
        std::fwrite(jm.ptx.data(), 1, jm.ptx.size(), f);
        std::fclose(f);
      }
      if (FILE* f = std::fopen((base + ".cubin").c_str(), "wb")) {
        std::fwrite(jm.cubin.data(), 1, jm.cubin.size(), f);
        std::fclose(f);
      }
    }
    std::string().swap(jm.ptx);  // the cubin is what is kept
  }
  return SPARSE_OK;
}

int jit_load(Plan& p, std::string& err) {
  const DriverApi& d = driver();
  if (!d.ok) {
    err = "jit: driver entry points unavailable";
    return SPARSE_ECUDA;
  }
  for (auto& jm : p.jit) {
    CUmodule mod;
    CUresult r = d.moduleLoadData(&mod, jm.cubin.data());
    if (r != CUDA_SUCCESS) {
      char buf[96];
      snprintf(buf, sizeof buf, "jit: cuModuleLoadData failed (%d)", (int)r);
      err = buf;
      return SPARSE_ECUDA;
    }
    CUfunction fn;
    r = d.moduleGetFunction(&fn, mod, "srt_jit");
    if (r == CUDA_SUCCESS)
      r = d.funcSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, p.jit_smem);
    if (r != CUDA_SUCCESS) {
      d.moduleUnload(mod);
      err = "jit: cuModuleGetFunction/cuFuncSetAttribute failed";
      return SPARSE_ECUDA;
    }
    jm.mod = (void*)mod;
    jm.fn = (void*)fn;
  }
  return SPARSE_OK;
}

void jit_unload(Plan& p) {
  const DriverApi& d = driver();
  for (auto& jm : p.jit) {
    if (jm.mod && d.ok) d.moduleUnload((CUmodule)jm.mod);
    jm.mod = jm.fn = nullptr;
  }
}

int64_t jit_panel_code_bytes(const Plan& p) {
  int64_t maxf = 0;
  for (const auto& jm : p.jit) maxf = std::max<int64_t>(maxf, jm.fmas / std::max(1, jm.npanels));
  return maxf * 16;  // one 16-byte FFMA per nonzero dominates the code
}

bool jit_can_launch(const Plan& p, const void* X, int64_t ldx) {
  const int S = p.dtype == SPARSE_F16 ? 2 : 4;
  return p.executor == 1 && !p.jit.empty() && p.jit[0].fn != nullptr && driver().ok &&
         ((uintptr_t)X % 16 == 0) && ((ldx * S) % 16 == 0);
}

int jit_launch(const Plan& p, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy,
               void* stream, std::string& err) {
  const DriverApi& d = driver();
  const bool f16 = p.dtype == SPARSE_F16;
  const int S = f16 ? 2 : 4;
  const int NT = 32 * p.jit_warps;
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof tmap);
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)p.K};
  cuuint64_t strides[1] = {(cuuint64_t)(ldx * S)};
  cuuint32_t box[2] = {(cuuint32_t)NT, (cuuint32_t)p.jit_kc};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = d.tensorMapEncodeTiled(
      &tmap, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
      const_cast<void*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "jit: cuTensorMapEncodeTiled failed";
    return SPARSE_ECUDA;
  }
  uint64_t yp = (uint64_t)Y, ldy_b = (uint64_t)(ldy * S), n = (uint64_t)N;
  void* params[] = {&tmap, &yp, &ldy_b, &n};
  const int64_t ntn = (N + NT - 1) / NT;
  if (ntn > 0x7fffffff) {
    err = "jit: N too large";
    return SPARSE_EUNSUPPORTED;
  }
  for (const auto& jm : p.jit) {
    // row ids are baked per panel; the module's panels are consecutive in Y rows via
    // immediates, so only the grid changes between modules
    r = d.launchKernel((CUfunction)jm.fn, (unsigned)ntn, (unsigned)jm.npanels, 1,
                       (unsigned)((p.jit_warps + 1) * 32), 1, 1, (unsigned)p.jit_smem,
                       (CUstream)stream, params, nullptr);
    if (r != CUDA_SUCCESS) {
      char buf[96];
      snprintf(buf, sizeof buf, "jit: cuLaunchKernel failed (%d)", (int)r);
      err = buf;
      return SPARSE_ECUDA;
    }
  }
  return SPARSE_OK;
}

}  // namespace srt
