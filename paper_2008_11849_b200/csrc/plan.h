// Internal plan representation shared by the host inspector (inspector.cpp),
// the C ABI (capi.cpp) and the executor kernels (kernels.cu).
//
// A plan is the paper's compile-time artefact (Sec. 2.3, Sec. 3.4):
// the sparse weight matrix after block-level load balancing (row panels,
// strategy (b) of Fig. 2b), thread-group assignment (rows per warp,
// optional split-K groups) and K-chunking, packed so that one
// (panel, chunk) block is a single contiguous, 16-byte aligned byte range that
// a CTA stages into shared memory next to the X tile it multiplies.
//
// Block layout (byte offsets relative to blob + blk_off[panel*nchunks+chunk]).
//
// SpMM plans (kernel spmm_kernel): every block occupies max_blk_bytes (fixed stride,
// block bi at bi * max_blk_bytes, zero padded) so its address needs no table lookup.
//   uint32 hdr[Mp * gk]        unit_start | unit_count << 16 of thread group g of
//                              row slot s = warp*R + r at index s*gk + g; a "unit"
//                              is one 16-byte broadcast load = entry_align entries;
//                              unit_start is relative to the block's entry array;
//                              padded to 16 B
//   units[...]                 slot-major, group-major inside a slot, k ascending
//                              fp32: {uint32 xoff; float w} x 2 per unit, xoff =
//                                    k_local * n_tile * 4 (byte offset of X row k
//                                    inside the staged tile)
//                              fp16: {uint16 xoff16; half w} x 4 per unit, xoff16 =
//                                    k_local * n_tile * 2 / 16 (16-byte units)
//                              a group's last unit is completed with neutral
//                              entries {xoff of row k_local = kc (the zero row
//                              every stage carries after its kc X rows), w = -0.0}:
//                              fma(-0, +0, acc) == acc bit for bit, so padding
//                              never changes a result
//   The split of a row's chunk entries into gk groups: every group but the last
//   takes per = ceil(cnt / gk) rounded up to entry_align entries (Fig. 3b).
//
// Conv plans (kernel conv3x3_kernel):
//   uint32 slot_hdr[Mp]        start | count << 16 in entries, start a multiple of
//                              entry_align; padded to 16 B
//   entries[...]               fp32 {int32 smem_off; float w} (8 B),
//                              fp16 {int16 smem_off; half w} (4 B), row-slot-major,
//                              k ascending, zero padding between slots
//   zero padding to 16 bytes
//
// Vectorised conv plans (conv_vec 1 / 2 / 4) use the SpMM unit format above with the entry
// offset pointing into the staged shifted copies (kernels.cu); interleaved conv plans
// (conv_vec 4) with 16-bit values carry the offset in 8-byte units.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace srt {

constexpr int kMaxWarps = 16;
constexpr int kMaxStages = 8;

struct Plan {
  // problem
  int32_t M = 0, K = 0, dtype = 0, kind = 0;
  int32_t c_in = 0, h = 0, w = 0;
  int64_t nnz = 0;
  int64_t n_hint = 0;

  // tiling (thread block = `warps` thread groups of 32/gk lanes x gk groups)
  int32_t warps = 4;     // consumer warps per CTA (SpMM adds one producer warp)
  int32_t R = 4;         // row slots per warp
  int32_t Mp = 16;       // rows per panel = warps * R
  int32_t gk = 1;        // split-K groups per warp
  int32_t C = 4;         // columns (SpMM) / positions (conv) per lane
  int32_t n_tile = 128;  // columns per CTA (SpMM) / tile positions (conv)
  int32_t kc = 64;       // K rows per chunk (SpMM) ; conv: K rows = 9 * cc
  int32_t cc = 0;        // conv: input channels per chunk
  int32_t nchunks = 1;
  int32_t npanels = 1;
  int32_t entry_bytes = 8;
  int32_t entry_align = 2;  // entries per 16-byte broadcast load
  int32_t hdr_bytes = 16;   // block header bytes (slot table)
  int32_t ks = 1;           // cluster K-split: CTAs of a cluster take disjoint chunk ranges
  int32_t cm = 1;           // X multicast cluster: CTAs (consecutive panels) sharing X tiles
  int32_t row_order = 0;    // 0 = LPT load balancing (default), 1 = natural order (ablation)
  int32_t tm = 0;           // X source: 0 = shared memory, 1 = tensor memory (tcgen05.ld)
  int32_t ps = 0;           // plan source: 0 = staged per chunk with X, 1 = kernel parameters

  // conv geometry (kind == CONV3X3)
  int32_t conv_rb = 0;    // output rows per tile
  int32_t conv_ipt = 0;   // images per tile
  int32_t conv_wp = 0;    // padded row length W + 2
  int32_t conv_simg = 0;  // smem elements per (ci, image) = (rb + 2) * wp
  int32_t conv_sci = 0;   // smem elements per ci = ipt * simg
  int32_t conv_guard = 0; // guard elements before/after the stage
  int32_t conv_stage_elems = 0;
  int32_t conv_vec = 0;   // 1: vectorised kernel (three dx-shifted copies, SpMM unit entries)
  int32_t conv_cs = 0;    // vectorised: elements per shifted copy = cc * conv_sci
  // interleaved conv (conv_vec == 4, conv3x3_il_kernel): il_g images interleaved per row group
  // (pitch il_g * w), per chunk three TMA boxes of il_lc elements x cc channels (copy dx at
  // dx * conv_cs elements), a zero block of il_lc, then the plan block at il_blk_at bytes
  int32_t il_g = 0, il_lc = 0, il_stage_bytes = 0, il_blk_at = 0;
  // conv on the tcgen05 block executor (executor 4, conv_kernel 5): images per row group of the
  // interleaved copies (pitch tcg_g * w a multiple of 8 elements: 16-byte TMA box starts)
  int32_t tcg_g = 0, tcg_ncb = 0;
  // tcgen05 block executor: CTAs per cluster (tcg_cs consecutive 128-row blocks = one group
  // that shares every X tile through TMA multicast; each CTA loads 1 / tcg_cs of it), the
  // number of groups, and the k-block depth (64 for 16-bit data, 32 for fp32 = 3xTF32)
  int32_t tcg_cs = 1, tcg_ngroups = 0, tcg_bk = 64;
  // CTA pairs (tcg_cs = 2): one cta_group::2 M = 256 MMA per step, each CTA stages its W block
  // and half of the X tile
  int32_t tcg_pair = 0;
  // K slices per tile (k_split for executor 4): fp32 partials to a workspace, then tcg_ksum
  int32_t tcg_ks = 1;

  // packed plan (host copy)
  std::vector<int32_t> row_id;   // npanels * Mp, -1 = empty slot
  std::vector<int64_t> blk_off;  // npanels * nchunks + 1 byte offsets into blob
  std::vector<uint8_t> blob;
  int32_t max_blk_bytes = 0;
  int32_t x_stage_bytes = 0;     // bytes of the staged X tile per stage
  int32_t smem_bytes = 0;        // dynamic smem per CTA (all stages)
  int32_t stages = 2;
  int32_t red_bytes = 0;         // smem for the cross-CTA (DSMEM) reduction tile

  // stats
  int64_t max_panel_nnz = 0, min_panel_nnz = 0;
  double build_ms = 0.0;
  uint64_t digest = 0;

  // JIT executor (the paper's unrolled, value-baked code generator, Sec. 3.5
  // P:183-185): per row panel, straight-line PTX that walks the panel's K
  // union in ascending order, loads X[k, lane column] once and issues one FFMA
  // with the weight as an immediate per nonzero of column k (Alg. 3).
  int32_t executor = 0;      // 0 = plan-driven kernels, 1 = JIT, 3 = tensor-core condensed panels
  struct JitModule {
    std::string ptx;
    std::vector<char> cubin;
    int32_t panel_begin = 0, npanels = 0;
    int64_t fmas = 0;
    void* mod = nullptr;  // CUmodule
    void* fn = nullptr;   // CUfunction
  };
  std::vector<JitModule> jit;
  int32_t jit_mp = 0, jit_warps = 0, jit_kc = 0, jit_stages = 0, jit_npanels = 0;
  int32_t jit_smem = 0;
  std::vector<int32_t> jit_row_id;  // jit_npanels * jit_mp
  double jit_compile_ms = 0.0;
  double tuned_us = 0.0;  // autotuner: measured time of the chosen configuration
  int64_t jit_cubin_bytes = 0;

  // device copy
  int device = -1;
  void* d_mem = nullptr;
  const int32_t* d_row_id = nullptr;
  const int64_t* d_blk_off = nullptr;
  const uint8_t* d_blob = nullptr;
  int64_t plan_bytes = 0;
  mutable int32_t grid_cache = 0;  // resident CTAs (clusters) of the persistent launch

  // Tensor-core sub-block path (fp16 SpMM plans): aligned 16 x 16 tiles of W
  // with at least tc_min_pct % nonzeros are taken out of the CUDA-core plan and multiplied
  // as dense blocks with mma.sync m16n8k16 (fp16 x fp16 -> fp32) into an fp32 workspace that
  // the CUDA-core kernel adds before its single rounding.
  int32_t tc_min_pct = 0;
  int32_t tc_nrb = 0;                // row blocks (16 rows) holding >= 1 dense tile
  int64_t tc_ntiles = 0;
  int64_t tc_nnz = 0;                // nonzeros carried by the dense tiles
  std::vector<int32_t> tc_rb;        // [tc_nrb] row-block index (rows 16 rb .. 16 rb + 15)
  std::vector<int32_t> tc_tile_begin;  // [tc_nrb + 1] tile ranges, k-block ascending
  std::vector<int32_t> tc_cb;        // [tc_ntiles] k-block index (K columns 16 cb ..)
  std::vector<uint16_t> tc_a;        // [tc_ntiles][32 lanes][8] fp16, mma A-fragment order
  std::vector<int32_t> ws_row;       // [M] workspace row of W row m, or -1
  const int32_t* d_tc_rb = nullptr;
  const int32_t* d_tc_tile_begin = nullptr;
  const int32_t* d_tc_cb = nullptr;
  const uint16_t* d_tc_a = nullptr;
  const int32_t* d_ws_row = nullptr;

  // Condensed-panel tensor-core executor (executor = 3; fp16 SpMM): panel q =
  // rows 16 q .. 16 q + 15 (group G = q / kTcpPanels, i = q % kTcpPanels); chunk c = K rows
  // kTcpKc c ..; its steps are the bytes [off[(G nch + c)(kTcpPanels + 1) + i], ... + i + 1)
  // of tcp_steps; one step = the mma A fragment (32 lanes x 8 fp16) of W[16 rows x 16 union
  // slots] + the 16 slot rows (uint8 k_local): packed (SRT_TCP_PACK, inspector.cpp: per-lane
  // masks + the nonzero halves) or dense (kTcpStepBytes); one group's chunk is contiguous
  int32_t tcp_npanels = 0, tcp_nchunks = 0, tcp_max_blk = 0;
  int64_t tcp_nsteps = 0;
  std::vector<int32_t> tcp_step_off;
  std::vector<uint8_t> tcp_steps;
  const int32_t* d_tcp_step_off = nullptr;
  const uint8_t* d_tcp_steps = nullptr;
};
#ifndef SRT_TCP_KC
#define SRT_TCP_KC 64
#endif
constexpr int kTcpKc = SRT_TCP_KC;  // K rows per staged chunk (TMA box rows, 128-byte swizzled)
#ifndef SRT_TCP_PANELS
#define SRT_TCP_PANELS 8
#endif
#ifndef SRT_TCP_STRICT
#define SRT_TCP_STRICT 1
#endif
constexpr int kTcpPanels = SRT_TCP_PANELS;  // panels (warps) per CTA
constexpr int kTcpStepBytes = 528;  // dense step: 512 B A fragment + 16 B slot rows
#ifndef SRT_TCP_PACK
#define SRT_TCP_PACK 0
#endif

struct BuildOpts {
  int32_t kind = 0, c_in = 0, h = 0, w = 0;
  int64_t n_hint = 0;
  int32_t drop_zeros = 0;
  int32_t warps = 0, rows_per_warp = 0, k_chunk = 0, split_k = 0;
  int32_t k_split = 0, stages = 0;
  int32_t executor = 0, jit_rows = 0, jit_warps = 0;
  int32_t cm = 0;
  int32_t tm = 0;
  int32_t conv_vec = 1;   // allow the vectorised conv kernel
  int32_t row_order = 0;  // 0 = LPT panels (load balancing), 1 = natural contiguous rows
  int32_t tc_min_pct = 50;  // tensor-core sub-blocks: min % of nonzeros in a 16x16 tile (0 = off)
  int32_t ps = 0;           // plan source (sparse_plan_opts.plan_source)
  int32_t pair = 0;         // executor 4: CTA pairs (sparse_plan_opts.cta_pair)
};

// JIT executor (jit.cpp).  Row entries per row (k ascending) as validated by the
// inspector; builds jit_row_id and one PTX module per group of panels.
struct RowEntry {
  int32_t k;
  float w;
};
int jit_generate(Plan& p, const std::vector<std::vector<RowEntry>>& rows, const BuildOpts& o,
                 std::string& err);
int jit_compile(Plan& p, std::string& err);  // PTX -> cubin (host only, no GPU needed)
int jit_load(Plan& p, std::string& err);     // cubin -> CUmodule on p.device
void jit_unload(Plan& p);
int jit_launch(const Plan& p, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy,
               void* stream, std::string& err);
bool jit_can_launch(const Plan& p, const void* X, int64_t ldx);
// Per-panel straight-line code size (bytes) of a JIT plan, max over modules.
int64_t jit_panel_code_bytes(const Plan& p);

// Autotuner (tune.cu): builds, uploads and times every candidate on `device` and
// leaves the fastest (uploaded, JIT loaded) in `best`.
int tune_plan(Plan& best, int32_t M, int32_t K, int64_t nnz, const int32_t* row_ptr,
              const int32_t* col_idx, const float* values, int32_t dtype, const BuildOpts& base,
              int device, std::string& err);

// Inspector: validate the CSR (a1), group rows into nnz-balanced panels (a2),
// choose split-K / chunking (a3, a5) and pack (a4).  Returns a sparse_status
// code; on error `err` holds the detail.
int build_plan(Plan& p, int32_t M, int32_t K, int64_t nnz, const int32_t* row_ptr,
               const int32_t* col_idx, const float* values, int32_t dtype,
               const BuildOpts& o, std::string& err);

// fp32 -> fp16 bits, round-to-nearest-even (host side, exact IEEE semantics).
uint16_t f32_to_f16_rn(float f);
float f16_to_f32(uint16_t h);

// Device side (kernels.cu)
int upload_plan(Plan& p, std::string& err);
void free_plan_device(Plan& p);
struct Epilogue {  // Y = act(acc + bias + beta * Y); see sparse_epilogue
  float beta = 0.0f;
  const void* bias = nullptr;
  int32_t relu = 0;
  bool trivial() const { return beta == 0.0f && bias == nullptr && relu == 0; }
};
int launch_spmm(const Plan& p, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy,
                void* stream, std::string& err, const Epilogue& ep = Epilogue());
int launch_conv3x3_nhwc(const Plan& p, int64_t batch, const void* x, void* y, void* stream, std::string& err);
int launch_conv3x3(const Plan& p, int64_t batch, const void* x, void* y, void* stream,
                   std::string& err, const Epilogue& ep = Epilogue());
// Unaligned X (base or row stride not a 16-byte multiple): stream-ordered copy into a
// padded scratch buffer so the TMA paths apply; free_repack releases it (stream-ordered).
int launch_repack(int device, int64_t K, int64_t N, int S, const void* X, int64_t ldx, void** Xp,
                  int64_t* ldp, void* stream, std::string& err);
void free_repack(int device, void* Xp, void* stream);
// xs[k][(b ho + oy) wo + ox] = x[k][b][oy s][ox s] (x CNHW [K][B][h][w]), stream ordered
int launch_stride_gather(int device, int S, const void* x, int64_t K, int64_t B, int h, int w, int s, void* xs,
                         void* stream, std::string& err);
// out[c][r] = in[r][c] for a rows x cols matrix (element size S), stream ordered
int launch_transpose(int device, int S, const void* in, int64_t ldi, void* out, int64_t ldo, int64_t rows,
                     int64_t cols, void* stream, std::string& err);

}  // namespace srt
