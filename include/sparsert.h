/*
 * sparsert.h — C ABI of the B200-native SparseRT hot path (arXiv 2008.11849).
 *
 * The operation (Sec. 3.2 "Terminology"):  A x B = C with the
 * sparse matrix A = W (M x K, pruned, pattern fixed before inference) and the
 * dense matrix B = X (K x N), C = Y (M x N), "C-style row-major default layout".
 * Batch is folded into N (N = batch*H*W for 1x1 convs, batch*seq for FC layers).
 * Sparse 3x3 convolutions are the same SpMM on a "virtual" im2col B
 * (Sec. 3.6).
 *
 * Inspector / executor split (Sec. 2.3): sparse_plan_create is the
 * offline inspector (validation, row grouping, nnz-balanced row panels, K
 * chunking and packing, tile selection; Sec. 3.4, Sec. 3.7
 * P:259-263); sparse_spmm / sparse_conv3x3 are the executors (Alg. 3,
 * P:187-206), launched asynchronously on the caller's CUDA stream.
 *
 * All entry points are extern "C", never throw, and return a sparse_status.
 * A failing call leaves a thread-local human-readable detail retrievable with
 * sparse_last_error().  No entry point ever falls back to a CPU computation.
 */
#ifndef SPARSERT_H_
#define SPARSERT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t is passed as an opaque pointer so this header does not need the
 * CUDA headers; 0 / NULL means the legacy default stream of the current thread. */
typedef void* sparse_stream_t;

typedef struct sparse_plan_s* sparse_plan_t; /* opaque, immutable after create */

enum sparse_status {
  SPARSE_OK = 0,
  SPARSE_EINVAL = 1,       /* bad argument: null pointer, negative/zero dim, bad dtype/kind,
                              misuse (conv call on an SpMM plan, compute on a host-only plan) */
  SPARSE_EMATRIX = 2,      /* invalid CSR: row_ptr[0] != 0, row_ptr not monotone, row_ptr[M] != nnz,
                              col_idx out of [0,K), columns not strictly increasing within a row
                              (unsorted or duplicate), non-finite value, explicit zero (unless
                              opts->drop_zeros), a value that rounds to fp16 infinity
                              (|value| >= 65520) for an fp16 plan.  The detail
                              names the row. */
  SPARSE_EUNSUPPORTED = 3, /* e.g. K > 65535, conv with K != 9*c_in, tile override out of range */
  SPARSE_ENOMEM = 4,       /* host or device allocation failed */
  SPARSE_ECUDA = 5,        /* CUDA error (no device, launch failure); detail in sparse_last_error() */
  SPARSE_EINTERNAL = 6
};

/* X, Y and the plan's values share the dtype; accumulation is always fp32.
 * SPARSE_F16: W is rounded to fp16 (RN-even) at plan time; each product
 * f16 x f16 is exact in fp32; Y is rounded RN-even to fp16 once.
 * SPARSE_BF16 (NEXT #4): the same with bfloat16 (FHFMA.BF16 / mma .bf16): SpMM on the CUDA-core
 * kernels or the tensor-core panels (executor 3), conv on the TMA-fed kernel (JIT, dense-tile
 * tensor cores, the TMEM X source and the other conv kernels: EUNSUPPORTED). */
enum sparse_dtype { SPARSE_F32 = 0, SPARSE_F16 = 1, SPARSE_BF16 = 2 };
enum sparse_kind { SPARSE_SPMM = 0, SPARSE_CONV3X3 = 1 };

/* Device value for a host-only plan: the inspector runs and the plan can be
 * inspected (sparse_plan_info / sparse_plan_dump) but nothing is uploaded and
 * the compute calls return SPARSE_EINVAL.  Used by CPU-only tests. */
#define SPARSE_DEVICE_HOST_ONLY (-2)

typedef struct {
  int32_t kind;       /* SPARSE_SPMM (default) | SPARSE_CONV3X3 */
  int32_t c_in, h, w; /* conv only: K must equal 9*c_in; H, W fixed at plan time (the paper
                         specialises each kernel to its problem shape) */
  int64_t n_hint;     /* expected N (SpMM) or batch (conv); 0 = unknown.  Drives the tile heuristic. */
  int32_t tune;       /* 0 = heuristic; 1 = timed search over <= 100 candidates on the
                         plan's device with synthetic X of n_hint columns (tile parameters,
                         cluster K-split, split-K groups, JIT executor); requires n_hint > 0.
                         The choice depends on measured times, so two tuned plans of one matrix
                         may differ in summation order (pass the chosen options explicitly to
                         build identical replicas). */
  int32_t device;     /* CUDA ordinal; -1 = current device; SPARSE_DEVICE_HOST_ONLY = no upload */
  int32_t drop_zeros; /* 0 = reject explicit zeros; 1 = drop them */
  /* Tile overrides (0 = automatic).  None of these changes a result except split_k,
     k_chunk and k_split, which fix the per-row summation order. */
  int32_t warps;         /* warps per CTA (thread groups of the paper's block): 1..16 */
  int32_t rows_per_warp; /* R: 1, 2, 4, 8 or 16 (R * cols_per_lane <= 128) */
  int32_t k_chunk;       /* Kc: K rows staged per pipeline stage (SpMM: multiple of 8, 8..256);
                            conv: input channels per stage (1..64) */
  int32_t split_k;       /* G_k thread groups splitting each row's nonzeros: 1,2,4,8 */
  int32_t k_split;       /* SpMM: CTAs of a thread-block cluster splitting the K chunks, partial
                            tiles reduced in fixed rank order through distributed shared
                            memory (the paper's strategy (a), Fig. 2a): 1,2,4,8 */
  int32_t stages;        /* SpMM: X/plan pipeline stages (TMA + mbarrier ring): 1..8 */
  int32_t executor;      /* SpMM: 0 = plan-driven kernels (default); 2 = auto (JIT where each
                            panel's code is <= 24 KB, else plan-driven); 1 = JIT: the paper's code
                            generator (Sec. 3.5) - per row panel, straight-line PTX with
                            the weights as FFMA immediates, assembled in-process at plan creation
                            (slow to create: seconds for 10^5 nonzeros).  X that is not 16-byte
                            aligned falls back to the plan-driven kernels (same results, bitwise).
                            3 = tensor-core condensed panels (fp16 only): per 16-row
                            panel and 64-row K chunk the union of the panel's nonzero columns runs
                            as a dense mma.sync m16n8k16 block (fp32 accumulate) with the union's X
                            rows gathered by ldmatrix; summation order differs from the CUDA-core
                            kernels (within tolerance; exact on integer data).
                            4 = tcgen05 blocks (SURVEY NEXT #1 on Blackwell tensor cores): W's
                            nonzero 128-row x 64-column (fp32: 32-column) blocks stored dense and
                            pre-swizzled, tcgen05.mma M128 N256 with fp32 accumulators in TMEM;
                            fp16 / bf16 directly, fp32 as 3xTF32 (W and X each split into two
                            TF32 halves, W_hi X_hi + W_lo X_hi + W_hi X_lo: relative error
                            ~2^-22 per product; X is split on the device into a stream-ordered
                            scratch).  Summation order differs from the CUDA-core kernels
                            (within tolerance; exact on integer data). */
  int32_t jit_rows;      /* JIT: rows per panel (accumulator registers per thread), 0 = auto */
  int32_t jit_warps;     /* JIT: warps per CTA (each owns 32 columns), 0 = auto */
  int32_t x_multicast;   /* SpMM, k_split == 1: CTAs of a thread-block cluster (consecutive row
                            panels, same N tile) that share every staged X tile through one TMA
                            multicast load, dividing the L2 -> SM traffic of X: 1, 2, 4 or 8;
                            0 = 1.  Result-neutral.  With executor 4 (and conv_kernel 5): CTAs
                            of a cluster = consecutive 128-row blocks on the same N tile, each
                            loading 1 / x_multicast of every X tile and multicasting it (1, 2
                            or 4); the group walks the union of its row blocks' nonzero
                            k-blocks. */
  int32_t x_source;      /* SpMM: where the executor's FMA loop reads X from.  0 = shared memory
                            (LDS.128, default); 1 = tensor memory: every staged X chunk is copied
                            smem -> TMEM (tcgen05.cp, replicated to the 4 lane quarters) and read
                            with warp-uniform tcgen05.ld, which has ~2x the shared-memory
                            bandwidth.  Needs split_k = 1, k_split = 1,
                            x_multicast = 1, k_chunk <= 56 (default 56).  Result-neutral. */
  int32_t conv_kernel;   /* conv: 0 = auto (the TMA-fed vectorised kernel - three dx-shifted copies
                            of the staged input, 128-bit loads of C consecutive positions - when a
                            padded row of W + 2 positions fits twice in 32 * C positions, else the
                            position-strided kernel); 1 = position-strided kernel; 2 = TMA-fed
                            vectorised kernel: the shifted copies are written once to a stream-
                            ordered scratch by a pre-pass, then each is one 5-D TMA box per chunk;
                            3 = register-staged vectorised kernel; 4 = image-interleaved kernel:
                            g images side by side per row so that no output position is padding
                            (copies from a pre-pass, one TMA span box per copy and chunk; images
                            up to ~28 wide).  All result-identical.  5 = the tcgen05 block
                            executor (executor 4): implicit im2col over interleaved dx-shifted
                            copies, k-blocks = (tap, 64 channels; fp32: 32 channels as 3xTF32,
                            the pre-pass writes the copies split into TF32 halves); summation
                            order of the tensor cores (within tolerance; exact on integer data). */
  int32_t row_order;     /* 0 = load-balanced panels (rows sorted by nnz, LPT-binned, P:163-165;
                            default); 1 = natural contiguous row ranges (the "no load balancing"
                            ablation of P:385).  Result-neutral for split_k = k_split = 1. */
  int32_t tc_min_density; /* fp16 SpMM plans (not JIT): aligned 16 x 16 tiles of W holding at least
                            this % of nonzeros are multiplied as dense blocks on the tensor
                            cores (mma.sync m16n8k16, fp32 accumulate) and added to the CUDA-core
                            result before its single rounding.  0 = default
                            (50 %), -1 = off, 1..100 = threshold.  Changes the summation order
                            of the rows concerned (within tolerance; exact on integer data). */
  int32_t plan_source;   /* SpMM plan-driven executor: 0 = the plan's (panel, chunk) blocks are
                            staged into shared memory with each X chunk (default); 1 = the whole
                            plan (<= 30 KB) is passed as a kernel parameter and read through the
                            constant cache; the paper keeps A's values in the constant cache,
                            P:185.  Needs split_k = k_split = x_multicast = 1, x_source = 0,
                            no tensor-core sub-blocks.  Result-neutral (bitwise). */
  int32_t cta_pair;      /* executor 4 (tcgen05 blocks, SpMM and conv_kernel 5): 1 = CTA pairs -
                            the two CTAs of a 2-CTA cluster (two consecutive 128-row blocks) run
                            one tcgen05.mma.cta_group::2 M = 256 per step, each holding its own
                            W block and HALF of the X tile (the pair's tensor cores read both
                            halves), so every SM receives A + B/2 bytes per k-block instead of
                            A + B; x_multicast must be 0, 1 or 2 (the pair is the cluster).
                            0 = one CTA per 128-row block (default).  Same per-column products
                            (within tolerance; exact on integer data). */
} sparse_plan_opts;

/* Fill *opts with defaults (kind SPMM, device -1, everything else 0). */
void sparse_plan_opts_init(sparse_plan_opts* opts);

/* Inspector (offline).  W is M x K in CSR: row_ptr int32[M+1], col_idx int32[nnz],
 * values float32[nnz] — host arrays, borrowed for the duration of the call only.
 * On success *out owns the plan and its device memory on opts->device.
 * Errors: EINVAL (null out / arrays, M or K < 1, nnz < 0, bad dtype/kind),
 * EMATRIX (invalid CSR, see above), EUNSUPPORTED, ENOMEM, ECUDA.
 * Side effect: the device's default stream-ordered memory pool is set to keep its memory
 * (cudaMemPoolAttrReleaseThreshold = max): the executors take per-call scratch from it
 * (unaligned-X repack, conv input copies, tensor-core workspace) with cudaMallocAsync. */
int sparse_plan_create(sparse_plan_t* out, int32_t M, int32_t K, int64_t nnz,
                       const int32_t* row_ptr, const int32_t* col_idx,
                       const float* values, int32_t dtype,
                       const sparse_plan_opts* opts);

/* Executor, Y[M x N] = W[M x K] * X[K x N] (overwrite, beta = 0).
 * X, Y: DEVICE pointers on the plan's device, dtype of the plan, row-major with
 * N contiguous; ldx, ldy in elements (>= N).  Caller-owned; must not alias.
 * Every element of Y[:, :N] is written exactly once (rows without nonzeros get +0).
 * Asynchronous on `stream`.  N == 0 is a no-op.  16-byte aligned X/Y and ldx*s,
 * ldy*s take the vectorised path; anything else takes the element-wise GPU path.
 * Errors: EINVAL (null plan/pointers with N > 0, ld < N, conv plan, host-only
 * plan), ECUDA (launch failure). */
int sparse_spmm(sparse_plan_t plan, int64_t N, const void* X, int64_t ldx, void* Y,
                int64_t ldy, sparse_stream_t stream);

/* Executor for a SPARSE_CONV3X3 plan (Sec. 3.6):
 *   y[co][b][oy][ox] = sum_{ci,dy,dx} W[co][(ci*3+dy)*3+dx] * x[ci][b][oy+dy-1][ox+dx-1]
 * stride 1, zero padding 1, cross-correlation (== PyTorch conv2d with OIHW weight
 * W.reshape(C_out, C_in, 3, 3)).  x: DEVICE [C_in][batch][H][W], y: DEVICE
 * [C_out][batch][H][W], contiguous ("CNHW", so N = batch*H*W).  batch == 0 is a
 * no-op.  Errors: EINVAL (SpMM plan, null pointers, host-only plan), ECUDA. */
int sparse_conv3x3(sparse_plan_t plan, int64_t batch, const void* x, void* y,
                   sparse_stream_t stream);

/* Fused epilogue (NEXT #4; the paper leaves inter-op fusion to future work):
 *   Y = act(W*X + bias + beta*Y)
 * evaluated in fp32 on the plan-fixed accumulator (bias added after the last nonzero, then
 * beta*Y_old, then the activation), rounded once to the output dtype.  beta == 0 never reads
 * Y (NaN in Y is ignored); relu keeps NaN (x < 0 ? 0 : x). */
typedef struct {
  float beta;          /* 0 = overwrite */
  const void* bias;    /* DEVICE, M values (SpMM) or C_out values (conv), plan dtype; NULL = none */
  int32_t relu;        /* 0 = identity, 1 = ReLU */
} sparse_epilogue;

/* sparse_spmm / sparse_conv3x3 with an epilogue (ep == NULL: plain overwrite).  A JIT plan
 * (executor 1) runs its plan-driven kernel when ep is non-trivial. */
int sparse_spmm_ex(sparse_plan_t plan, int64_t N, const void* X, int64_t ldx, void* Y,
                   int64_t ldy, const sparse_epilogue* ep, sparse_stream_t stream);
int sparse_conv3x3_ex(sparse_plan_t plan, int64_t batch, const void* x, void* y,
                      const sparse_epilogue* ep, sparse_stream_t stream);

/* Token-major layout (NEXT #4; the PyTorch nn.Linear convention, e.g. BERT activations):
 *   Y[N x M] = X[N x K] * W^T        X, Y row-major (features contiguous), ldx >= K, ldy >= M
 * i.e. the same product as sparse_spmm on the transposed operands.  Implemented as a tiled
 * device transpose of X into a stream-ordered scratch (K x N), sparse_spmm, and a tiled
 * transpose of the result into Y - two extra passes over X and Y in HBM, never a host copy.
 * Results are bitwise those of sparse_spmm on X^T.  N == 0 is a no-op.  Errors as sparse_spmm
 * (+ ENOMEM when the scratch cannot be allocated). */
int sparse_linear(sparse_plan_t plan, int64_t N, const void* X, int64_t ldx, void* Y, int64_t ldy,
                  sparse_stream_t stream);

/* Strided 1x1 convolution (NEXT #4: the stride-2 projection shortcuts of ResNet-50, SURVEY
 * Appendix D) on a SPARSE_SPMM plan of W [C_out x C_in]:
 *   y[co][b][oy][ox] = sum_ci W[co][ci] * x[ci][b][oy*stride][ox*stride]
 * x: DEVICE [C_in][batch][h][w] (CNHW), y: DEVICE [C_out][batch][ho][wo], ho = ceil(h/stride),
 * wo = ceil(w/stride), contiguous.  stride 1 is sparse_spmm on x viewed as C_in x (batch h w).
 * stride > 1: a device gather of the sampled pixels into a stream-ordered scratch
 * [C_in][batch ho wo], then sparse_spmm (bitwise that product).  Errors as sparse_spmm
 * (+ EINVAL for stride < 1 or h, w < 1; ENOMEM for the scratch). */
int sparse_conv1x1(sparse_plan_t plan, int64_t batch, int32_t h, int32_t w, int32_t stride,
                   const void* x, void* y, sparse_stream_t stream);

/* NHWC (channels-last) 3x3 convolution on a SPARSE_CONV3X3 plan: x DEVICE [batch][H][W][C_in],
 * y DEVICE [batch][H][W][C_out], contiguous; the same sum as sparse_conv3x3.  Implemented as a
 * tiled device transpose of x into a CNHW scratch, sparse_conv3x3, and a transpose of the result
 * (results bitwise those of sparse_conv3x3 on the CNHW tensors).  Errors as sparse_conv3x3
 * (+ ENOMEM for the scratch). */
int sparse_conv3x3_nhwc(sparse_plan_t plan, int64_t batch, const void* x, void* y,
                        sparse_stream_t stream);

/* Free the plan and its device memory (north-star name).  Must not race with
 * work still enqueued that uses the plan.  NULL is a no-op. */
int plan_destroy(sparse_plan_t plan);
int sparse_plan_destroy(sparse_plan_t plan); /* alias */

typedef struct {
  int64_t nnz;          /* nonzeros carried by the plan (after drop_zeros) */
  int64_t plan_bytes;   /* device bytes of the packed plan (read by every call) */
  int32_t M, K, dtype, kind;
  int32_t panels;       /* row panels (thread-block rows, Fig. 2b) */
  int32_t warps;        /* warps per CTA */
  int32_t rows_per_warp;
  int32_t cols_per_lane;
  int32_t n_tile;       /* columns per CTA */
  int32_t k_chunk;      /* K rows per stage (conv: input channels per stage) */
  int32_t chunks;
  int32_t split_k;
  int32_t k_split;      /* CTAs per cluster splitting K */
  int32_t stages;
  int32_t smem_bytes;   /* dynamic shared memory per CTA */
  int32_t device;
  int32_t conv_rows_per_tile, conv_images_per_tile; /* conv tiling */
  int64_t max_panel_nnz, min_panel_nnz;            /* load-balance metrics */
  double build_ms;      /* host inspector wall time */
  int32_t executor;     /* 0 plan-driven, 1 JIT, 3 tensor-core condensed panels */
  int32_t jit_modules;  /* JIT: compiled modules (launches per call) */
  int32_t jit_rows, jit_warps;
  int64_t jit_cubin_bytes;
  double jit_compile_ms;
  double tuned_us;      /* tune = 1: measured time of the chosen configuration (us) */
  uint64_t digest;      /* FNV-1a of the packed plan: equal digests <=> identical replicas */
  int32_t x_multicast;  /* CTAs per cluster sharing X tiles (TMA multicast) */
  int32_t x_source;     /* 0 shared memory, 1 tensor memory */
  int32_t conv_kernel;  /* conv: 1 position-strided, 2 TMA-fed vectorised, 3 register-staged vectorised,
                           4 image-interleaved, 5 tcgen05 blocks */
  int32_t row_order;    /* 0 LPT panels, 1 natural order */
  int32_t tc_min_density; /* effective threshold (%), 0 = no tensor-core sub-blocks */
  int32_t tc_row_blocks;  /* 16-row blocks with >= 1 dense tile */
  int64_t tc_tiles;       /* dense 16 x 16 tiles on the tensor cores */
  int64_t tc_nnz;         /* nonzeros inside them (counted in nnz) */
  int64_t tc_panel_steps; /* executor 3: k16 steps over all (panel, chunk) pairs; the tensor cores
                             execute 2 * 16 * 16 * N flops per step (useful: 2 * nnz * N) */
  int32_t plan_source;  /* 0 staged with X, 1 kernel parameters */
  int32_t cta_pair;     /* executor 4: 1 = CTA pairs (cta_group::2, M = 256) */
} sparse_plan_info_t;

int sparse_plan_info(sparse_plan_t plan, sparse_plan_info_t* out);

/* Decode the packed plan back into one record per carried nonzero, in the
 * plan's storage order (test/inspection aid).  Arrays of length >= nnz (any may
 * be NULL): row and column of the nonzero, its stored value widened to fp32,
 * the panel, K-chunk and row slot (warp*R + r) it lives in, and the split-K
 * group that processes it.  Errors: EINVAL if cap < nnz. */
int sparse_plan_dump(sparse_plan_t plan, int64_t cap, int32_t* row, int32_t* col,
                     float* value, int32_t* panel, int32_t* chunk, int32_t* slot,
                     int32_t* group);

/* Thread-local detail of the last failing call on this thread ("" if none). */
const char* sparse_last_error(void);

/* Library version string, e.g. "sparsert-b200 0.1 sm_100a". */
const char* sparse_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPARSERT_H_ */
