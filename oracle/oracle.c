/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the SparseRT hot path
 * (arXiv 2008.11849).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no
 * source, header, table or helper with the CUDA path (paper_2008_11849_b200/),
 * and the CUDA path never loads it.
 *
 * What the method computes:  SparseRT "start[s] from a dense
 * matrix multiplication and simply remove[s] unnecessary computations"
 * (PAPER.md P:50); "The sparse matrix is first treated as a dense matrix,
 * casting the problem to a GeMM"; the compact transform keeps "only the
 * computations that correspond to nonzero matrix elements in A" (P:183,
 * Alg. 3).  The result is therefore exactly the plain dense product
 * A x B = C, A = M x K, B = K x N, C = M x N, C-style row-major — and
 * this oracle is that definition written out: densify A, then the m-k-n
 * triple loop in double precision, skipping nothing.
 *
 * Convolution: 3x3 filters, zero padding 1, stride 1 (output keeps
 * H x W, Table 3), filter k = (ci*3+dy)*3+dx is a row of A
 * ("each filter is materialized as a row of the A matrix"), i.e.
 * cross-correlation.  The oracle is the direct 7-loop convolution (the
 * "classic 7-loop convolution algorithm"), NOT im2col, so that
 * ref_im2col_f64 + ref_gemm_f64 gives an independent cross-check.
 * Activation layout CNHW [C][B][H][W] (reading R12).
 *
 * Parity status: every function here is pinned by tests/test_oracle.py
 * (printed worked examples, closed forms, brute force, library routines).
 *
 * Accumulation is in double; each output's summation order is fixed
 * (k ascending / ci,dy,dx ascending), so OpenMP thread count never changes
 * results.  Build: gcc -O2 -fopenmp -ffp-contract=off (no fast-math).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* to_dense(A): "cuBLAS performs the sparse matrix multiplication as a dense
 * matrix multiplication" (Fig. 4 caption).  Wd is M*K,
 * row-major, zero-initialised here. */
void ref_to_dense_f64(int32_t M, int32_t K, const int32_t* row_ptr,
                      const int32_t* col_idx, const double* val, double* Wd) {
    memset(Wd, 0, sizeof(double) * (size_t)M * (size_t)K);
    for (int32_t m = 0; m < M; ++m)
        for (int32_t e = row_ptr[m]; e < row_ptr[m + 1]; ++e)
            Wd[(size_t)m * K + col_idx[e]] = val[e];
}

/* Dense GEMM C = A x B: A M x K (lda), B K x N (ldb), C M x N (ldc).
 * Loop order m, k, n; C overwritten. */
void ref_gemm_f64(int32_t M, int32_t K, int64_t N, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double* C, int64_t ldc,
                  int32_t threads) {
    (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int32_t m = 0; m < M; ++m) {
        double* c = C + (size_t)m * ldc;
        for (int64_t n = 0; n < N; ++n) c[n] = 0.0;
        for (int32_t k = 0; k < K; ++k) {
            const double a = A[(size_t)m * lda + k];
            const double* b = B + (size_t)k * ldb;
            for (int64_t n = 0; n < N; ++n) c[n] += a * b[n];
        }
    }
}

/* Y = W x X with W given in CSR (M x K), X K x N (ldx), Y M x N (ldy).
 * Expands W to dense, then the plain m-k-n triple loop over ALL k (zeros
 * included; nothing skipped).  Returns 0, or -1 if the dense buffer cannot be
 * allocated. */
int ref_spmm_f64(int32_t M, int32_t K, int64_t N, const int32_t* row_ptr,
                 const int32_t* col_idx, const double* val, const double* X,
                 int64_t ldx, double* Y, int64_t ldy, int32_t threads) {
    double* Wd = (double*)malloc(sizeof(double) * (size_t)M * (size_t)K + 8);
    if (!Wd) return -1;
    ref_to_dense_f64(M, K, row_ptr, col_idx, val, Wd);
    ref_gemm_f64(M, K, N, Wd, K, X, ldx, Y, ldy, threads);
    free(Wd);
    return 0;
}

/* im2col: cols is (9*C_in) x (B*H*W), row k =
 * (ci*3+dy)*3+dx, column n = (b*H + y)*W + x, entry = x[ci][b][y+dy-1][x+dx-1]
 * or 0 outside the image (zero padding 1). */
void ref_im2col_f64(int32_t C_in, int32_t B, int32_t H, int32_t W,
                    const double* x, double* cols) {
    const int64_t N = (int64_t)B * H * W;
    for (int32_t ci = 0; ci < C_in; ++ci)
        for (int32_t dy = 0; dy < 3; ++dy)
            for (int32_t dx = 0; dx < 3; ++dx) {
                const int64_t k = ((int64_t)ci * 3 + dy) * 3 + dx;
                for (int32_t b = 0; b < B; ++b)
                    for (int32_t y = 0; y < H; ++y)
                        for (int32_t xx = 0; xx < W; ++xx) {
                            const int32_t sy = y + dy - 1, sx = xx + dx - 1;
                            const int64_t n = ((int64_t)b * H + y) * W + xx;
                            double v = 0.0;
                            if (sy >= 0 && sy < H && sx >= 0 && sx < W)
                                v = x[(((int64_t)ci * B + b) * H + sy) * W + sx];
                            cols[k * N + n] = v;
                        }
            }
}

/* Direct 3x3 convolution, stride 1, zero pad 1, cross-correlation:
 *   y[co][b][y][x] = sum_{ci,dy,dx} Wd[co][(ci*3+dy)*3+dx] * x~[ci][b][y+dy-1][x+dx-1]
 * with W in CSR (C_out x 9*C_in), x [C_in][B][H][W], y [C_out][B][H][W].
 * Expands W to dense and loops over every tap (nothing skipped). */
int ref_conv3x3_f64(int32_t C_out, int32_t C_in, int32_t B, int32_t H, int32_t W,
                    const int32_t* row_ptr, const int32_t* col_idx,
                    const double* val, const double* x, double* y,
                    int32_t threads) {
    const int32_t K = 9 * C_in;
    double* Wd = (double*)malloc(sizeof(double) * (size_t)C_out * (size_t)K + 8);
    if (!Wd) return -1;
    ref_to_dense_f64(C_out, K, row_ptr, col_idx, val, Wd);
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int32_t co = 0; co < C_out; ++co)
        for (int32_t b = 0; b < B; ++b)
            for (int32_t oy = 0; oy < H; ++oy)
                for (int32_t ox = 0; ox < W; ++ox) {
                    double acc = 0.0;
                    for (int32_t ci = 0; ci < C_in; ++ci)
                        for (int32_t dy = 0; dy < 3; ++dy)
                            for (int32_t dx = 0; dx < 3; ++dx) {
                                const int32_t sy = oy + dy - 1, sx = ox + dx - 1;
                                if (sy < 0 || sy >= H || sx < 0 || sx >= W) continue;
                                acc += Wd[(size_t)co * K + (ci * 3 + dy) * 3 + dx] *
                                       x[(((int64_t)ci * B + b) * H + sy) * W + sx];
                            }
                    y[(((int64_t)co * B + b) * H + oy) * W + ox] = acc;
                }
    free(Wd);
    return 0;
}

/* rel_l2 = ||a - ref||_2 / ||ref||_2 (north star parity metric).  If ||ref||
 * is 0, returns 0 when a is identically 0, else +inf. */
double ref_rel_l2(const double* a, const double* ref, int64_t n) {
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = a[i] - ref[i];
        num += d * d;
        den += ref[i] * ref[i];
    }
    if (den == 0.0) return num == 0.0 ? 0.0 : INFINITY;
    return sqrt(num) / sqrt(den);
}
