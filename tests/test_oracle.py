"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself:
printed worked examples (tests/golden/, cited), closed forms, invariants, brute force on
tiny inputs and independent library routines (numpy / torch float64).  Each check is
chosen so that a plausible mistake in the oracle (dropped term, wrong sign or index,
transposed operand, wrong tap orientation, wrong padding) fails at least one of them.
"""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from synth import gen
from sparsert_testutil import golden

pytestmark = pytest.mark.filterwarnings("ignore")


def _csr_of_dense(d):
    d = np.asarray(d, dtype=np.float64)
    M, K = d.shape
    rp, ci, v = [0], [], []
    for m in range(M):
        for k in range(K):
            if d[m, k] != 0:
                ci.append(k)
                v.append(d[m, k])
        rp.append(len(ci))
    return (np.array(rp, np.int32), np.array(ci, np.int32), np.array(v, np.float64))


# ----------------------------------------------------------------------------------------
# Printed worked examples, stored under tests/golden/ with citations
# ----------------------------------------------------------------------------------------

def test_spec_csr4x4_to_dense_identity_ones():
    g = golden("spec_csr4x4.json")
    M, K = g["M"], g["K"]
    d = oracle.to_dense(M, K, g["row_ptr"], g["col_idx"], g["values"])
    assert np.array_equal(d, np.array(g["dense"], np.float64))
    y = oracle.spmm(M, K, g["row_ptr"], g["col_idx"], g["values"], np.eye(4))
    assert np.array_equal(y, np.array(g["times_identity"], np.float64))
    y = oracle.spmm(M, K, g["row_ptr"], g["col_idx"], g["values"], np.ones((4, 4)))
    assert np.array_equal(y, np.array(g["times_ones"], np.float64))


def test_spec_gemm2x2():
    g = golden("spec_gemm2x2.json")
    A = np.array(g["A"], np.float64)
    assert np.array_equal(oracle.gemm(A, np.eye(2)), A)
    assert np.array_equal(oracle.gemm(A, np.array(g["B"], np.float64)),
                          np.array(g["A_times_B"], np.float64))
    assert np.array_equal(oracle.gemm(A, np.zeros((2, 2))), np.zeros((2, 2)))


def test_spec_conv_examples():
    g = golden("spec_conv.json")
    x = np.array(g["center_tap_input"], np.float64).reshape(1, 1, 3, 3)
    # single center-tap filter: k = (0*3+1)*3+1 = 4
    y = oracle.conv3x3(1, [0, 1], [4], [1.0], x)
    assert np.array_equal(y, x)
    ones = np.ones((1, 1, 3, 3))
    y = oracle.conv3x3(1, [0, 9], list(range(9)), [1.0] * 9, ones)
    assert np.array_equal(y.reshape(3, 3), np.array(g["ones_output"], np.float64))
    y = oracle.conv3x3(1, [0, 0], [], [], x)
    assert np.array_equal(y, np.zeros_like(x))


def test_spec_im2col_examples():
    g = golden("spec_im2col.json")
    v = g["single_pixel_value"]
    cols = oracle.im2col(np.full((1, 1, 1, 1), v))
    assert cols.shape == (9, 1)
    for k in range(9):
        assert cols[k, 0] == (v if k == g["single_pixel_center_k"] else 0.0)
    x = np.array(g["x_1x2x2"], np.float64).reshape(1, 1, 2, 2)
    cols = oracle.im2col(x)
    assert cols[g["k_dy1_dx2"], 0] == g["expected_n0"]


def test_nnz_rounding_rule():
    g = golden("nnz_rounding.json")
    for M, K, p, nnz in g["cases"]:
        assert gen.nnz_for(M, K, p) == nnz
        if M * K <= 4096 * 4:
            assert gen.pruned_weights(M, K, p, 1).nnz == nnz


# ----------------------------------------------------------------------------------------
# Brute force on tiny inputs: every sparsity pattern of a 3x3 W, integer values -> exact
# ----------------------------------------------------------------------------------------

def test_brute_force_all_patterns_3x3():
    rng = np.random.default_rng(0)
    M = K = 3
    N = 4
    X = rng.integers(-5, 6, size=(K, N)).astype(np.int64)
    for bits in range(1 << (M * K)):
        mask = np.array([(bits >> i) & 1 for i in range(M * K)], bool).reshape(M, K)
        vals = rng.integers(1, 8, size=(M, K)) * rng.choice([-1, 1], size=(M, K))
        d = np.where(mask, vals, 0).astype(np.int64)
        rp, ci, v = _csr_of_dense(d)
        y = oracle.spmm(M, K, rp, ci, v, X.astype(np.float64))
        assert np.array_equal(y, (d @ X).astype(np.float64)), bits


def test_brute_force_rectangular_patterns():
    # M=2, K=3 and M=3, K=2: all 64 patterns each, catches transposed operands
    rng = np.random.default_rng(1)
    for M, K in [(2, 3), (3, 2), (1, 4), (4, 1)]:
        N = 5
        X = rng.integers(-4, 5, size=(K, N)).astype(np.int64)
        for bits in range(1 << (M * K)):
            mask = np.array([(bits >> i) & 1 for i in range(M * K)], bool).reshape(M, K)
            d = np.where(mask, rng.integers(1, 5, size=(M, K)), 0).astype(np.int64)
            rp, ci, v = _csr_of_dense(d)
            y = oracle.spmm(M, K, rp, ci, v, X.astype(np.float64))
            assert np.array_equal(y, (d @ X).astype(np.float64))


# ----------------------------------------------------------------------------------------
# Library routines (independent float64 implementations)
# ----------------------------------------------------------------------------------------

@pytest.mark.parametrize("M,K,N,p", [(64, 64, 128, 90), (37, 53, 71, 80), (128, 300, 33, 95),
                                     (5, 700, 9, 98), (200, 17, 300, 50)])
def test_spmm_vs_torch_float64(M, K, N, p):
    w = gen.pruned_weights(M, K, p, seed=M * 1000 + K)
    X = gen.uniform_x(K, N, seed=N).astype(np.float64)
    y = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values, X)
    d = torch.zeros(M, K, dtype=torch.float64)
    rows = np.repeat(np.arange(M), np.diff(w.row_ptr))
    d[torch.from_numpy(rows), torch.from_numpy(w.col_idx.astype(np.int64))] = \
        torch.from_numpy(w.values.astype(np.float64))
    ref = (d @ torch.from_numpy(X)).numpy()
    assert np.max(np.abs(y - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_to_dense_vs_torch_sparse():
    w = gen.pruned_weights(50, 70, 90, seed=3)
    d = oracle.to_dense(50, 70, w.row_ptr, w.col_idx, w.values)
    t = torch.sparse_csr_tensor(torch.from_numpy(w.row_ptr.astype(np.int64)),
                                torch.from_numpy(w.col_idx.astype(np.int64)),
                                torch.from_numpy(w.values.astype(np.float64)), size=(50, 70))
    assert np.array_equal(d, t.to_dense().numpy())


def test_gemm_vs_numpy():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((31, 47))
    B = rng.standard_normal((47, 19))
    assert np.allclose(oracle.gemm(A, B), A @ B, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("Cin,Cout,B,H,W", [(3, 4, 2, 5, 7), (8, 5, 1, 14, 14), (2, 3, 3, 1, 1),
                                            (1, 2, 1, 2, 9), (4, 4, 2, 7, 7)])
def test_conv_vs_torch_conv2d_float64(Cin, Cout, B, H, W):
    w = gen.pruned_weights(Cout, 9 * Cin, 70, seed=Cin * 31 + Cout)
    x = gen.relu_normal_x((Cin, B, H, W), seed=H * W).astype(np.float64)
    y = oracle.conv3x3(Cout, w.row_ptr, w.col_idx, w.values, x)
    wd = torch.zeros(Cout, 9 * Cin, dtype=torch.float64)
    rows = np.repeat(np.arange(Cout), np.diff(w.row_ptr))
    wd[torch.from_numpy(rows), torch.from_numpy(w.col_idx.astype(np.int64))] = \
        torch.from_numpy(w.values.astype(np.float64))
    # OIHW weight = W.reshape(C_out, C_in, 3, 3)  (k = (ci*3+dy)*3+dx); NCHW input
    xt = torch.from_numpy(x).permute(1, 0, 2, 3)
    ref = F.conv2d(xt, wd.reshape(Cout, Cin, 3, 3), padding=1).permute(1, 0, 2, 3).numpy()
    assert np.max(np.abs(y - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_im2col_vs_torch_unfold():
    x = gen.relu_normal_x((3, 2, 5, 6), seed=9).astype(np.float64)
    cols = oracle.im2col(x)
    xt = torch.from_numpy(x).permute(1, 0, 2, 3)  # B C H W
    u = F.unfold(xt, kernel_size=3, padding=1)  # B, C*9, H*W
    ref = u.permute(1, 0, 2).reshape(27, -1).numpy()
    assert np.array_equal(cols, ref)


def test_conv_equals_gemm_of_im2col():
    # SPEC S:360 coherence: gemm(filter_dense, im2col(x)) == conv_direct(x, filter)
    # integer data -> exact under any summation order
    Cin, Cout, B, H, W = 4, 6, 2, 6, 5
    w = gen.int_weights(Cout, 9 * Cin, 60, seed=2)
    x = gen.int_x(Cin, B * H * W, seed=3).reshape(Cin, B, H, W).astype(np.float64)
    y = oracle.conv3x3(Cout, w.row_ptr, w.col_idx, w.values, x)
    wd = oracle.to_dense(Cout, 9 * Cin, w.row_ptr, w.col_idx, w.values)
    y2 = oracle.gemm(wd, oracle.im2col(x)).reshape(Cout, B, H, W)
    assert np.array_equal(y, y2)


# ----------------------------------------------------------------------------------------
# Closed forms and invariants
# ----------------------------------------------------------------------------------------

def test_closed_forms():
    rng = np.random.default_rng(11)
    K, N = 40, 23
    X = rng.standard_normal((K, N))
    # W = 0
    y = oracle.spmm(7, K, np.zeros(8, np.int32), [], [], X)
    assert np.array_equal(y, np.zeros((7, N)))
    # W = I
    I = gen.identity_csr(K)
    assert np.array_equal(oracle.spmm(K, K, I.row_ptr, I.col_idx, I.values, X), X)
    # row selection W[m, sigma(m)] = 1  -> Y[m] = X[sigma(m)]
    S = gen.row_selection_csr(55, K, seed=4)
    y = oracle.spmm(55, K, S.row_ptr, S.col_idx, S.values, X)
    assert np.array_equal(y, X[S.col_idx])
    # W = diag(2^e) -> exact scaling
    e = rng.integers(-5, 6, size=K)
    y = oracle.spmm(K, K, np.arange(K + 1), np.arange(K), 2.0 ** e, X)
    assert np.array_equal(y, X * (2.0 ** e)[:, None])
    # X = one-hot columns e_j -> Y[:, j] = W[:, j]
    w = gen.pruned_weights(30, K, 80, seed=6)
    y = oracle.spmm(30, K, w.row_ptr, w.col_idx, w.values, np.eye(K))
    assert np.array_equal(y, oracle.to_dense(30, K, w.row_ptr, w.col_idx, w.values))
    assert np.array_equal(y, gen.to_dense(w))
    # X = ones with integer W -> row sums
    wi = gen.int_weights(30, K, 80, seed=6)
    y = oracle.spmm(30, K, wi.row_ptr, wi.col_idx, wi.values, np.ones((K, 3)))
    sums = np.add.reduceat(np.r_[wi.values, 0], wi.row_ptr[:-1])
    sums[np.diff(wi.row_ptr) == 0] = 0
    assert np.array_equal(y[:, 0], sums.astype(np.float64))


def test_permutation_invariances():
    rng = np.random.default_rng(12)
    M, K, N = 33, 45, 29
    w = gen.pruned_weights(M, K, 85, seed=7)
    X = rng.standard_normal((K, N))
    y = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values, X)
    # column permutation of X -> column permutation of Y (bitwise)
    pc = rng.permutation(N)
    assert np.array_equal(oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values, X[:, pc]), y[:, pc])
    # row permutation of W -> row permutation of Y (bitwise)
    pr = rng.permutation(M)
    d = gen.to_dense(w)[pr]
    rp, ci, v = _csr_of_dense(d)
    assert np.array_equal(oracle.spmm(M, K, rp, ci, v, X), y[pr])
    # N split into slabs -> concatenation equal (columns independent)
    parts = [oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values, X[:, a:b])
             for a, b in [(0, 10), (10, 11), (11, N)]]
    assert np.array_equal(np.concatenate(parts, axis=1), y)


def test_linearity():
    rng = np.random.default_rng(13)
    w = gen.pruned_weights(20, 30, 90, seed=8)
    X1, X2 = rng.standard_normal((30, 7)), rng.standard_normal((30, 7))
    f = lambda X: oracle.spmm(20, 30, w.row_ptr, w.col_idx, w.values, X)
    assert np.allclose(f(2.0 * X1 - 3.0 * X2), 2.0 * f(X1) - 3.0 * f(X2), rtol=1e-12, atol=1e-12)


def test_conv_delta_inputs():
    # x = 1 at (ci, b, y0, x0): y[co][b][y0-dy+1][x0-dx+1] = W[co][(ci*3+dy)*3+dx] inside
    Cin, Cout, B, H, W = 2, 3, 2, 5, 6
    w = gen.random_pattern(Cout, 9 * Cin, 30, seed=9)
    wd = gen.to_dense(w)
    for (ci, b, y0, x0) in [(0, 0, 0, 0), (1, 1, H - 1, W - 1), (0, 1, 0, 3), (1, 0, 2, 0), (1, 1, 2, 3)]:
        x = np.zeros((Cin, B, H, W))
        x[ci, b, y0, x0] = 1.0
        y = oracle.conv3x3(Cout, w.row_ptr, w.col_idx, w.values, x)
        exp = np.zeros((Cout, B, H, W))
        taps = 0
        for dy, dx in itertools.product(range(3), range(3)):
            oy, ox = y0 - dy + 1, x0 - dx + 1
            if 0 <= oy < H and 0 <= ox < W:
                exp[:, b, oy, ox] = wd[:, (ci * 3 + dy) * 3 + dx]
                taps += 1
        assert np.array_equal(y, exp)
        if (y0, x0) in [(0, 0), (H - 1, W - 1)]:
            assert taps == 4  # corner: exactly the 4 in-bounds taps


def test_thread_count_invariance():
    w = gen.pruned_weights(64, 96, 90, seed=10)
    X = gen.uniform_x(96, 50, seed=11).astype(np.float64)
    y1 = oracle.spmm(64, 96, w.row_ptr, w.col_idx, w.values, X, threads=1)
    y8 = oracle.spmm(64, 96, w.row_ptr, w.col_idx, w.values, X, threads=8)
    assert np.array_equal(y1, y8)


def test_rel_l2():
    ref = np.array([3.0, 4.0])
    assert oracle.rel_l2(ref, ref) == 0.0
    assert abs(oracle.rel_l2(ref * (1 + 1e-3), ref) - 1e-3) < 1e-15
    assert abs(oracle.rel_l2(np.array([3.0, 4.0 + 5.0]), ref) - 1.0) < 1e-15
    assert oracle.rel_l2(np.zeros(3), np.zeros(3)) == 0.0
    assert oracle.rel_l2(np.array([0.0, 1.0, 0.0]), np.zeros(3)) == float("inf")


def test_generator_determinism_and_structure():
    a = gen.pruned_weights(128, 64, 90, seed=5)
    b = gen.pruned_weights(128, 64, 90, seed=5)
    assert np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.values, b.values)
    assert a.nnz == gen.nnz_for(128, 64, 90)
    for m in range(a.M):
        c = a.col_idx[a.row_ptr[m]:a.row_ptr[m + 1]]
        assert np.all(np.diff(c) > 0)
    assert np.all(a.values != 0) and np.all(np.isfinite(a.values))
