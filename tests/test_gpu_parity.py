"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Bars (north star): rel-L2 <= 1e-5 for fp32 and <= 1e-2 for fp16 on
generated inputs at 80/90/95/98% sparsity; BITWISE equality on integer-valued inputs
(every fp32 partial sum exact) at the full BASELINE sizes; bitwise closed forms and
invariances (W = 0, W = I, row selection, X = I_K, permutations, N-sharding).
"""
import numpy as np
import pytest
import torch

import oracle
from synth import gen
from sparsert_testutil import as_f16_f64

import paper_2008_11849_b200 as srt

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5
F16_TOL = 1e-2


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _tdt(f16):
    return torch.float16 if f16 else torch.float32


def _w64(w, f16):
    return as_f16_f64(w.values) if f16 else w.values.astype(np.float64)


def _x64(x, f16):
    return as_f16_f64(x) if f16 else x.astype(np.float64)


def _run_spmm(w, X_np, f16, N=None, ld=None, ldy=None, **opts):
    dev = _dev()
    K, Ncols = X_np.shape
    N = Ncols if N is None else N
    plan = srt.Plan.from_csr(w, dtype=_tdt(f16), n_hint=opts.pop("n_hint", N), **opts)
    X = torch.from_numpy(X_np).to(dev).to(_tdt(f16))
    if ld is not None and ld != Ncols:
        buf = torch.zeros((K, ld), dtype=_tdt(f16), device=dev)
        buf[:, :Ncols] = X
        X = buf[:, :N]
    else:
        X = X[:, :N]
    if ldy is not None:
        Ybuf = torch.full((w.M, ldy), float("nan"), dtype=_tdt(f16), device=dev)
        Y = Ybuf[:, :N]
    else:
        Y = torch.full((w.M, N), float("nan"), dtype=_tdt(f16), device=dev)
    plan.spmm(X, Y)
    torch.cuda.synchronize()
    return Y.float().cpu().numpy().astype(np.float64), plan


def _ref(w, X_np, f16, N=None):
    X = _x64(X_np, f16)
    if N is not None:
        X = X[:, :N]
    y = oracle.spmm(w.M, w.K, w.row_ptr, w.col_idx, _w64(w, f16), X)
    return y


def _f16_round(y):
    return y.astype(np.float16).astype(np.float64)


# --------------------------------------------------------------------------- tolerance

@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("p", [80, 90, 95, 98])
@pytest.mark.parametrize("M,K,N", [(64, 64, 128), (300, 200, 517), (1000, 64, 49), (77, 1111, 300)])
def test_spmm_rel_l2(M, K, N, p, f16):
    w = gen.pruned_weights(M, K, p, seed=gen.case_seed(f"{M}x{K}x{N}", p))
    X = gen.uniform_x(K, N, seed=N + p)
    y, _ = _run_spmm(w, X, f16)
    ref = _ref(w, X, f16)
    err = oracle.rel_l2(y, ref)
    assert err <= (F16_TOL if f16 else F32_TOL), err
    if not f16:
        assert err < 2e-6  # expected ~3e-7; catches gross order bugs


# --------------------------------------------------------------------------- exactness

def _exact_case(M, K, N, p, f16, seed, **kw):
    vmax_w, vmax_x = (2, 4) if f16 else (3, 3)
    w = gen.int_weights(M, K, p, seed=seed, vmax=vmax_w)
    X = gen.int_x(K, N, seed=seed + 1, vmax=vmax_x)
    y, plan = _run_spmm(w, X, f16, **kw)
    ref = _ref(w, X, f16)
    if f16:
        ref = _f16_round(ref)
    assert np.array_equal(y, ref), (np.argwhere(y != ref)[:5], plan.info)
    return plan


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("case", [
    (64, 256, 3136), (256, 64, 3136), (128, 512, 784), (512, 128, 784), (256, 1024, 196),
    (1024, 256, 196), (512, 2048, 49), (2048, 512, 49),          # RN50 Table 1, batch 1
    (2048, 512, 392), (512, 2048, 392),                           # RN50 p7/p8 batch 8
    (64, 32, 12544), (1024, 1024, 49), (512, 512, 196),           # MobileNetV1
    (3072, 768, 512), (768, 3072, 512),                           # BERT FC, 1x512
])
@pytest.mark.parametrize("p", [90, 95])
def test_spmm_integer_exact_table_shapes(case, p, f16):
    M, K, N = case
    _exact_case(M, K, N, p, f16, seed=gen.case_seed(str(case), p))


@pytest.mark.parametrize("f16", [False, True])
def test_spmm_integer_exact_bert_full(f16):
    # BERT FC at N = 32 x 512 = 16384 (BASELINE configs[3] maximum), both orientations
    for M, K in [(3072, 768), (768, 3072)]:
        _exact_case(M, K, 16384, 90, f16, seed=M)


# --------------------------------------------------------------------------- closed forms

@pytest.mark.parametrize("f16", [False, True])
def test_closed_forms(f16):
    dev = _dev()
    K, N = 300, 777
    X = gen.uniform_x(K, N, seed=3)
    # W = 0 (nnz = 0) -> Y identically +0
    z = gen.stress_pattern("empty", 50, K, seed=1)
    y, _ = _run_spmm(z, X, f16)
    assert np.array_equal(y, np.zeros_like(y)) and not np.signbit(y).any()
    # W = I -> Y = X exactly
    y, _ = _run_spmm(gen.identity_csr(K), X, f16)
    assert np.array_equal(y, _x64(X, f16))
    # row selection -> Y[m] = X[sigma(m)] exactly, with ragged N and ldx > N
    s = gen.row_selection_csr(1000, K, seed=5)
    y, _ = _run_spmm(s, X, f16, N=701, ld=777)
    assert np.array_equal(y, _x64(X, f16)[s.col_idx][:, :701])
    # X = I_K -> Y = dense(W) exactly: pins the position and value of every carried nonzero
    w = gen.pruned_weights(513, K, 90, seed=6)
    y, _ = _run_spmm(w, np.eye(K, dtype=np.float32), f16)
    wd = gen.to_dense(w.with_values(_w64(w, f16).astype(np.float32)))
    assert np.array_equal(y, wd)


@pytest.mark.parametrize("f16", [False, True])
def test_identity_full_size(f16):
    # X = I_K tiled along N at a BERT size: every nonzero of a 3072 x 768 plan checked
    w = gen.pruned_weights(3072, 768, 90, seed=7)
    X = np.tile(np.eye(768, dtype=np.float32), (1, 3))
    y, _ = _run_spmm(w, X, f16)
    wd = gen.to_dense(w.with_values(_w64(w, f16).astype(np.float32)))
    assert np.array_equal(y, np.tile(wd, (1, 3)))


# --------------------------------------------------------------------------- invariances

@pytest.mark.parametrize("f16", [False, True])
def test_permutation_and_sharding_invariance(f16):
    rng = np.random.default_rng(0)
    M, K, N = 700, 500, 1000
    w = gen.pruned_weights(M, K, 90, seed=11)
    X = gen.uniform_x(K, N, seed=12)
    y, plan = _run_spmm(w, X, f16)
    # column permutation of X -> column permutation of Y, bitwise
    pc = rng.permutation(N)
    y2, _ = _run_spmm(w, np.ascontiguousarray(X[:, pc]), f16, n_hint=N)
    assert np.array_equal(y2, y[:, pc])
    # row permutation of W -> row permutation of Y, bitwise
    pr = rng.permutation(M)
    d = gen.to_dense(w)[pr]
    wp = gen.csr_from_mask(M, K, np.flatnonzero(d), d.astype(np.float32))
    y3, _ = _run_spmm(wp, X, f16, n_hint=N)
    assert np.array_equal(y3, y[pr])
    # N-sharding: column slabs with the same plan -> concatenation bitwise equal
    dev = _dev()
    Xt = torch.from_numpy(X).to(dev).to(_tdt(f16))
    parts = []
    for a, b in [(0, 256), (256, 640), (640, 1000)]:
        parts.append(plan.spmm(Xt[:, a:b].contiguous()).float().cpu().numpy())
    assert np.array_equal(np.concatenate(parts, axis=1).astype(np.float64), y)
    # determinism: repeated call bitwise identical
    assert np.array_equal(plan.spmm(Xt).float().cpu().numpy().astype(np.float64), y)


# --------------------------------------------------------------------------- edge cases

@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("kind", ["zipf", "empty_rows", "dense_row", "block_dense", "one_column"])
def test_stress_patterns(kind, f16):
    M, K, N = 400, 600, 333
    w = gen.stress_pattern(kind, M, K, seed=21)
    X = gen.uniform_x(K, N, seed=22)
    y, _ = _run_spmm(w, X, f16)
    ref = _ref(w, X, f16)
    assert oracle.rel_l2(y, ref) <= (F16_TOL if f16 else F32_TOL)


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("N,ld,ldy", [(49, 49, 49), (49, 53, 51), (196, 196, 197), (1, 1, 1),
                                      (130, 131, 130), (7, 8, 9)])
def test_unaligned_and_tiny_n(N, ld, ldy, f16):
    w = gen.int_weights(300, 257, 85, seed=N)
    X = gen.int_x(257, ld, seed=N + 1, vmax=2)
    y, _ = _run_spmm(w, X, f16, N=N, ld=ld, ldy=ldy)
    ref = _ref(w, X, f16, N=N)
    if f16:
        ref = _f16_round(ref)
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("R,warps,kc,gk,ks,st", [(1, 1, 8, 1, 1, 1), (2, 8, 16, 2, 8, 2),
                                                 (8, 4, 256, 8, 1, 3), (4, 2, 40, 4, 2, 4),
                                                 (8, 3, 64, 1, 4, 2), (16, 8, 32, 1, 8, 3)])
def test_tile_overrides_exact(R, warps, kc, gk, ks, st, f16):
    if f16 and R == 16:
        pytest.skip("R=16 exceeds the fp16 accumulator budget")
    _exact_case(333, 700, 250, 90, f16, seed=R * 10 + gk, rows_per_warp=R, warps=warps,
                k_chunk=kc, split_k=gk, k_split=ks, stages=st)


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("warps,R,kc,st,cm", [(16, 4, 32, 8, 1), (16, 2, 128, 0, 2), (8, 4, 64, 3, 4),
                                              (16, 1, 32, 6, 8), (5, 2, 48, 2, 2), (16, 8, 64, 0, 1)])
def test_wide_ctas_deep_rings_and_multicast_exact(warps, R, kc, st, cm, f16):
    # 16-warp CTAs, rings up to 8 stages, X multicast clusters of 2-8 CTAs (one TMA box
    # feeds every CTA of the cluster): exact on integer data, incl. ragged M / N / K, and
    # x_multicast never changes a result (it only changes who loads X)
    if f16 and R * 8 > 64:
        pytest.skip("accumulator budget")
    for M, K, N in [(333, 700, 250), (2048, 512, 392), (64, 256, 3136)]:
        plan = _exact_case(M, K, N, 90, f16, seed=warps + R + cm, rows_per_warp=R, warps=warps,
                           k_chunk=kc, stages=st, x_multicast=cm)
        assert plan.info["x_multicast"] == cm and plan.info["warps"] == warps
        assert plan.info["panels"] % cm == 0


@pytest.mark.parametrize("f16", [False, True])
def test_row_order_natural_bitwise(f16):
    # load balancing only moves rows between CTAs: bitwise the same output
    w = gen.stress_pattern("zipf", 700, 300, seed=61)
    X = gen.uniform_x(300, 333, seed=62)
    y0, _ = _run_spmm(w, X, f16, warps=8, rows_per_warp=4)
    y1, p1 = _run_spmm(w, X, f16, warps=8, rows_per_warp=4, row_order=1)
    assert p1.info["row_order"] == 1 and np.array_equal(y0, y1)


@pytest.mark.parametrize("f16", [False, True])
def test_multicast_bitwise_equals_unicast(f16):
    w = gen.pruned_weights(1024, 768, 90, seed=41)
    X = gen.uniform_x(768, 1000, seed=42)
    y1, _ = _run_spmm(w, X, f16, warps=8, rows_per_warp=4, x_multicast=1)
    for cm in (2, 4, 8):
        y, _ = _run_spmm(w, X, f16, warps=8, rows_per_warp=4, x_multicast=cm)
        assert np.array_equal(y, y1)


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("warps,R,kc", [(16, 4, 56), (8, 8, 56), (8, 2, 32), (4, 1, 16), (12, 8, 48)])
def test_tmem_x_source_exact(warps, R, kc, f16):
    # X read from tensor memory (tcgen05.cp smem -> TMEM, tcgen05.ld): exact on integer data
    # for ragged shapes and the Table-1 / BERT shapes, including neutral padding entries
    # (zero row of each TMEM buffer) and K not a multiple of k_chunk
    if f16 and R * 8 > 64:
        pytest.skip("accumulator budget")
    for M, K, N in [(333, 700, 250), (2048, 512, 392), (64, 256, 3136), (3072, 768, 512)]:
        plan = _exact_case(M, K, N, 90, f16, seed=warps * R + kc, rows_per_warp=R, warps=warps,
                           k_chunk=kc, x_source=1)
        assert plan.info["x_source"] == 1


@pytest.mark.parametrize("f16", [False, True])
def test_tmem_bitwise_equals_smem(f16):
    # the X source never changes the arithmetic: same plan options, bitwise equal outputs
    w = gen.pruned_weights(1024, 768, 90, seed=51)
    X = gen.uniform_x(768, 1000, seed=52)
    kw = dict(warps=8, rows_per_warp=4, k_chunk=56)
    y0, _ = _run_spmm(w, X, f16, x_source=0, **kw)
    y1, p1 = _run_spmm(w, X, f16, x_source=1, **kw)
    assert p1.info["x_source"] == 1
    assert np.array_equal(y0, y1)
    assert oracle.rel_l2(y1, _ref(w, X, f16)) <= (F16_TOL if f16 else F32_TOL)


@pytest.mark.parametrize("f16", [False, True])
def test_k_split_changes_order_not_value(f16):
    # k_split fixes a different (still deterministic) summation order: equal within tolerance,
    # bitwise on integer data, and repeated calls are bitwise identical.
    w = gen.pruned_weights(256, 2048, 90, seed=31)
    X = gen.uniform_x(2048, 392, seed=32)
    ys = []
    for ks in (1, 2, 4, 8):
        y, plan = _run_spmm(w, X, f16, k_split=ks, rows_per_warp=4)
        assert plan.info["k_split"] == ks
        ys.append(y)
        assert oracle.rel_l2(y, _ref(w, X, f16)) <= (F16_TOL if f16 else F32_TOL)
    for ks in (1, 8):
        _exact_case(256, 2048, 392, 90, f16, seed=33, k_split=ks, rows_per_warp=4)


def test_api_errors_on_device():
    dev = _dev()
    w = gen.pruned_weights(64, 64, 90, seed=1)
    plan = srt.Plan.from_csr(w)
    with pytest.raises(ValueError):
        plan.conv3x3(torch.zeros(1, 1, 3, 3, device=dev))
    with pytest.raises(TypeError):
        plan.spmm(torch.zeros(64, 8, device=dev, dtype=torch.float16))
    # N = 0 is a no-op
    plan.spmm(torch.zeros(64, 0, device=dev))
    info = plan.info
    assert info["device"] == 0 and info["plan_bytes"] > 0


# --------------------------------------------------------------------------- conv

def _conv_run(w, cin, x_np, f16, **opts):
    dev = _dev()
    C, B, H, W = x_np.shape
    plan = srt.Plan.from_csr(w, dtype=_tdt(f16), kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W,
                             n_hint=opts.pop("n_hint", B), **opts)
    x = torch.from_numpy(x_np).to(dev).to(_tdt(f16)).contiguous()
    y = plan.conv3x3(x)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64), plan


def _conv_ref(w, x_np, f16):
    return oracle.conv3x3(w.M, w.row_ptr, w.col_idx, _w64(w, f16), _x64(x_np, f16))


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("cin,cout,B,H,W,p", [(64, 64, 2, 56, 56, 90), (128, 128, 2, 28, 28, 90),
                                              (256, 256, 3, 14, 14, 90), (512, 512, 2, 7, 7, 95),
                                              (3, 5, 3, 5, 9, 50), (16, 40, 1, 1, 1, 80),
                                              (8, 8, 5, 2, 3, 80)])
def test_conv_rel_l2(cin, cout, B, H, W, p, f16):
    w = gen.pruned_weights(cout, 9 * cin, p, seed=cin + H)
    x = gen.relu_normal_x((cin, B, H, W), seed=B * H)
    y, _ = _conv_run(w, cin, x, f16)
    err = oracle.rel_l2(y, _conv_ref(w, x, f16))
    assert err <= (F16_TOL if f16 else F32_TOL), err


@pytest.mark.parametrize("f16", [False, True])
def test_conv_integer_exact_and_delta(f16):
    cin, cout, B, H, W = 32, 48, 3, 14, 14
    w = gen.int_weights(cout, 9 * cin, 80, seed=3, vmax=2)
    x = gen.int_x(cin, B * H * W, seed=4, vmax=3).reshape(cin, B, H, W)
    y, _ = _conv_run(w, cin, x, f16)
    ref = _conv_ref(w, x, f16)
    if f16:
        ref = _f16_round(ref)
    assert np.array_equal(y, ref)
    # delta inputs at corners / edges / interior: exact taps (orientation + zero halo)
    wd = gen.to_dense(w)
    for (ci, b, y0, x0) in [(0, 0, 0, 0), (5, 2, H - 1, W - 1), (31, 1, 0, 7), (7, 0, 6, 0),
                            (9, 1, 7, 8)]:
        xd = np.zeros((cin, B, H, W), np.float32)
        xd[ci, b, y0, x0] = 1.0
        y, _ = _conv_run(w, cin, xd, f16)
        exp = np.zeros((cout, B, H, W))
        for dy in range(3):
            for dx in range(3):
                oy, ox = y0 - dy + 1, x0 - dx + 1
                if 0 <= oy < H and 0 <= ox < W:
                    exp[:, b, oy, ox] = wd[:, (ci * 3 + dy) * 3 + dx]
        assert np.array_equal(y, exp)


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("cin,cout,B,H,W,R,warps,cc", [
    (16, 24, 3, 14, 14, 2, 16, 5), (256, 64, 2, 14, 14, 8, 16, 16), (8, 40, 2, 7, 7, 4, 8, 3),
    (32, 16, 1, 56, 56, 2, 16, 8), (12, 20, 2, 28, 28, 8, 8, 4), (5, 9, 3, 5, 9, 1, 4, 2)])
def test_conv_vectorised_exact_and_bitwise(cin, cout, B, H, W, R, warps, cc, f16):
    # the vectorised conv kernels (three dx-shifted input copies, 128-bit position loads;
    # register-staged (0) and TMA-fed (2)): exact on integer data, bitwise equal to the
    # position-strided kernel (same k order)
    dev = _dev()
    vmax_w, vmax_x = (2, 4) if f16 else (3, 3)
    w = gen.int_weights(cout, 9 * cin, 90, seed=cin + H, vmax=vmax_w)
    x = gen.int_x(cin * B * H, W, seed=cout, vmax=vmax_x).reshape(cin, B, H, W)
    xt = torch.from_numpy(x).to(dev).to(_tdt(f16))
    ys = []
    for ck in (3, 1, 2):
        kw = dict(rows_per_warp=R, warps=warps, k_chunk=cc) if ck != 1 else {}
        plan = srt.Plan.from_csr(w, dtype=_tdt(f16), kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W,
                                 n_hint=B, conv_kernel=ck, **kw)
        assert plan.info["conv_kernel"] == ck
        y = plan.conv3x3(xt)
        torch.cuda.synchronize()
        ys.append(y.float().cpu().numpy().astype(np.float64))
    ref = oracle.conv3x3(cout, w.row_ptr, w.col_idx, _w64(w, f16), _x64(x, f16))
    if f16:
        ref = _f16_round(ref)
    assert np.array_equal(ys[0], ref)
    assert np.array_equal(ys[0], ys[1])
    assert np.array_equal(ys[2], ys[1])


@pytest.mark.parametrize("dt", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("cin,cout,B,H,W,R,warps,cc", [
    (16, 24, 3, 14, 14, 8, 16, 5), (256, 64, 2, 14, 14, 8, 16, 16), (256, 256, 5, 14, 14, 8, 16, 0),
    (32, 16, 1, 28, 28, 4, 16, 8), (12, 20, 2, 28, 28, 8, 8, 4), (5, 9, 3, 10, 6, 2, 16, 2),
    (8, 8, 5, 4, 4, 8, 16, 3), (64, 128, 4, 14, 14, 1, 16, 8), (40, 33, 7, 10, 6, 2, 8, 7),
    (512, 64, 3, 7, 8, 4, 16, 12), (16, 20, 9, 4, 4, 2, 4, 5), (24, 16, 3, 4, 8, 1, 4, 12)])
def test_conv_packed_exact_and_bitwise(cin, cout, B, H, W, R, warps, cc, dt):
    # the image-interleaved implicit-im2col kernel (conv_kernel 4: g images side by side per
    # row, no junk positions except the padding images of a batch not a multiple of g): exact on
    # integer data and bitwise equal to the register-staged vectorised kernel (same k order)
    dev = _dev()
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dt]
    vmax_w, vmax_x = (3, 3) if dt == "f32" else (2, 4)
    w = gen.int_weights(cout, 9 * cin, 90, seed=cin + H + W, vmax=vmax_w)
    x = gen.int_x(cin * B * H, W, seed=cout + B, vmax=vmax_x).reshape(cin, B, H, W)
    xt = torch.from_numpy(x).to(dev).to(tdt)
    kw = dict(rows_per_warp=R, warps=warps)
    if cc:
        kw["k_chunk"] = cc
    plan = srt.Plan.from_csr(w, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B,
                             conv_kernel=4, **kw)
    assert plan.info["conv_kernel"] == 4
    y = torch.full((cout, B, H, W), float("nan"), dtype=tdt, device=dev)
    plan.conv3x3(xt, y)
    torch.cuda.synchronize()
    got = y.double().cpu().numpy()
    ref = oracle.conv3x3(cout, w.row_ptr, w.col_idx, w.values.astype(np.float64), x.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(got, ref)
    if dt != "bf16":
        other = srt.Plan.from_csr(w, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B,
                                  conv_kernel=3)
        y3 = other.conv3x3(xt)
        torch.cuda.synchronize()
        assert np.array_equal(y3.double().cpu().numpy(), got)
    # the plan decodes back to W exactly (every nonzero once, at its (ci, dy, dx))
    d = plan.dump()
    dense = np.zeros((cout, 9 * cin))
    dense[d.row, d.col] = d.value
    assert np.array_equal(dense, gen.to_dense(w))


def test_conv_packed_real_valued_and_unsupported():
    dev = _dev()
    cin, cout, B, H, W = 128, 128, 6, 28, 28
    w = gen.pruned_weights(cout, 9 * cin, 95, seed=77)
    x = gen.relu_normal_x((cin, B, H, W), seed=78)
    for f16 in (False, True):
        y, plan = _conv_run(w, cin, x, f16, conv_kernel=4)
        assert plan.info["conv_kernel"] == 4
        err = oracle.rel_l2(y, _conv_ref(w, x, f16))
        assert err <= (F16_TOL if f16 else F32_TOL), err
    w7 = gen.pruned_weights(16, 9 * 8, 90, seed=79)
    with pytest.raises(srt.SparseRTError):  # 56-wide images: span beyond one TMA box
        srt.Plan.from_csr(w7, kind=srt.SPARSE_CONV3X3, c_in=8, h=56, w=56, n_hint=2, conv_kernel=4)


@pytest.mark.parametrize("f16", [False, True])
def test_conv_center_tap_equals_spmm(f16):
    # a W using only the center tap (dy = dx = 1) is a 1x1 conv: conv3x3 == spmm bitwise
    cin, cout, B, H, W = 64, 96, 4, 14, 14
    base = gen.pruned_weights(cout, cin, 80, seed=8)
    w = gen.Csr(cout, 9 * cin, base.row_ptr, (base.col_idx * 9 + 4).astype(np.int32), base.values)
    x = gen.relu_normal_x((cin, B, H, W), seed=9)
    y, _ = _conv_run(w, cin, x, f16)
    ys, _ = _run_spmm(base, x.reshape(cin, -1), f16)
    assert np.array_equal(y.reshape(cout, -1), ys)


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("ck", [2, 3, 4])
def test_conv_c5_full_batch_sampled(ck, f16):
    # BASELINE configs[4] at full size (256 ch, 14x14, batch 256, 90%), in the bench's launch
    # configuration; integer data, images {0, 101, 255} checked bitwise against the oracle,
    # and image-slab sharding (the N-sharded multi-GPU split) checked bitwise.
    cin = cout = 256
    B, H, W = 256, 14, 14
    w = gen.int_weights(cout, 9 * cin, 90, seed=5, vmax=2)
    x = gen.int_x(cin, B * H * W, seed=6, vmax=2).reshape(cin, B, H, W)
    y, plan = _conv_run(w, cin, x, f16, conv_kernel=ck)
    assert plan.info["conv_kernel"] == ck
    idx = [0, 101, 255]
    ref = _conv_ref(w, np.ascontiguousarray(x[:, idx]), f16)
    if f16:
        ref = _f16_round(ref)
    assert np.array_equal(y[:, idx], ref)
    dev = _dev()
    xt = torch.from_numpy(x).to(dev).to(_tdt(f16))
    half = plan.conv3x3(xt[:, 128:].contiguous()).float().cpu().numpy()
    assert np.array_equal(half.astype(np.float64), y[:, 128:])


# --------------------------------------------------------------------------- JIT executor

@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("case", [(64, 64, 128), (300, 200, 517), (2048, 512, 392), (512, 2048, 49),
                                  (256, 64, 25088), (1000, 333, 1001)])
def test_jit_integer_exact(case, f16):
    M, K, N = case
    plan = _exact_case(M, K, N, 90, f16, seed=M + K + N, executor=1)
    assert plan.info["executor"] == 1 and plan.info["jit_modules"] >= 1


@pytest.mark.parametrize("f16", [False, True])
def test_jit_bitwise_equals_plan_driven(f16):
    # same per-output summation order (k ascending, sequential) -> bitwise identical
    w = gen.pruned_weights(768, 512, 90, seed=41)
    X = gen.uniform_x(512, 3000, seed=42)
    y_jit, pj = _run_spmm(w, X, f16, executor=1)
    y_ref, pr = _run_spmm(w, X, f16, split_k=1, k_split=1)
    assert pj.info["executor"] == 1 and pr.info["executor"] == 0
    assert np.array_equal(y_jit, y_ref)
    assert oracle.rel_l2(y_jit, _ref(w, X, f16)) <= (F16_TOL if f16 else F32_TOL)


@pytest.mark.parametrize("f16", [False, True])
def test_jit_closed_forms_and_fallback(f16):
    K = 300
    w = gen.pruned_weights(513, K, 90, seed=6)
    y, _ = _run_spmm(w, np.eye(K, dtype=np.float32), f16, executor=1)
    wd = gen.to_dense(w.with_values(_w64(w, f16).astype(np.float32)))
    assert np.array_equal(y, wd)
    # unaligned X (ld = 301, odd) -> plan-driven fallback, still exact
    s = gen.row_selection_csr(700, K, seed=5)
    X = gen.uniform_x(K, 301, seed=9)
    y, _ = _run_spmm(s, X, f16, N=299, ld=301, executor=1)
    assert np.array_equal(y, _x64(X, f16)[s.col_idx][:, :299])
    # empty matrix
    z = gen.stress_pattern("empty", 50, K, seed=1)
    y, _ = _run_spmm(z, gen.uniform_x(K, 64, seed=3), f16, executor=1)
    assert np.array_equal(y, np.zeros_like(y))


# --------------------------------------------------------------------------- autotuner

@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("case", [(2048, 512, 392), (256, 64, 3136)])
def test_tuned_plan_exact_and_replicable(case, f16):
    # tune=1 picks a configuration by measurement; whatever it picks is exact on
    # integer data, and its chosen options rebuild an identical replica (same digest)
    M, K, N = case
    plan = _exact_case(M, K, N, 90, f16, seed=M + N, tune=1)
    assert plan.info["tuned_us"] > 0
    w = gen.int_weights(M, K, 90, seed=M + N, vmax=2 if f16 else 3)
    rep = srt.Plan.from_csr(w, dtype=_tdt(f16), n_hint=N, **plan.chosen_opts())
    assert rep.info["digest"] == plan.info["digest"]


def test_auto_executor_choice():
    # auto: JIT for small per-panel code (RN50 p2), plan-driven for large (BERT)
    small = srt.Plan.from_csr(gen.pruned_weights(256, 64, 90, seed=1), n_hint=25088, executor=2)
    big = srt.Plan.from_csr(gen.pruned_weights(768, 3072, 90, seed=1), n_hint=16384, executor=2)
    assert small.info["executor"] == 1 and big.info["executor"] == 0


# --------------------------------------------------------------------------- fused epilogue

@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("opts", [dict(), dict(k_split=4, rows_per_warp=4), dict(executor=1),
                                  dict(split_k=2, warps=8)])
def test_spmm_epilogue_exact(opts, f16):
    # Y = relu(W X + bias + beta Y0) on integer data: exact (fp32 accumulate, one rounding);
    # also through the cluster (k_split) store, a JIT plan (falls back to plan-driven) and
    # split-K groups
    dev = _dev()
    M, K, N = 300, 500, 260
    vmax_w, vmax_x = (2, 4) if f16 else (3, 3)
    w = gen.int_weights(M, K, 90, seed=71, vmax=vmax_w)
    X = gen.int_x(K, N, seed=72, vmax=vmax_x)
    rng = np.random.default_rng(73)
    bias = rng.integers(-8, 9, M).astype(np.float32)
    Y0 = rng.integers(-8, 9, (M, N)).astype(np.float32)
    plan = srt.Plan.from_csr(w, dtype=_tdt(f16), n_hint=N, **opts)
    Xd = torch.from_numpy(X).to(dev).to(_tdt(f16))
    for beta, relu, use_bias in [(0.0, True, True), (2.0, False, True), (-1.0, True, False), (0.0, False, False)]:
        Y = torch.from_numpy(Y0).to(dev).to(_tdt(f16))
        b = torch.from_numpy(bias).to(dev).to(_tdt(f16)) if use_bias else None
        plan.spmm(Xd, Y, bias=b, beta=beta, relu=relu)
        torch.cuda.synchronize()
        ref = _ref(w, X, f16) + (bias[:, None] if use_bias else 0.0) + beta * Y0
        if relu:
            ref = np.maximum(ref, 0.0)
        if f16:
            ref = _f16_round(ref)
        assert np.array_equal(Y.double().cpu().numpy(), ref), (beta, relu, use_bias)


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("ck", [1, 2, 3, 4, 5])
def test_conv_epilogue_exact(ck, f16):
    dev = _dev()
    cin, cout, B, H, W = 24, 40, 2, 14, 14
    vmax_w, vmax_x = (2, 4) if f16 else (3, 3)
    w = gen.int_weights(cout, 9 * cin, 90, seed=81, vmax=vmax_w)
    x = gen.int_x(cin * B * H, W, seed=82, vmax=vmax_x).reshape(cin, B, H, W)
    rng = np.random.default_rng(83)
    bias = rng.integers(-8, 9, cout).astype(np.float32)
    y0 = rng.integers(-8, 9, (cout, B, H, W)).astype(np.float32)
    plan = srt.Plan.from_csr(w, dtype=_tdt(f16), kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W,
                             n_hint=B, conv_kernel=ck)
    y = torch.from_numpy(y0).to(dev).to(_tdt(f16))
    plan.conv3x3(torch.from_numpy(x).to(dev).to(_tdt(f16)), y,
                 bias=torch.from_numpy(bias).to(dev).to(_tdt(f16)), beta=0.5, relu=True)
    torch.cuda.synchronize()
    ref = oracle.conv3x3(cout, w.row_ptr, w.col_idx, _w64(w, f16), _x64(x, f16))
    ref = np.maximum(ref + bias[:, None, None, None] + 0.5 * y0, 0.0)
    if f16:
        ref = _f16_round(ref)
    assert np.array_equal(y.double().cpu().numpy(), ref)


# --------------------------------------------------------------------------- tensor-core sub-blocks

@pytest.mark.parametrize("opts", [dict(), dict(k_split=2, rows_per_warp=4), dict(split_k=2, warps=8),
                                  dict(tc_min_density=25)])
@pytest.mark.parametrize("M,K,N", [(256, 512, 392), (200, 300, 131), (1024, 256, 3136)])
def test_tensor_core_subblocks_exact(M, K, N, opts):
    # dense 16x16 tiles on mma.sync (fp16 x fp16 -> fp32) + the rest on CUDA cores, summed in
    # fp32 before one rounding: exact on integer data, also with the fused epilogue
    dev = _dev()
    w = gen.stress_pattern("block16", M, K, seed=M + K, density=0.1)
    w = w.with_values((np.sign(w.values) * np.random.default_rng(1).integers(1, 3, w.nnz)).astype(np.float32))
    X = gen.int_x(K, N, seed=N, vmax=4)
    y, plan = _run_spmm(w, X, True, **opts)
    assert plan.info["tc_tiles"] > 0
    ref = _f16_round(_ref(w, X, True))
    assert np.array_equal(y, ref)
    bias = torch.arange(M, device=dev, dtype=torch.float16) % 7 - 3
    Xd = torch.from_numpy(X).to(dev).half()
    Y = torch.zeros((M, N), device=dev, dtype=torch.float16)
    plan.spmm(Xd, Y, bias=bias, relu=True)
    torch.cuda.synchronize()
    ref2 = _f16_round(np.maximum(_ref(w, X, True) + bias.double().cpu().numpy()[:, None], 0))
    assert np.array_equal(Y.double().cpu().numpy(), ref2)


def test_tensor_core_subblocks_rel_l2():
    w = gen.stress_pattern("block16", 768, 1024, seed=9, density=0.2)
    X = gen.uniform_x(1024, 2000, seed=10)
    y_tc, p_tc = _run_spmm(w, X, True)
    y_cc, p_cc = _run_spmm(w, X, True, tc_min_density=-1)
    assert p_tc.info["tc_tiles"] > 0 and p_cc.info["tc_tiles"] == 0
    ref = _ref(w, X, True)
    assert oracle.rel_l2(y_tc, ref) <= F16_TOL and oracle.rel_l2(y_cc, ref) <= F16_TOL


# --------------------------------------------------------------------------- condensed-panel tensor cores

@pytest.mark.parametrize("p", [80, 90, 95, 98])
@pytest.mark.parametrize("M,K,N", [(64, 64, 128), (300, 200, 517), (1000, 64, 49), (77, 1111, 300),
                                   (3072, 768, 512)])
def test_tcp_rel_l2(M, K, N, p):
    # executor 3: per 16-row panel the union of nonzero columns runs as a dense
    # mma.sync block (fp16 x fp16, fp32 accumulate), X rows gathered by ldmatrix
    w = gen.pruned_weights(M, K, p, seed=gen.case_seed(f"tcp{M}x{K}x{N}", p))
    X = gen.uniform_x(K, N, seed=N + p + 7)
    y, plan = _run_spmm(w, X, True, executor=3)
    assert plan.info["executor"] == 3
    err = oracle.rel_l2(y, _ref(w, X, True))
    assert err <= F16_TOL, err


@pytest.mark.parametrize("case", [(64, 256, 3136), (512, 2048, 49), (2048, 512, 392), (1024, 1024, 1568),
                                  (3072, 768, 512), (768, 3072, 512), (17, 70, 33), (40, 300, 1),
                                  (48, 128, 8), (16, 64, 4099)])
@pytest.mark.parametrize("p", [0, 50, 90, 98])
def test_tcp_integer_exact(case, p):
    # integer data: every fp32 partial sum is exact, so the tensor-core path (any summation
    # order inside the mma) must equal the RN-even fp16 rounding of the exact result
    M, K, N = case
    _exact_case(M, K, N, p, True, seed=gen.case_seed("tcp" + str(case), p), executor=3)


def test_tcp_closed_forms_and_epilogue():
    dev = _dev()
    K, N = 300, 777
    X = gen.uniform_x(K, N, seed=3)
    z = gen.stress_pattern("empty", 50, K, seed=1)
    y, _ = _run_spmm(z, X, True, executor=3)
    assert np.array_equal(y, np.zeros_like(y))
    y, _ = _run_spmm(gen.identity_csr(K), X, True, executor=3)
    assert np.array_equal(y, _x64(X, True))
    # fused epilogue: relu(W X + bias + 0.5 Y0), integer data -> exact
    M = 96
    w = gen.int_weights(M, K, 90, seed=91, vmax=2)
    Xi = gen.int_x(K, N, seed=92, vmax=4)
    rng = np.random.default_rng(93)
    bias = rng.integers(-8, 9, M).astype(np.float32)
    Y0 = rng.integers(-8, 9, (M, N)).astype(np.float32)
    plan = srt.Plan.from_csr(w, dtype=torch.float16, n_hint=N, executor=3)
    Y = torch.from_numpy(Y0).to(dev).half()
    plan.spmm(torch.from_numpy(Xi).to(dev).half(), Y, bias=torch.from_numpy(bias).to(dev).half(), beta=0.5,
              relu=True)
    torch.cuda.synchronize()
    ref = np.maximum(_ref(w, Xi, True) + bias[:, None] + 0.5 * Y0, 0.0)
    assert np.array_equal(Y.double().cpu().numpy(), _f16_round(ref))


# --------------------------------------------------------------------------- token-major layout

@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("M,K,N,ex", [(3072, 768, 512, 0), (768, 3072, 333, 0), (77, 1111, 49, 0),
                                      (300, 200, 1, 0), (3072, 768, 512, 3)])
def test_linear_token_major(M, K, N, ex, f16):
    # sparse_linear (nn.Linear layout): Y (N, M) = X (N, K) @ W^T, bitwise equal to sparse_spmm on
    # X^T (the transposes are pure data movement), and exact on integer data
    if ex == 3 and not f16:
        pytest.skip("tensor-core panels are fp16 only")
    dev = _dev()
    vmax_w, vmax_x = (2, 4) if f16 else (3, 3)
    w = gen.int_weights(M, K, 90, seed=M + N, vmax=vmax_w)
    Xkn = gen.int_x(K, N, seed=K, vmax=vmax_x)
    plan = srt.Plan.from_csr(w, dtype=_tdt(f16), n_hint=N, executor=ex)
    Xt = torch.from_numpy(np.ascontiguousarray(Xkn.T)).to(dev).to(_tdt(f16))
    Y = plan.linear(Xt)
    Yref = plan.spmm(Xt.t().contiguous())
    torch.cuda.synchronize()
    assert Y.shape == (N, M)
    assert torch.equal(Y, Yref.t())
    ref = _ref(w, Xkn, f16)
    if f16:
        ref = _f16_round(ref)
    assert np.array_equal(Y.double().cpu().numpy(), ref.T)


# --------------------------------------------------------------------------- bf16 (NEXT #4)

def _bf16_f64(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("opts", [dict(), dict(k_split=2, rows_per_warp=4), dict(split_k=2, warps=8),
                                  dict(rows_per_warp=8, k_chunk=64)])
@pytest.mark.parametrize("M,K,N,p", [(64, 64, 128, 90), (300, 200, 517, 80), (1000, 64, 49, 95),
                                     (3072, 768, 512, 90), (77, 1111, 300, 98)])
def test_bf16_rel_l2_and_exact(M, K, N, p, opts):
    # bfloat16 X / W / Y with fp32 accumulation (FHFMA.BF16): rel-L2 <= 1e-2 against the oracle
    # on bf16-rounded inputs, and exact (= RN-even bf16 of the exact sum) on integer data
    dev = _dev()
    w = gen.pruned_weights(M, K, p, seed=gen.case_seed(f"bf{M}x{K}", p))
    X = gen.uniform_x(K, N, seed=N + 3)
    plan = srt.Plan.from_csr(w, dtype=torch.bfloat16, n_hint=N, **opts)
    Y = plan.spmm(torch.from_numpy(X).to(dev).to(torch.bfloat16))
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, _bf16_f64(w.values), _bf16_f64(X))
    err = oracle.rel_l2(Y.double().cpu().numpy(), ref)
    assert err <= F16_TOL, err
    wi = gen.int_weights(M, K, p, seed=M + 1, vmax=2)
    Xi = gen.int_x(K, N, seed=K + 1, vmax=4)
    plan = srt.Plan.from_csr(wi, dtype=torch.bfloat16, n_hint=N, **opts)
    Y = plan.spmm(torch.from_numpy(Xi).to(dev).to(torch.bfloat16))
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), Xi.astype(np.float64))
    assert np.array_equal(Y.double().cpu().numpy(), _bf16_f64(ref))


def test_bf16_epilogue_and_unsupported():
    dev = _dev()
    M, K, N = 96, 300, 777
    w = gen.int_weights(M, K, 90, seed=5, vmax=2)
    Xi = gen.int_x(K, N, seed=6, vmax=4)
    rng = np.random.default_rng(7)
    bias = rng.integers(-8, 9, M).astype(np.float32)
    Y0 = rng.integers(-8, 9, (M, N)).astype(np.float32)
    plan = srt.Plan.from_csr(w, dtype=torch.bfloat16, n_hint=N)
    Y = torch.from_numpy(Y0).to(dev).to(torch.bfloat16)
    plan.spmm(torch.from_numpy(Xi).to(dev).to(torch.bfloat16), Y,
              bias=torch.from_numpy(bias).to(dev).to(torch.bfloat16), beta=0.5, relu=True)
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), Xi.astype(np.float64))
    ref = np.maximum(ref + bias[:, None] + 0.5 * Y0, 0.0)
    assert np.array_equal(Y.double().cpu().numpy(), _bf16_f64(ref))
    for kw in [dict(executor=1), dict(x_source=1)]:
        with pytest.raises(srt.SparseRTError):
            srt.Plan.from_csr(w, dtype=torch.bfloat16, n_hint=N, **kw)


@pytest.mark.parametrize("case", [(64, 256, 3136), (512, 2048, 49), (3072, 768, 512), (17, 70, 33), (16, 64, 4099)])
def test_bf16_tcp_exact(case):
    # the tensor-core panels with bf16 operands (mma.sync ... .bf16): exact on integer data
    dev = _dev()
    M, K, N = case
    w = gen.int_weights(M, K, 90, seed=M + K, vmax=2)
    Xi = gen.int_x(K, N, seed=N, vmax=4)
    plan = srt.Plan.from_csr(w, dtype=torch.bfloat16, n_hint=N, executor=3)
    assert plan.info["executor"] == 3
    Y = plan.spmm(torch.from_numpy(Xi).to(dev).to(torch.bfloat16))
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), Xi.astype(np.float64))
    assert np.array_equal(Y.double().cpu().numpy(), _bf16_f64(ref))


@pytest.mark.parametrize("cin,cout,B,H,W", [(32, 48, 3, 14, 14), (256, 64, 2, 14, 14), (16, 24, 2, 28, 28)])
def test_bf16_conv_exact(cin, cout, B, H, W):
    # bf16 implicit-im2col conv on the TMA-fed kernel: exact on integer data (RN-even bf16 of the
    # exact sum), fused epilogue included; the other conv kernels refuse bf16
    dev = _dev()
    w = gen.int_weights(cout, 9 * cin, 90, seed=cin + W, vmax=2)
    x = gen.int_x(cin * B * H, W, seed=cout, vmax=4).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(w, dtype=torch.bfloat16, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B)
    assert plan.info["conv_kernel"] == 2
    y = plan.conv3x3(torch.from_numpy(x).to(dev).to(torch.bfloat16))
    torch.cuda.synchronize()
    ref = oracle.conv3x3(cout, w.row_ptr, w.col_idx, w.values.astype(np.float64), x.astype(np.float64))
    assert np.array_equal(y.double().cpu().numpy(), _bf16_f64(ref))
    with pytest.raises(srt.SparseRTError):
        srt.Plan.from_csr(w, dtype=torch.bfloat16, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B,
                          conv_kernel=3)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16, torch.float32])
def test_auto_executor_all_dtypes(dt):
    # executor = 2 (auto) builds for every dtype: the JIT where it applies (fp32 / fp16 SpMM with
    # small panels), the plan-driven kernel otherwise (bf16 always); exact on integer data
    dev = _dev()
    M, K, N = 256, 64, 3136
    vw, vx = (3, 3) if dt == torch.float32 else (2, 4)
    w = gen.int_weights(M, K, 90, seed=11, vmax=vw)
    Xi = gen.int_x(K, N, seed=12, vmax=vx)
    plan = srt.Plan.from_csr(w, dtype=dt, n_hint=N, executor=2)
    if dt == torch.bfloat16:
        assert plan.info["executor"] == 0
    Y = plan.spmm(torch.from_numpy(Xi).to(dev).to(dt))
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), Xi.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(dt).double().numpy()
    assert np.array_equal(Y.double().cpu().numpy(), ref)


def test_tune_keeps_current_device():
    _dev()
    torch.cuda.set_device(0)
    w = gen.pruned_weights(128, 128, 90, seed=3)
    plan = srt.Plan.from_csr(w, n_hint=1024, tune=1, device=0)
    assert torch.cuda.current_device() == 0 and plan.info["tuned_us"] > 0


# --------------------------------------------------------------------------- the timed configurations

import glob as _glob
import json as _json
import os as _os

_ROOT = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))


def _tuned_cases():
    import bench
    cases = []
    for path in sorted(_glob.glob(_os.path.join(_ROOT, "profiles", "tuned_*.json"))):
        m = _os.path.basename(path)[len("tuned_"):-len(".json")].split("_")
        # tuned_<workload>_<dtype>_s<sparsity>_x<executor>.json
        wl, dt, sp = "_".join(m[:-3]), m[-3], int(m[-2][1:])
        layers, _, _ = bench.workload_layers(wl, 1, 0)
        opts = _json.load(open(path))
        for L in layers:
            if L["name"] in opts:
                cases.append(pytest.param(L, dt, sp, opts[L["name"]], id=f"{wl}-{dt}-s{sp}-{L['name']}"))
    return cases


@pytest.mark.parametrize("L,dt,sp,opts", _tuned_cases())
def test_tuned_configuration_exact_at_full_size(L, dt, sp, opts):
    # every configuration bench.py times (profiles/tuned_*.json), built with exactly those options
    # at the workload's full size, on integer data: sampled outputs bitwise equal to the oracle
    import bench
    dev = _dev()
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dt]
    w, x = bench.make_inputs(L, sp, 0, integer=True, f16=dt != "f32")
    if L["kind"] == "spmm":
        plan = srt.Plan.from_csr(w, dtype=tdt, n_hint=L["N"], **opts)
        Y = plan.spmm(torch.from_numpy(x).to(dev).to(tdt))
        ids = np.unique(np.r_[0, L["N"] - 1, np.random.default_rng(1).integers(0, L["N"], 48)])
        ref = oracle.spmm(w.M, w.K, w.row_ptr, w.col_idx, w.values.astype(np.float64), x[:, ids].astype(np.float64))
    else:
        plan = srt.Plan.from_csr(w, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=L["c_in"], h=L["H"], w=L["W"],
                                 n_hint=L["B"], **opts)
        Y = plan.conv3x3(torch.from_numpy(x).to(dev).to(tdt))
        ids = np.array([0, 37, 128, 255])
        ref = oracle.conv3x3(w.M, w.row_ptr, w.col_idx, w.values.astype(np.float64), x[:, ids].astype(np.float64))
    torch.cuda.synchronize()
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    got = Y[:, torch.from_numpy(ids).to(dev)].double().cpu().numpy()
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("dt", ["f32", "f16"])
def test_bert_full_size_real_valued(dt):
    # BASELINE configs[3] at full size (N = 32 x 512) with the real-valued synthetic inputs and the
    # tuned options bench.py times: rel-L2 over 256 sampled columns within the north-star gate
    import bench
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    path = _os.path.join(_ROOT, "profiles", f"tuned_bert_{dt}_s90_x2.json")
    tuned = _json.load(open(path)) if _os.path.exists(path) else {}
    layers, _, _ = bench.workload_layers("bert", 1, 0)
    for L in layers:
        w, x = bench.make_inputs(L, 90, 0)
        plan = srt.Plan.from_csr(w, dtype=tdt, n_hint=L["N"], **tuned.get(L["name"], {}))
        Y = plan.spmm(torch.from_numpy(x).to(dev).to(tdt))
        ids = np.unique(np.random.default_rng(2).integers(0, L["N"], 256))
        ref = oracle.spmm(w.M, w.K, w.row_ptr, w.col_idx, _w64(w, dt == "f16"), _x64(x[:, ids], dt == "f16"))
        torch.cuda.synchronize()
        err = oracle.rel_l2(Y[:, torch.from_numpy(ids).to(dev)].double().cpu().numpy(), ref)
        assert err <= (F16_TOL if dt == "f16" else F32_TOL), (L["name"], err)


@pytest.mark.parametrize("dt", ["f32", "f16"])
def test_conv_full_batch_real_valued(dt):
    # BASELINE configs[4] at full size (batch 256) with the real-valued inputs and the tuned
    # options: rel-L2 over 32 sampled images within the north-star gate
    import bench
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    path = _os.path.join(_ROOT, "profiles", f"tuned_conv_{dt}_s90_x2.json")
    tuned = _json.load(open(path)) if _os.path.exists(path) else {}
    L = bench.workload_layers("conv", 1, 0)[0][0]
    w, x = bench.make_inputs(L, 90, 0)
    plan = srt.Plan.from_csr(w, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=256, h=14, w=14, n_hint=256,
                             **tuned.get(L["name"], {}))
    y = plan.conv3x3(torch.from_numpy(x).to(dev).to(tdt))
    ids = np.sort(np.random.default_rng(3).choice(256, 32, replace=False))
    ref = oracle.conv3x3(256, w.row_ptr, w.col_idx, _w64(w, dt == "f16"), _x64(x[:, ids], dt == "f16"))
    torch.cuda.synchronize()
    err = oracle.rel_l2(y[:, torch.from_numpy(ids).to(dev)].double().cpu().numpy(), ref)
    assert err <= (F16_TOL if dt == "f16" else F32_TOL), err


# --------------------------------------------------------------------------- strided 1x1 / NHWC conv (NEXT #4)

@pytest.mark.parametrize("dt", ["f32", "f16"])
@pytest.mark.parametrize("cin,cout,B,h,w,s", [(256, 512, 2, 56, 56, 2), (512, 1024, 3, 28, 28, 2),
                                               (1024, 2048, 2, 14, 14, 2), (64, 96, 3, 15, 9, 2),
                                               (32, 48, 2, 14, 14, 1), (40, 24, 1, 10, 7, 3)])
def test_conv1x1_strided_exact(cin, cout, B, h, w, s, dt):
    # the ResNet-50 stride-2 projection shapes and ragged cases: exact on
    # integer data against the oracle product on the sampled pixels (sampling = input plumbing)
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    vw, vx = (3, 3) if dt == "f32" else (2, 4)
    wi = gen.int_weights(cout, cin, 90, seed=cin + h, vmax=vw)
    x = gen.int_x(cin * B * h, w, seed=cout + s, vmax=vx).reshape(cin, B, h, w)
    plan = srt.Plan.from_csr(wi, dtype=tdt, n_hint=B * ((h + s - 1) // s) * ((w + s - 1) // s))
    y = plan.conv1x1(torch.from_numpy(x).to(dev).to(tdt), stride=s)
    torch.cuda.synchronize()
    xs = np.ascontiguousarray(x[:, :, ::s, ::s])
    ho, wo = xs.shape[2], xs.shape[3]
    ref = oracle.spmm(cout, cin, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64),
                      xs.reshape(cin, -1).astype(np.float64)).reshape(cout, B, ho, wo)
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert y.shape == (cout, B, ho, wo)
    assert np.array_equal(y.double().cpu().numpy(), ref)


@pytest.mark.parametrize("opts", [{}, {"conv_kernel": 5}, {"conv_kernel": 5, "cta_pair": 1}])
@pytest.mark.parametrize("dt", ["f32", "f16"])
@pytest.mark.parametrize("cin,cout,B,H,W", [(64, 64, 2, 56, 56), (256, 256, 3, 14, 14), (12, 20, 2, 7, 9)])
def test_conv3x3_nhwc_exact(cin, cout, B, H, W, dt, opts):
    # channels-last activations: exact on integer data, and bitwise the CNHW call (conv_kernel 5:
    # the im2col TMA reads NHWC in place and the epilogue writes NHWC, no transposes)
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    vw, vx = (3, 3) if dt == "f32" else (2, 4)
    wi = gen.int_weights(cout, 9 * cin, 90, seed=cin + W, vmax=vw)
    x = gen.int_x(cin * B * H, W, seed=cout, vmax=vx).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(wi, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, **opts)
    xt = torch.from_numpy(x).to(dev).to(tdt)
    y_nhwc = plan.conv3x3_nhwc(xt.permute(1, 2, 3, 0).contiguous())
    y_cnhw = plan.conv3x3(xt)
    torch.cuda.synchronize()
    assert torch.equal(y_nhwc, y_cnhw.permute(1, 2, 3, 0))
    ref = oracle.conv3x3(cout, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), x.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(y_cnhw.double().cpu().numpy(), ref)


# --------------------------------------------------------------------------- plan in kernel parameters (NEXT #2)

@pytest.mark.parametrize("dt", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("M,K,N,opts", [(64, 64, 128, {}), (64, 256, 25088, dict(rows_per_warp=2)),
                                         (256, 64, 3136, {}), (64, 32, 12544, dict(warps=8)),
                                         (128, 64, 1000, dict(rows_per_warp=8, k_chunk=32, stages=4)),
                                         (96, 100, 77, dict(rows_per_warp=1))])
def test_param_plan_exact_and_bitwise(M, K, N, opts, dt):
    # plan_source = 1: the plan as a kernel parameter read through the constant cache:
    # exact on integer data and bitwise equal to the staged-plan kernel on real-valued data
    dev = _dev()
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dt]
    vw, vx = (3, 3) if dt == "f32" else (2, 4)
    wi = gen.int_weights(M, K, 90, seed=M + K, vmax=vw)
    xi = gen.int_x(K, N, seed=N, vmax=vx)
    plan = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, plan_source=1, **opts)
    assert plan.info["plan_source"] == 1
    y = plan.spmm(torch.from_numpy(xi).to(dev).to(tdt))
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), xi.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(y.double().cpu().numpy(), ref)
    w = gen.pruned_weights(M, K, 90, seed=M * 3 + K)
    x = torch.from_numpy(gen.uniform_x(K, N, seed=5)).to(dev).to(tdt)
    p1 = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, plan_source=1, **opts)
    p0 = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, plan_source=0, tc_min_density=-1, split_k=1, k_split=1, **opts)
    assert torch.equal(p1.spmm(x), p0.spmm(x))
    with pytest.raises(srt.SparseRTError):  # too large for the parameter space
        srt.Plan.from_csr(gen.pruned_weights(3072, 768, 90, seed=1), dtype=tdt, n_hint=N, plan_source=1)


@pytest.mark.parametrize("dt", ["f32", "f16"])
def test_conv_interleaved_overlapped_prepass_exact(dt, monkeypatch):
    # the opt-in overlapped form (pre-pass and conv kernel concurrently, per-image-group ready
    # counters): exact on integer data, bitwise equal to the sequential form
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    cin, cout, B, H, W = 64, 48, 9, 14, 14
    vw, vx = (3, 3) if dt == "f32" else (2, 4)
    w = gen.int_weights(cout, 9 * cin, 90, seed=91, vmax=vw)
    x = gen.int_x(cin * B * H, W, seed=92, vmax=vx).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(w, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B,
                             conv_kernel=4, rows_per_warp=4, k_chunk=8, stages=2)
    xt = torch.from_numpy(x).to(dev).to(tdt)
    monkeypatch.setenv("SPARSERT_CONV_OVERLAP", "1")
    y1 = plan.conv3x3(xt)
    torch.cuda.synchronize()
    monkeypatch.setenv("SPARSERT_CONV_OVERLAP", "0")
    y0 = plan.conv3x3(xt)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    ref = oracle.conv3x3(cout, w.row_ptr, w.col_idx, w.values.astype(np.float64), x.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(y1.double().cpu().numpy(), ref)


# --------------------------------------------------------------------------- tcgen05 blocks (executor 4)

@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("M,K,N,p", [(3072, 768, 2048, 90), (768, 3072, 512, 90), (300, 200, 517, 80),
                                      (128, 64, 256, 95), (77, 1111, 300, 98), (2048, 512, 392, 90),
                                      (16, 64, 4099, 90), (512, 2048, 49, 95)])
def test_tcgen05_blocks_exact_and_rel_l2(M, K, N, p, dt):
    # W's nonzero 128 x 64 blocks on tcgen05.mma (TMEM accumulators): exact on integer data
    # (every partial sum an exact integer < 2^24, so the tensor core's internal order does not
    # matter; 16-bit output = RN of the exact sum), rel-L2 <= 1e-2 on real-valued data
    dev = _dev()
    tdt = torch.bfloat16 if dt == "bf16" else torch.float16
    wi = gen.int_weights(M, K, p, seed=M + K + N, vmax=2)
    xi = gen.int_x(K, N, seed=N + 1, vmax=4)
    plan = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, executor=4)
    assert plan.info["executor"] == 4
    Y = torch.full((M, N), float("nan"), dtype=tdt, device=dev)
    plan.spmm(torch.from_numpy(xi).to(dev).to(tdt), Y)
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), xi.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(Y.double().cpu().numpy(), ref)
    w = gen.pruned_weights(M, K, p, seed=M * 7 + K)
    x = gen.uniform_x(K, N, seed=3)
    plan = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, executor=4)
    Y = plan.spmm(torch.from_numpy(x).to(dev).to(tdt))
    torch.cuda.synchronize()
    wv = torch.from_numpy(w.values).to(tdt).double().numpy()
    xv = torch.from_numpy(x).to(tdt).double().numpy()
    err = oracle.rel_l2(Y.double().cpu().numpy(), oracle.spmm(M, K, w.row_ptr, w.col_idx, wv, xv))
    assert err <= F16_TOL, err


def test_tcgen05_blocks_empty_rows_epilogue_and_ld():
    # empty row blocks (-> +0), ldx / ldy > N, fused bias + beta + ReLU
    dev = _dev()
    M, K, N = 400, 192, 300
    base = gen.int_weights(M, K, 90, seed=4, vmax=2)
    dense = gen.to_dense(base)
    dense[128:256] = 0.0  # a whole empty 128-row block
    keep = np.flatnonzero(dense)
    w = gen.csr_from_mask(M, K, keep, dense.astype(np.float32))
    xi = gen.int_x(K, N, seed=5, vmax=4)
    rng = np.random.default_rng(6)
    bias = rng.integers(-8, 9, M).astype(np.float32)
    y0 = rng.integers(-8, 9, (M, N)).astype(np.float32)
    plan = srt.Plan.from_csr(w, dtype=torch.float16, n_hint=N, executor=4)
    Xb = torch.zeros((K, N + 40), dtype=torch.float16, device=dev)
    Xb[:, :N] = torch.from_numpy(xi).to(dev).half()
    Yb = torch.zeros((M, N + 24), dtype=torch.float16, device=dev)
    Yb[:, :N] = torch.from_numpy(y0).to(dev).half()
    plan.spmm(Xb[:, :N], Yb[:, :N], bias=torch.from_numpy(bias).to(dev).half(), beta=0.5, relu=True)
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), xi.astype(np.float64))
    ref = np.maximum(ref + bias[:, None] + 0.5 * y0, 0.0)
    assert np.array_equal(Yb[:, :N].double().cpu().numpy(), _f16_round(ref))
    assert torch.count_nonzero(Yb[:, N:]) == 0


@pytest.mark.parametrize("dt", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("cin,cout,B,H,W,p", [(256, 256, 6, 14, 14, 90), (64, 64, 3, 56, 56, 90),
                                              (128, 128, 4, 28, 28, 95), (512, 512, 3, 7, 7, 90),
                                              (40, 200, 5, 10, 6, 80), (16, 24, 2, 14, 14, 90)])
def test_conv_tcgen05_exact(cin, cout, B, H, W, p, dt):
    # conv_kernel 5: implicit im2col over the interleaved copies on the tcgen05 block executor
    # (k-blocks = (tap, 64 channels); fp32: (tap, 32 channels) as 3xTF32): exact on integer
    # data, rel-L2 <= 1e-2 (16-bit) / 1e-5 (fp32) on real data
    dev = _dev()
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[dt]
    wi = gen.int_weights(cout, 9 * cin, p, seed=cin + H, vmax=2)
    x = gen.int_x(cin * B * H, W, seed=cout, vmax=4).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(wi, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, conv_kernel=5)
    assert plan.info["conv_kernel"] == 5
    y = torch.full((cout, B, H, W), float("nan"), dtype=tdt, device=dev)
    plan.conv3x3(torch.from_numpy(x).to(dev).to(tdt), y)
    torch.cuda.synchronize()
    ref = oracle.conv3x3(cout, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), x.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(y.double().cpu().numpy(), ref)
    w = gen.pruned_weights(cout, 9 * cin, p, seed=cin * 5 + H)
    xr = gen.relu_normal_x((cin, B, H, W), seed=B + 5)
    plan = srt.Plan.from_csr(w, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, conv_kernel=5)
    y = plan.conv3x3(torch.from_numpy(xr).to(dev).to(tdt))
    torch.cuda.synchronize()
    wv = torch.from_numpy(w.values).to(tdt).double().numpy()
    xv = torch.from_numpy(xr).to(tdt).double().numpy()
    err = oracle.rel_l2(y.double().cpu().numpy(), oracle.conv3x3(cout, w.row_ptr, w.col_idx, wv, xv))
    assert err <= (F32_TOL if dt == "f32" else F16_TOL), err


# ------------------------------------------- tcgen05 blocks: multicast clusters, fp32 as 3xTF32

@pytest.mark.parametrize("dt", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("cs", [1, 2, 4])
@pytest.mark.parametrize("M,K,N,p", [(3072, 768, 2048, 90), (768, 3072, 512, 95), (300, 200, 517, 80),
                                      (77, 1111, 300, 98), (640, 512, 392, 90), (16, 64, 4099, 90)])
def test_tcgen05_clusters_and_tf32_exact(M, K, N, p, cs, dt):
    # executor 4 with x_multicast = cs (row blocks of a cluster share every X tile; a group walks
    # the union of its row blocks' k-blocks, zero blocks where a row block lacks one) and fp32
    # plans as 3xTF32: BITWISE on integer data (|w| <= 2, |x| <= 4 are exact TF32 values, the
    # low halves are 0 and every partial sum is an exact integer < 2^24)
    dev = _dev()
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[dt]
    wi = gen.int_weights(M, K, p, seed=M + K + N + cs, vmax=2)
    xi = gen.int_x(K, N, seed=N + cs, vmax=4)
    plan = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, executor=4, x_multicast=cs)
    assert plan.info["executor"] == 4 and plan.info["x_multicast"] == cs
    Y = torch.full((M, N), float("nan"), dtype=tdt, device=dev)
    plan.spmm(torch.from_numpy(xi).to(dev).to(tdt), Y)
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), xi.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(Y.double().cpu().numpy(), ref)
    # the replica rebuilt from chosen_opts has the same digest (cluster size in the digest)
    again = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, **plan.chosen_opts())
    assert again.info["digest"] == plan.info["digest"]


@pytest.mark.parametrize("cs", [1, 2, 4])
@pytest.mark.parametrize("M,K,N,p", [(3072, 768, 2048, 90), (768, 3072, 1000, 90), (300, 200, 517, 80),
                                      (512, 2048, 392, 95), (77, 1111, 300, 98), (128, 64, 49, 90)])
def test_tcgen05_tf32x3_rel_l2(M, K, N, p, cs):
    # fp32 on the tensor cores: 3xTF32 (W_hi X_hi + W_lo X_hi + W_hi X_lo) must meet the fp32
    # bar of the north star (rel-L2 <= 1e-5) on real-valued data; one TF32 product alone would
    # not (~1e-4)
    dev = _dev()
    w = gen.pruned_weights(M, K, p, seed=M * 3 + K + cs)
    x = gen.uniform_x(K, N, seed=N + 7)
    plan = srt.Plan.from_csr(w, dtype=torch.float32, n_hint=N, executor=4, x_multicast=cs)
    Y = plan.spmm(torch.from_numpy(x).to(dev))
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), x.astype(np.float64))
    err = oracle.rel_l2(Y.double().cpu().numpy(), ref)
    assert err <= F32_TOL, err


def test_tcgen05_tf32x3_epilogue_ld_unaligned():
    # fp32 / 3xTF32: empty 128-row block (-> +0), X with an odd row stride (not 16-byte
    # aligned: the on-device split handles any ldx), ldy > N, fused bias + beta + ReLU
    dev = _dev()
    M, K, N = 400, 192, 301
    base = gen.int_weights(M, K, 90, seed=14, vmax=3)
    dense = gen.to_dense(base)
    dense[128:256] = 0.0
    keep = np.flatnonzero(dense)
    w = gen.csr_from_mask(M, K, keep, dense.astype(np.float32))
    xi = gen.int_x(K, N, seed=15, vmax=3)
    rng = np.random.default_rng(16)
    bias = rng.integers(-8, 9, M).astype(np.float32)
    y0 = rng.integers(-8, 9, (M, N)).astype(np.float32)
    for cs in (1, 2, 4):
        plan = srt.Plan.from_csr(w, dtype=torch.float32, n_hint=N, executor=4, x_multicast=cs)
        Xb = torch.zeros((K, N + 3), dtype=torch.float32, device=dev)
        Xb[:, :N] = torch.from_numpy(xi).to(dev)
        Yb = torch.zeros((M, N + 24), dtype=torch.float32, device=dev)
        Yb[:, :N] = torch.from_numpy(y0).to(dev)
        plan.spmm(Xb[:, :N], Yb[:, :N], bias=torch.from_numpy(bias).to(dev), beta=0.5, relu=True)
        torch.cuda.synchronize()
        ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), xi.astype(np.float64))
        ref = np.maximum(ref + bias[:, None] + 0.5 * y0, 0.0)
        assert np.array_equal(Yb[:, :N].double().cpu().numpy(), ref.astype(np.float32).astype(np.float64))
        assert torch.count_nonzero(Yb[:, N:]) == 0


@pytest.mark.parametrize("dt", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("cin,cout,B,H,W,p", [(256, 256, 6, 14, 14, 90), (128, 384, 3, 28, 28, 95),
                                              (40, 200, 5, 10, 6, 80)])
def test_conv_tcgen05_cluster_exact(cin, cout, B, H, W, p, dt):
    # conv_kernel 5 with the two (or more) 128-channel row blocks in one multicast cluster
    dev = _dev()
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[dt]
    wi = gen.int_weights(cout, 9 * cin, p, seed=cin + H + 1, vmax=2)
    x = gen.int_x(cin * B * H, W, seed=cout + 1, vmax=4).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(wi, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, conv_kernel=5,
                             x_multicast=2)
    assert plan.info["conv_kernel"] == 5 and plan.info["x_multicast"] == 2
    y = torch.full((cout, B, H, W), float("nan"), dtype=tdt, device=dev)
    plan.conv3x3(torch.from_numpy(x).to(dev).to(tdt), y)
    torch.cuda.synchronize()
    ref = oracle.conv3x3(cout, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), x.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(y.double().cpu().numpy(), ref)


# ------------------------------------------- tcgen05 blocks: split tail (column slices)

@pytest.mark.parametrize("dt", ["f16", "f32"])
@pytest.mark.parametrize("M,K,N,cs", [(128, 512, 38300, 1), (256, 320, 38400, 2), (128, 64, 37000, 1)])
def test_tcgen05_split_tail(M, K, N, cs, dt, monkeypatch):
    # ~150 tiles on 148 (74) persistent CTAs (clusters): the last round's tiles run as column
    # slices on otherwise idle clusters (N = 256 / sp MMAs).  Exact on integer data with and
    # without the split, and the split changes nothing on real-valued data beyond the tolerance
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    tol = F16_TOL if dt == "f16" else F32_TOL
    wi = gen.int_weights(M, K, 90, seed=M + K + cs, vmax=2)
    xi = gen.int_x(K, N, seed=N % 1000, vmax=4)
    plan = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, executor=4, x_multicast=cs)
    ref = oracle.spmm(M, K, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), xi.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    X = torch.from_numpy(xi).to(dev).to(tdt)
    outs = {}
    for st in ("0", "8"):
        monkeypatch.setenv("SRT_TCG_SPLIT_TAIL", st)
        Y = torch.full((M, N), float("nan"), dtype=tdt, device=dev)
        plan.spmm(X, Y)
        torch.cuda.synchronize()
        assert np.array_equal(Y.double().cpu().numpy(), ref), st
    w = gen.pruned_weights(M, K, 90, seed=M * 5 + K)
    x = gen.uniform_x(K, N, seed=11)
    plan = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, executor=4, x_multicast=cs)
    wv = torch.from_numpy(w.values).to(tdt).double().numpy()
    xv = torch.from_numpy(x).to(tdt).double().numpy()
    exact = oracle.spmm(M, K, w.row_ptr, w.col_idx, wv, xv)
    for st in ("0", "8"):
        monkeypatch.setenv("SRT_TCG_SPLIT_TAIL", st)
        Y = plan.spmm(torch.from_numpy(x).to(dev).to(tdt))
        torch.cuda.synchronize()
        outs[st] = Y.double().cpu().numpy()
        assert oracle.rel_l2(outs[st], exact) <= tol
    assert oracle.rel_l2(outs["8"], outs["0"]) <= tol


@pytest.mark.parametrize("dt", ["f16", "f32"])
def test_conv_tcgen05_split_tail(dt, monkeypatch):
    # the C5 conv at batch 256: 224 tiles on 74 clusters -> 2 tail tiles as column slices
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    cin = cout = 256
    B, H, W = 256, 14, 14
    wi = gen.int_weights(cout, 9 * cin, 90, seed=71, vmax=2)
    x = gen.int_x(cin * B * H, W, seed=72, vmax=4).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(wi, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, conv_kernel=5,
                             x_multicast=2)
    xd = torch.from_numpy(x).to(dev).to(tdt)
    outs = {}
    for st in ("0", "8"):
        monkeypatch.setenv("SRT_TCG_SPLIT_TAIL", st)
        y = torch.full((cout, B, H, W), float("nan"), dtype=tdt, device=dev)
        plan.conv3x3(xd, y)
        torch.cuda.synchronize()
        outs[st] = y
    assert torch.equal(outs["0"], outs["8"])
    # the last images (the tail tiles' span) against the oracle
    sel = list(range(B - 12, B))
    ref = oracle.conv3x3(cout, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64),
                         np.ascontiguousarray(x[:, sel]).astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(outs["8"][:, sel].double().cpu().numpy(), ref)


# ------------------------------------------- tcgen05 blocks: CTA pairs (cta_group::2, M = 256)

@pytest.mark.parametrize("dt", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("M,K,N,p", [(3072, 768, 2048, 90), (768, 3072, 512, 95), (300, 200, 517, 80),
                                      (256, 64, 256, 90), (640, 512, 392, 90), (130, 1111, 300, 98),
                                      (512, 256, 38300, 90)])
def test_tcgen05_pair_exact(M, K, N, p, dt):
    # two consecutive 128-row blocks per CTA pair: one tcgen05.mma.cta_group::2 (M = 256) per
    # step, each CTA staging its W block and half of the X tile.  Bitwise on integer data;
    # real-valued data within the dtype's tolerance
    dev = _dev()
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[dt]
    wi = gen.int_weights(M, K, p, seed=M + 3 * K + N, vmax=2)
    xi = gen.int_x(K, N, seed=N + 5, vmax=4)
    plan = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, executor=4, cta_pair=1)
    assert plan.info["executor"] == 4 and plan.info["cta_pair"] == 1 and plan.info["x_multicast"] == 2
    Y = torch.full((M, N), float("nan"), dtype=tdt, device=dev)
    plan.spmm(torch.from_numpy(xi).to(dev).to(tdt), Y)
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), xi.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(Y.double().cpu().numpy(), ref)
    again = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, **plan.chosen_opts())
    assert again.info["digest"] == plan.info["digest"] and again.info["cta_pair"] == 1
    w = gen.pruned_weights(M, K, p, seed=M * 11 + K)
    x = gen.uniform_x(K, N, seed=N + 9)
    plan = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, executor=4, cta_pair=1)
    Y = plan.spmm(torch.from_numpy(x).to(dev).to(tdt))
    torch.cuda.synchronize()
    wv = torch.from_numpy(w.values).to(tdt).double().numpy()
    xv = torch.from_numpy(x).to(tdt).double().numpy()
    err = oracle.rel_l2(Y.double().cpu().numpy(), oracle.spmm(M, K, w.row_ptr, w.col_idx, wv, xv))
    assert err <= (F32_TOL if dt == "f32" else F16_TOL), err


@pytest.mark.parametrize("dt", ["f16", "f32"])
def test_tcgen05_pair_epilogue(dt):
    # empty 128-row block (-> +0 in one CTA of a pair), ldx / ldy > N, bias + beta + ReLU
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    M, K, N = 400, 192, 300
    base = gen.int_weights(M, K, 90, seed=24, vmax=2)
    dense = gen.to_dense(base)
    dense[128:256] = 0.0
    keep = np.flatnonzero(dense)
    w = gen.csr_from_mask(M, K, keep, dense.astype(np.float32))
    xi = gen.int_x(K, N, seed=25, vmax=4)
    rng = np.random.default_rng(26)
    bias = rng.integers(-8, 9, M).astype(np.float32)
    y0 = rng.integers(-8, 9, (M, N)).astype(np.float32)
    plan = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, executor=4, cta_pair=1)
    Xb = torch.zeros((K, N + 40), dtype=tdt, device=dev)
    Xb[:, :N] = torch.from_numpy(xi).to(dev).to(tdt)
    Yb = torch.zeros((M, N + 24), dtype=tdt, device=dev)
    Yb[:, :N] = torch.from_numpy(y0).to(dev).to(tdt)
    plan.spmm(Xb[:, :N], Yb[:, :N], bias=torch.from_numpy(bias).to(dev).to(tdt), beta=0.5, relu=True)
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), xi.astype(np.float64))
    ref = np.maximum(ref + bias[:, None] + 0.5 * y0, 0.0)
    ref = _f16_round(ref) if dt == "f16" else ref.astype(np.float32).astype(np.float64)
    assert np.array_equal(Yb[:, :N].double().cpu().numpy(), ref)
    assert torch.count_nonzero(Yb[:, N:]) == 0


@pytest.mark.parametrize("dt", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("cin,cout,B,H,W,p", [(256, 256, 6, 14, 14, 90), (128, 384, 3, 28, 28, 95),
                                              (40, 200, 5, 10, 6, 80), (256, 256, 256, 14, 14, 90)])
def test_conv_tcgen05_pair_exact(cin, cout, B, H, W, p, dt):
    # conv_kernel 5 on CTA pairs; batch 256 = the C5 bench shape (split tail included)
    dev = _dev()
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[dt]
    wi = gen.int_weights(cout, 9 * cin, p, seed=cin + H + 7, vmax=2)
    x = gen.int_x(cin * B * H, W, seed=cout + 7, vmax=4).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(wi, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, conv_kernel=5,
                             cta_pair=1)
    assert plan.info["conv_kernel"] == 5 and plan.info["cta_pair"] == 1
    y = torch.full((cout, B, H, W), float("nan"), dtype=tdt, device=dev)
    plan.conv3x3(torch.from_numpy(x).to(dev).to(tdt), y)
    torch.cuda.synchronize()
    sel = list(range(B)) if B <= 8 else [0, 1, 2, B // 2, B - 3, B - 2, B - 1]
    ref = oracle.conv3x3(cout, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64),
                         np.ascontiguousarray(x[:, sel]).astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(y[:, sel].double().cpu().numpy(), ref)


# ------------------------------------------- tcgen05 blocks: K slices per tile (small N)

@pytest.mark.parametrize("dt", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("pair", [0, 1])
@pytest.mark.parametrize("M,K,N,ks", [(512, 2048, 392, 16), (2048, 512, 392, 4), (256, 1024, 1568, 8),
                                       (300, 200, 517, 2), (128, 3072, 49, 16)])
def test_tcgen05_kslices_exact(M, K, N, ks, pair, dt):
    # k_split = ks on the tcgen05 block executor: every tile's k-blocks cut into ks slices on
    # different CTAs, fp32 partials summed in slice order by tcg_ksum.  Bitwise on integer data;
    # real-valued data within the dtype's tolerance
    dev = _dev()
    if pair and M <= 128:
        pytest.skip("a CTA pair needs two row blocks")
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[dt]
    wi = gen.int_weights(M, K, 90, seed=M + K + ks, vmax=2)
    xi = gen.int_x(K, N, seed=N + ks, vmax=4)
    plan = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, executor=4, k_split=ks, cta_pair=pair)
    assert plan.info["executor"] == 4 and plan.info["k_split"] == ks
    Y = torch.full((M, N), float("nan"), dtype=tdt, device=dev)
    plan.spmm(torch.from_numpy(xi).to(dev).to(tdt), Y)
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), xi.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(Y.double().cpu().numpy(), ref)
    again = srt.Plan.from_csr(wi, dtype=tdt, n_hint=N, **plan.chosen_opts())
    assert again.info["digest"] == plan.info["digest"]
    w = gen.pruned_weights(M, K, 90, seed=M * 13 + K)
    x = gen.uniform_x(K, N, seed=N + 19)
    plan = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, executor=4, k_split=ks, cta_pair=pair)
    Y = plan.spmm(torch.from_numpy(x).to(dev).to(tdt))
    torch.cuda.synchronize()
    wv = torch.from_numpy(w.values).to(tdt).double().numpy()
    xv = torch.from_numpy(x).to(tdt).double().numpy()
    err = oracle.rel_l2(Y.double().cpu().numpy(), oracle.spmm(M, K, w.row_ptr, w.col_idx, wv, xv))
    assert err <= (F32_TOL if dt == "f32" else F16_TOL), err


@pytest.mark.parametrize("dt", ["f16", "f32"])
def test_tcgen05_kslices_epilogue(dt):
    # K slices + fused bias / beta / ReLU (applied once, by the ordered sum), ldy > N
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    M, K, N = 400, 1024, 300
    w = gen.int_weights(M, K, 90, seed=34, vmax=2)
    xi = gen.int_x(K, N, seed=35, vmax=4)
    rng = np.random.default_rng(36)
    bias = rng.integers(-8, 9, M).astype(np.float32)
    y0 = rng.integers(-8, 9, (M, N)).astype(np.float32)
    plan = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, executor=4, k_split=8, cta_pair=1)
    Yb = torch.zeros((M, N + 24), dtype=tdt, device=dev)
    Yb[:, :N] = torch.from_numpy(y0).to(dev).to(tdt)
    plan.spmm(torch.from_numpy(xi).to(dev).to(tdt), Yb[:, :N], bias=torch.from_numpy(bias).to(dev).to(tdt),
              beta=0.5, relu=True)
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), xi.astype(np.float64))
    ref = np.maximum(ref + bias[:, None] + 0.5 * y0, 0.0)
    ref = _f16_round(ref) if dt == "f16" else ref.astype(np.float32).astype(np.float64)
    assert np.array_equal(Yb[:, :N].double().cpu().numpy(), ref)
    assert torch.count_nonzero(Yb[:, N:]) == 0


@pytest.mark.parametrize("dt", ["f16", "f32"])
@pytest.mark.parametrize("opts", [{"conv_kernel": 5}, {"conv_kernel": 5, "cta_pair": 1},
                                  {"conv_kernel": 5, "x_multicast": 2}])
@pytest.mark.parametrize("cin,cout,B,H,W", [(256, 256, 1, 14, 14), (64, 130, 1, 56, 56), (128, 512, 1, 7, 7),
                                            (96, 256, 7, 13, 11)])
def test_conv_tcgen05_small_batch(cin, cout, B, H, W, opts, dt):
    # batch 1 (the Table-3 convs) and odd sizes on the im2col path: few tiles for 148 SMs (tile
    # widths / tail slices chosen at launch), pixels crossing image boundaries inside a tile
    dev = _dev()
    tdt = torch.float16 if dt == "f16" else torch.float32
    wi = gen.int_weights(cout, 9 * cin, 90, seed=cin + cout + H, vmax=2)
    x = gen.int_x(cin * B * H, W, seed=W + B, vmax=4).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(wi, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, **opts)
    y = torch.full((cout, B, H, W), float("nan"), dtype=tdt, device=dev)
    plan.conv3x3(torch.from_numpy(x).to(dev).to(tdt), y)
    torch.cuda.synchronize()
    ref = oracle.conv3x3(cout, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), x.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    assert np.array_equal(y.double().cpu().numpy(), ref)
