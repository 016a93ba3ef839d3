"""CPU-only tests of the C ABI library: it loads, exports every symbol include/sparsert.h
declares, and its host-side inspector (plans built with SPARSE_DEVICE_HOST_ONLY, no GPU)
keeps every nonzero exactly once, balances panels / groups as PAPER.md Sec. 3.4 describes,
is deterministic, and rejects invalid CSR input with the documented status codes."""
import ctypes
import os
import re
import subprocess

import numpy as np
import torch
import pytest

from synth import gen
from sparsert_testutil import golden, ROOT

import paper_2008_11849_b200 as srt
from paper_2008_11849_b200 import sparsert as S

HOST = dict(device=srt.SPARSE_DEVICE_HOST_ONLY)


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "sparsert.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(\w+)\s*\(", hdr, re.M))
    declared -= {"if", "return"}
    assert {"sparse_plan_create", "sparse_spmm", "sparse_conv3x3", "plan_destroy"} <= declared
    out = subprocess.check_output(["nm", "-D", "--defined-only", S.LIB_PATH]).decode()
    exported = {l.split()[-1] for l in out.splitlines() if l.strip()}
    missing = declared - exported
    assert not missing, missing
    assert declared == set(S.EXPORTED)
    for name in declared:
        assert hasattr(S.lib, name)


def test_version_and_sm100a_code():
    assert "sm_100a" in srt.version()
    sass = subprocess.run(["cuobjdump", "--list-elf", S.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in sass.stdout


def _plan(csr, dtype=None, **kw):
    import torch
    return srt.Plan.from_csr(csr, dtype=dtype or torch.float32, **HOST, **kw)


@pytest.mark.parametrize("M,K,p,n_hint", [(64, 64, 90, 128), (2048, 512, 90, 49), (3072, 768, 95, 512),
                                          (256, 1024, 90, 196), (37, 1000, 80, 7), (1, 1, 0, 1)])
@pytest.mark.parametrize("f16", [False, True])
def test_inspector_coverage_and_order(M, K, p, n_hint, f16):
    import torch
    w = gen.pruned_weights(M, K, p, seed=M + K)
    pl = _plan(w, torch.float16 if f16 else torch.float32, n_hint=n_hint)
    d = pl.dump()
    assert pl.info["nnz"] == w.nnz == d.row.size
    # every nonzero exactly once, with its value (fp16-rounded for fp16 plans)
    key = d.row.astype(np.int64) * K + d.col
    ref_rows = np.repeat(np.arange(M), np.diff(w.row_ptr)).astype(np.int64)
    ref_key = ref_rows * K + w.col_idx
    order = np.argsort(key)
    assert np.array_equal(key[order], np.sort(ref_key))
    ref_val = dict(zip(ref_key.tolist(), w.values.tolist()))
    exp = np.array([ref_val[k] for k in key[order].tolist()], np.float32)
    if f16:
        exp = exp.astype(np.float16).astype(np.float32)
    assert np.array_equal(d.value[order], exp)
    # storage order: within a (row, chunk) entries are k-ascending; chunks hold their k range
    info = pl.info
    kc = info["k_chunk"]
    assert np.all(d.col // kc == d.chunk)
    same = (d.row[1:] == d.row[:-1]) & (d.chunk[1:] == d.chunk[:-1])
    assert np.all(d.col[1:][same] > d.col[:-1][same])
    # every row lives in exactly one (panel, slot)
    ps = {}
    for r, q, s in zip(d.row, d.panel, d.slot):
        ps.setdefault(int(r), set()).add((int(q), int(s)))
    assert all(len(v) == 1 for v in ps.values())


def test_panel_balance_and_group_split():
    w = gen.pruned_weights(1024, 512, 90, seed=3)
    pl = _plan(w, n_hint=1024)
    info = pl.info
    mean = w.nnz / info["panels"]
    # LPT over nnz-sorted rows: max panel within one max-row of the mean
    max_row = np.diff(w.row_ptr).max()
    assert info["max_panel_nnz"] <= mean + max_row
    assert info["min_panel_nnz"] >= mean - max_row
    # split-K groups: all non-trailing groups hold exactly the same number of nonzeros
    # (P:167): ceil(cnt/G) rounded up to the 2-entry broadcast-load width of fp32 entries
    pl = _plan(w, n_hint=49, split_k=4)
    d = pl.dump()
    assert pl.info["split_k"] == 4
    for (r, c) in {(int(a), int(b)) for a, b in zip(d.row[:200], d.chunk[:200])}:
        sel = (d.row == r) & (d.chunk == c)
        cnt = int(sel.sum())
        per = -(-cnt // 4)
        per = -(-per // 2) * 2
        sizes = [int(((d.group == g) & sel).sum()) for g in range(4)]
        assert sizes == [min(per, max(0, cnt - g * per)) for g in range(4)]


def test_row_order_natural_panels():
    # row_order = 1 (the "no load balancing" ablation): panel q holds rows q*Mp..,
    # warp slots in natural order; default LPT panels are balanced within one max row
    w = gen.stress_pattern("zipf", 512, 256, seed=5)
    nat = _plan(w, n_hint=1024, warps=8, rows_per_warp=4, row_order=1)
    assert nat.info["row_order"] == 1
    d = nat.dump()
    assert np.array_equal(d.panel, d.row // 32)
    assert np.array_equal(d.slot, d.row % 32)
    lpt = _plan(w, n_hint=1024, warps=8, rows_per_warp=4)
    spread = lambda pl: pl.info["max_panel_nnz"] - pl.info["min_panel_nnz"]
    assert spread(lpt) <= np.diff(w.row_ptr).max()
    assert spread(nat) > spread(lpt)


def test_tensor_core_subblock_extraction():
    # NEXT #1: aligned 16x16 tiles with >= 50% nonzeros leave the CUDA-core plan (fp16 only);
    # the dump still carries every nonzero exactly once with its fp16 value
    import torch
    w = gen.stress_pattern("block16", 200, 300, seed=3, density=0.1)
    pl = _plan(w, torch.float16, n_hint=512)
    info = pl.info
    assert info["tc_tiles"] > 0 and info["tc_min_density"] == 50
    d = pl.dump()
    key = np.sort(d.row.astype(np.int64) * 300 + d.col)
    ref_rows = np.repeat(np.arange(200), np.diff(w.row_ptr)).astype(np.int64)
    assert np.array_equal(key, np.sort(ref_rows * 300 + w.col_idx))
    tc = d.panel == -1
    assert tc.sum() == info["tc_nnz"] > 0
    # every tensor-core nonzero lies in a 16x16 tile with >= 128 nonzeros of W
    dense = np.zeros((13, 19), np.int64)
    np.add.at(dense, (ref_rows // 16, w.col_idx // 16), 1)
    assert np.all(dense[d.row[tc] // 16, d.col[tc] // 16] >= 128)
    assert np.all(dense[d.row[~tc] // 16, d.col[~tc] // 16] < 128)
    # off switches, fp32 and uniform 90% sparsity never take the path
    assert _plan(w, torch.float16, n_hint=512, tc_min_density=-1).info["tc_tiles"] == 0
    assert _plan(w, torch.float32, n_hint=512).info["tc_tiles"] == 0
    assert _plan(gen.pruned_weights(512, 512, 90, seed=1), torch.float16, n_hint=512).info["tc_tiles"] == 0


def test_spec_partition_examples():
    g = golden("spec_partition.json")
    # 4x4 example, 2 blocks -> balanced 2 / 2 (membership may differ: LPT)
    gcsr = golden("spec_csr4x4.json")
    w = gen.Csr(4, 4, np.array(gcsr["row_ptr"], np.int32), np.array(gcsr["col_idx"], np.int32),
                np.array(gcsr["values"], np.float32))
    pl = _plan(w, warps=2, rows_per_warp=1, split_k=1)
    assert pl.info["panels"] == g["m_blocks"]
    exp_nnz = sorted(sum(g["row_nnz"][a:b]) for a, b in g["ranges"])
    assert [pl.info["min_panel_nnz"], pl.info["max_panel_nnz"]] == exp_nnz
    # block_nnz = 5 over gy = 4 -> [2, 2, 1, 0]
    w5 = gen.Csr(1, 16, np.array([0, 5], np.int32), np.array([1, 3, 4, 9, 12], np.int32),
                 np.ones(5, np.float32))
    d = _plan(w5, split_k=4, warps=1, rows_per_warp=1).dump()
    sizes = [int((d.group == k).sum()) for k in range(4)]
    assert sizes == g["group_split_sizes"]


def test_paper_tiling_example_arithmetic():
    # M=256, K=3056, N=512, M_blocks=8, N_blocks=16, Gy=16 -> 32x32 tiles, 191 K/group
    g = golden("paper_tiling_example.json")
    assert g["M"] // g["M_blocks"] == g["tile_m"] and g["N"] // g["N_blocks"] == g["tile_n"]
    assert g["K"] // g["Gy"] == g["k_per_group"] and g["Gsy"] == g["N"] // g["N_blocks"]
    # our plan for the same M, K with Mp = 32 rows per panel reproduces M_blocks = 8
    w = gen.pruned_weights(g["M"], g["K"], 90, seed=1)
    pl = _plan(w, warps=4, rows_per_warp=8)
    assert pl.info["panels"] == g["M_blocks"]


def test_determinism_digest():
    w = gen.pruned_weights(512, 512, 90, seed=9)
    a, b = _plan(w, n_hint=256), _plan(w, n_hint=256)
    assert a.info["digest"] == b.info["digest"]
    w2 = w.with_values(w.values * 2)
    assert _plan(w2, n_hint=256).info["digest"] != a.info["digest"]


def test_conv_plan_decode():
    cin, cout = 16, 24
    w = gen.pruned_weights(cout, 9 * cin, 80, seed=4)
    for (h, wd, nb) in [(14, 14, 8), (7, 7, 4), (28, 28, 2), (56, 56, 1), (5, 9, 3)]:
        pl = _plan(w, kind=srt.SPARSE_CONV3X3, c_in=cin, h=h, w=wd, n_hint=nb, k_chunk=5)
        d = pl.dump()
        ref_rows = np.repeat(np.arange(cout), np.diff(w.row_ptr))
        assert np.array_equal(np.sort(d.row.astype(np.int64) * 9 * cin + d.col),
                              np.sort(ref_rows.astype(np.int64) * 9 * cin + w.col_idx))


@pytest.mark.parametrize("dt", [torch.float32, torch.float16, torch.bfloat16])
def test_packed_conv_plan_decode(dt):
    # interleaved conv plans (conv_kernel 4): every nonzero decodes back to its (row, ci, dy, dx)
    # with its value (copy dx, channel ci, tap row dy of the staged span)
    cin, cout = 16, 24
    w = gen.pruned_weights(cout, 9 * cin, 80, seed=4)
    for (h, wd, nb, cc) in [(14, 14, 8, 5), (28, 28, 2, 3), (7, 8, 3, 16), (4, 4, 5, 7), (10, 6, 4, 4),
                            (4, 8, 2, 9)]:
        pl = _plan(w, dtype=dt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=h, w=wd, n_hint=nb, k_chunk=cc,
                   conv_kernel=4)
        assert pl.info["conv_kernel"] == 4
        d = pl.dump()
        dense = np.zeros((cout, 9 * cin))
        dense[d.row, d.col] = d.value
        ref = torch.from_numpy(gen.to_dense(w, np.float32)).to(dt).double().numpy()
        assert np.array_equal(dense, ref)
    with pytest.raises(S.SparseRTError):  # rows_per_warp > 8
        _plan(w, kind=srt.SPARSE_CONV3X3, c_in=cin, h=7, w=7, n_hint=2, conv_kernel=4, rows_per_warp=16)
    with pytest.raises(S.SparseRTError):  # 56-wide images: the tile's span exceeds one TMA box
        _plan(w, kind=srt.SPARSE_CONV3X3, c_in=cin, h=56, w=56, n_hint=2, conv_kernel=4)


def _rc(fn):
    with pytest.raises(S.SparseRTError) as ei:
        fn()
    return ei.value.code, ei.value.msg


def test_validation_errors():
    ok_rp = np.array([0, 2, 3], np.int32)
    ok_ci = np.array([0, 2, 1], np.int32)
    ok_v = np.array([1.0, 2.0, 3.0], np.float32)
    mk = lambda rp=ok_rp, ci=ok_ci, v=ok_v, M=2, K=4, dt=srt.SPARSE_F32, **kw: \
        S.sparse_plan_create(M, K, rp, ci, v, dt, **HOST, **kw)
    h = mk()
    S.plan_destroy(h)
    assert _rc(lambda: mk(rp=np.array([0, 3, 2], np.int32)))[0] == S.SPARSE_EMATRIX
    code, msg = _rc(lambda: mk(ci=np.array([0, 4, 1], np.int32)))
    assert code == S.SPARSE_EMATRIX and "row 0" in msg
    assert _rc(lambda: mk(ci=np.array([2, 0, 1], np.int32)))[0] == S.SPARSE_EMATRIX
    assert _rc(lambda: mk(ci=np.array([1, 1, 1], np.int32)))[0] == S.SPARSE_EMATRIX
    code, msg = _rc(lambda: mk(v=np.array([1.0, 2.0, np.nan], np.float32)))
    assert code == S.SPARSE_EMATRIX and "row 1" in msg
    assert _rc(lambda: mk(v=np.array([1.0, 0.0, 3.0], np.float32)))[0] == S.SPARSE_EMATRIX
    h = mk(v=np.array([1.0, 0.0, 3.0], np.float32), drop_zeros=1)
    assert S.sparse_plan_info(h)["nnz"] == 2
    S.plan_destroy(h)
    assert _rc(lambda: mk(v=np.array([1.0, 7e4, 3.0], np.float32), dt=srt.SPARSE_F16))[0] == S.SPARSE_EMATRIX
    assert _rc(lambda: mk(M=0))[0] == S.SPARSE_EINVAL
    assert _rc(lambda: mk(dt=7))[0] == S.SPARSE_EINVAL
    assert _rc(lambda: S.sparse_plan_create(1, 70000, [0, 0], [], [], 0, **HOST))[0] == S.SPARSE_EUNSUPPORTED
    assert _rc(lambda: mk(kind=srt.SPARSE_CONV3X3, c_in=1, h=3, w=3))[0] == S.SPARSE_EUNSUPPORTED
    assert _rc(lambda: mk(rows_per_warp=3))[0] == S.SPARSE_EUNSUPPORTED
    assert _rc(lambda: mk(x_multicast=3))[0] == S.SPARSE_EUNSUPPORTED
    assert _rc(lambda: mk(x_multicast=2, k_split=2, K=256))[0] == S.SPARSE_EUNSUPPORTED
    assert _rc(lambda: mk(warps=17))[0] == S.SPARSE_EUNSUPPORTED
    assert _rc(lambda: mk(stages=9))[0] == S.SPARSE_EUNSUPPORTED
    # compute calls on a host-only plan are rejected (never computed on the CPU)
    h = mk()
    assert S.lib.sparse_spmm(h, 4, ctypes.c_void_p(16), 4, ctypes.c_void_p(16), 4, None) == S.SPARSE_EINVAL
    assert S.lib.sparse_conv3x3(h, 1, ctypes.c_void_p(16), ctypes.c_void_p(16), None) == S.SPARSE_EINVAL
    assert S.lib.sparse_spmm(None, 4, None, 4, None, 4, None) == S.SPARSE_EINVAL
    assert S.lib.sparse_spmm(h, 0, None, 0, None, 0, None) == S.SPARSE_EINVAL  # host-only first
    S.plan_destroy(h)
    assert S.lib.plan_destroy(None) == S.SPARSE_OK


def test_fp16_rounding_matches_ieee():
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.standard_normal(2000).astype(np.float32) * 10.0 ** rng.integers(-7, 5, 2000),
                        np.array([65504.0, 65519.0, -65519.0, 6.0e-8, 2.0 ** -24, 3 * 2.0 ** -25,
                                  1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11], np.float32)])
    v = v[(v.astype(np.float16) != 0)]
    M = v.size
    w = gen.Csr(M, 1, np.arange(M + 1, dtype=np.int32), np.zeros(M, np.int32), v.astype(np.float32))
    import torch
    d = _plan(w, torch.float16).dump()
    got = np.empty(M, np.float32)
    got[d.row] = d.value
    assert np.array_equal(got, v.astype(np.float16).astype(np.float32))


def test_jit_codegen_compiles_on_host():
    # the JIT executor generates PTX per row panel and assembles it in-process;
    # both steps run without a GPU
    import torch
    w = gen.pruned_weights(200, 96, 90, seed=3)
    pl = _plan(w, n_hint=300, executor=1)
    i = pl.info
    assert i["executor"] == 1 and i["jit_modules"] >= 1 and i["jit_cubin_bytes"] > 0
    pl16 = _plan(w, torch.float16, n_hint=300, executor=1)
    assert pl16.info["jit_cubin_bytes"] > 0
    with pytest.raises(S.SparseRTError):
        _plan(w, kind=srt.SPARSE_CONV3X3, c_in=w.K // 9, h=4, w=4, executor=1)


@pytest.mark.parametrize("M,K,p", [(64, 64, 90), (300, 200, 90), (77, 1111, 80), (512, 512, 98), (33, 70, 50)])
def test_tensor_core_panel_steps(M, K, p):
    # executor 3 (condensed panels): per 16-row panel and 64-row K chunk the union's rows are
    # laid out in 8-row halves with pairwise distinct k mod 8, two halves per k16 step, so a
    # panel-chunk takes ceil(max_r |{k in union : k mod 8 = r}| / 2) steps.  Independent count:
    import torch
    w = gen.pruned_weights(M, K, p, seed=M + K)
    info = _plan(w, torch.float16, n_hint=256, executor=3).info
    assert info["executor"] == 3
    rows = np.repeat(np.arange(M), np.diff(w.row_ptr))
    expect = 0
    for q in range((M + 15) // 16):
        for c in range((K + 63) // 64):
            sel = (rows // 16 == q) & (w.col_idx // 64 == c)
            union = np.unique(w.col_idx[sel] - 64 * c)
            if union.size == 0:
                continue
            halves = np.bincount(union % 8, minlength=8).max()
            expect += (halves + 1) // 2
    assert info["tc_panel_steps"] == expect
    # fp32 plans and conv plans do not take it
    with pytest.raises(srt.SparseRTError):
        _plan(w, torch.float32, n_hint=256, executor=3)


@pytest.mark.parametrize("dt", ["f16", "f32"])
@pytest.mark.parametrize("M,K,p", [(300, 200, 90), (512, 512, 98), (768, 3072, 99), (130, 64, 95)])
@pytest.mark.parametrize("pair", [0, 1])
def test_tcgen05_block_list(M, K, p, dt, pair):
    # executor 4: the inspector keeps every (128-row block, BK-column block) holding a nonzero,
    # BK = 64 (16-bit) / 32 (fp32, 3xTF32); a CTA pair (two row blocks) walks the union of its
    # two blocks' k-block lists.  Independent count of the union entries:
    import torch
    w = gen.pruned_weights(M, K, p, seed=M * 3 + K)
    tdt = torch.float16 if dt == "f16" else torch.float32
    info = _plan(w, tdt, n_hint=512, executor=4, cta_pair=pair).info
    assert info["executor"] == 4 and info["cta_pair"] == pair
    assert info["x_multicast"] == (2 if pair else 1)
    bk = 64 if dt == "f16" else 32
    rows = np.repeat(np.arange(M), np.diff(w.row_ptr))
    grp = (rows // 128) // (2 if pair else 1)
    keys = np.unique(grp.astype(np.int64) * 100000 + w.col_idx // bk)
    assert info["tc_panel_steps"] == keys.size


@pytest.mark.parametrize("dt", ["f16", "f32"])
def test_tcgen05_conv_block_list(dt):
    # conv_kernel 5: k-blocks are (BK input channels, tap); K index k = ci * 9 + tap
    import torch
    cin, cout = 96, 200
    w = gen.pruned_weights(cout, 9 * cin, 95, seed=5)
    tdt = torch.float16 if dt == "f16" else torch.float32
    info = _plan(w, tdt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=14, w=14, n_hint=8, conv_kernel=5, cta_pair=1).info
    assert info["conv_kernel"] == 5 and info["cta_pair"] == 1
    bk = 64 if dt == "f16" else 32
    rows = np.repeat(np.arange(cout), np.diff(w.row_ptr))
    kb = (w.col_idx // 9) // bk * 9 + w.col_idx % 9
    keys = np.unique(((rows // 128) // 2).astype(np.int64) * 100000 + kb)
    assert info["tc_panel_steps"] == keys.size


def test_cta_pair_validation():
    w = gen.pruned_weights(256, 128, 90, seed=1)
    import torch
    with pytest.raises(srt.SparseRTError):   # CTA pairs are a tcgen05 block executor option
        _plan(w, torch.float16, n_hint=256, executor=0, cta_pair=1)
    with pytest.raises(srt.SparseRTError):   # the pair is the cluster
        _plan(w, torch.float16, n_hint=256, executor=4, cta_pair=1, x_multicast=4)
    with pytest.raises(srt.SparseRTError):
        _plan(w, torch.float16, n_hint=256, executor=4, cta_pair=2)
    a = _plan(w, torch.float16, n_hint=256, executor=4, cta_pair=1).info
    b = _plan(w, torch.float16, n_hint=256, executor=4, x_multicast=2).info
    assert a["digest"] != b["digest"]  # same blocks, different executor geometry


def test_tcgen05_kslices_option():
    # k_split on the tcgen05 block executor: 1, 2, 4, 8 or 16 K slices per tile (SpMM only)
    import torch
    w = gen.pruned_weights(256, 1024, 90, seed=2)
    info = _plan(w, torch.float16, n_hint=392, executor=4, k_split=16).info
    assert info["executor"] == 4 and info["k_split"] == 16
    with pytest.raises(srt.SparseRTError):
        _plan(w, torch.float16, n_hint=392, executor=4, k_split=3)
    with pytest.raises(srt.SparseRTError):   # the CUDA-core executor's cluster K split stops at 8
        _plan(w, torch.float16, n_hint=392, executor=0, k_split=16)
    a = _plan(w, torch.float16, n_hint=392, executor=4, k_split=4).info
    b = _plan(w, torch.float16, n_hint=392, executor=4, k_split=8).info
    assert a["digest"] != b["digest"]
