"""Tensor-core sub-block path vs CUDA cores only, on block-structured W (16x16 dense tiles
on a 5% background), fp16, warm graph replay.  python scripts/tc_probe.py"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11849_b200 as srt
from synth import gen


def t_graph(fn, reps=20):
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for _ in range(reps): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for (M, K, N, dens) in [(3072, 768, 16384, 0.1), (3072, 768, 16384, 0.3), (2048, 512, 392, 0.1), (1024, 1024, 1568, 0.2)]:
    w = gen.stress_pattern("block16", M, K, seed=1, density=dens)
    X = torch.rand(K, N, device="cuda", dtype=torch.float16)
    Y = torch.empty(M, N, device="cuda", dtype=torch.float16)
    res = {}
    for label, kw in [("tc", {}), ("cuda_cores", dict(tc_min_density=-1))]:
        p = srt.Plan.from_csr(w, dtype=torch.float16, n_hint=N, **kw)
        us = t_graph(lambda: p.spmm(X, Y))
        res[label] = (round(us, 1), round(2 * w.nnz * N / us / 1e6, 1), p.info["tc_tiles"])
    Wd = torch.from_numpy(gen.to_dense(w, __import__("numpy").float32)).cuda().half()
    res["dense_fp16_cublas"] = round(t_graph(lambda: torch.matmul(Wd, X)), 1)
    print(f"{M}x{K} N={N} tiles={dens:.0%} nnz={w.nnz} ({w.nnz/(M*K):.1%}):", res, flush=True)
