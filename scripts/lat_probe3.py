"""Fixed cost vs per-tile cost: warm graph-replayed time of one SpMM shape as N grows in whole
waves of N tiles (1 panel x t tiles per CTA), for an empty W (pure X streaming + Y stores) and
the 90%-sparse W.   python scripts/lat_probe3.py"""
import sys, torch
sys.path.insert(0, '.')
import paper_2008_11849_b200 as srt
from synth import gen
dev = torch.device("cuda:0")
def t_graph(fn, reps=50):
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for _ in range(reps): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
import os
CFG = eval(os.environ.get('LAT_CFG', '[(64, 256, 4, 128, 2), (64, 256, 4, 64, 4), (64, 1024, 4, 128, 2), (256, 256, 16, 128, 2)]'))
for (M, K, R, kc, st) in CFG:
    if R == 16:
        R, w_ = 4, 16
    else:
        w_ = 16
    w = gen.pruned_weights(M, K, 90, seed=1)
    e = gen.stress_pattern("empty", M, K, seed=1)
    for t in eval(os.environ.get('LAT_T', '(0.25, 0.5, 1, 2, 3, 4, 6)')):
        N = int(128 * 148 * t)
        X = torch.rand(K, N, device=dev); Y = torch.empty(M, N, device=dev)
        out = []
        for ww in (e, w):
            p = srt.Plan.from_csr(ww, dtype=torch.float32, n_hint=N, warps=w_, rows_per_warp=R, k_chunk=kc, stages=st)
            out.append(round(t_graph(lambda: p.spmm(X, Y)), 2))
        mb = (K + M) * N * 4 / 1e6
        print(f"M{M} K{K} R{R} kc{kc} st{st} tiles/CTA {t:5} N {N:6d}  empty {out[0]:7.2f} us  real {out[1]:7.2f} us   X+Y {mb:6.1f} MB -> {mb/out[0]:5.2f} TB/s empty", flush=True)
