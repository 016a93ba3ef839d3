"""Where does the time go?  Graph-replayed launches of the same shape with (a) an empty W
(pure X streaming + Y stores) and (b) the 90%-sparse W, over a few tile configurations."""
import sys, torch
sys.path.insert(0, '.')
import paper_2008_11849_b200 as srt
from synth import gen
dev = torch.device("cuda:0")
def t_graph(fn, reps=50):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for _ in range(reps): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
cfgs = [dict(warps=16, rows_per_warp=4, k_chunk=64, stages=4, x_multicast=m) for m in (1, 2, 4, 8)] + \
       [dict(warps=8, rows_per_warp=4, k_chunk=64, stages=4, x_multicast=m) for m in (1, 2, 4, 8)]
for (M, K, N) in [(64, 256, 25088), (2048, 512, 392)]:
    for dt in (torch.float32, torch.float16):
        w = gen.pruned_weights(M, K, 90, seed=1)
        e = gen.stress_pattern("empty", M, K, seed=1)
        X = torch.rand(K, N, device=dev, dtype=dt); Y = torch.empty(M, N, device=dev, dtype=dt)
        for kw in cfgs:
            out = []
            for ww in (e, w):
                try:
                    p = srt.Plan.from_csr(ww, dtype=dt, n_hint=N, **kw)
                except Exception as ex:
                    out.append(str(ex)[:30]); continue
                out.append(round(t_graph(lambda: p.spmm(X, Y)), 2))
            print(M, K, N, str(dt)[-7:], kw, "empty/real us:", out, flush=True)
