"""Per-launch latency probe: event-timed single launches and graph-replayed batches of the
tiny SpMM vs an empty torch kernel."""
import sys, statistics, torch
sys.path.insert(0, '.')
import paper_2008_11849_b200 as srt
from synth import gen
dev = torch.device("cuda:0")
def t_single(fn, n=50):
    ms = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ms), min(ms)
def t_graph(fn, reps=100):
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
a = torch.zeros(16, device=dev)
print("torch add single", t_single(lambda: a.add_(1)), "graph", t_graph(lambda: a.add_(1)))
for (M, K, N, kw) in [(64, 64, 128, {}), (64, 64, 128, dict(warps=8, rows_per_warp=2, stages=2)),
                      (64, 256, 25088, {}), (2048, 512, 392, {}), (2048, 512, 392, dict(warps=8, rows_per_warp=2, k_split=1))]:
    for dt in (torch.float32,):
        w = gen.pruned_weights(M, K, 90, seed=1)
        p = srt.Plan.from_csr(w, dtype=dt, n_hint=N, **kw)
        X = torch.rand(K, N, device=dev, dtype=dt); Y = torch.empty(M, N, device=dev, dtype=dt)
        f = lambda: p.spmm(X, Y)
        print(M, K, N, kw, {k: p.info[k] for k in ("warps", "rows_per_warp", "stages", "k_split", "split_k", "k_chunk", "panels")},
              "single", t_single(f), "graph", round(t_graph(f), 2), flush=True)
