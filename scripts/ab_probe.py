"""A/B timing of library variants: for each SPARSERT_LIB in argv, graph-replayed warm timing
of fixed (shape, config) cases.  python scripts/ab_probe.py lib1.so lib2.so ..."""
import json, os, subprocess, sys
CASES = [
    ((3072, 768, 16384), "f32", dict(warps=16, rows_per_warp=8, k_chunk=56, x_source=1)),
    ((3072, 768, 16384), "f32", dict(warps=16, rows_per_warp=4, k_chunk=56, x_source=1)),
    ((3072, 768, 16384), "f32", dict(warps=8, rows_per_warp=8, k_chunk=56, x_source=1)),
    ((3072, 768, 16384), "f16", dict(warps=16, rows_per_warp=4, k_chunk=56, x_source=1)),
    ((3072, 768, 16384), "f16", dict(warps=8, rows_per_warp=8, k_chunk=56, x_source=1)),
    ((768, 3072, 16384), "f16", dict(warps=16, rows_per_warp=4, k_chunk=56, x_source=1)),
    ((2048, 512, 392), "f32", dict(warps=16, rows_per_warp=4, k_chunk=56, x_source=1)),
    ((3072, 768, 16384), "f32", dict(warps=16, rows_per_warp=8, k_chunk=128, stages=2)),
    ((3072, 768, 16384), "f32", dict(warps=8, rows_per_warp=8, k_chunk=64, stages=3)),
    ((3072, 768, 16384), "f16", dict(warps=16, rows_per_warp=4, k_chunk=128, stages=2)),
    ((3072, 768, 16384), "f16", dict(warps=8, rows_per_warp=8, k_chunk=128, stages=2)),
    ((2048, 512, 392), "f32", dict(warps=16, rows_per_warp=4, k_chunk=64, stages=4)),
    ((512, 2048, 392), "f32", dict(warps=16, rows_per_warp=4, k_chunk=128, k_split=4)),
    ((64, 256, 25088), "f32", dict(warps=16, rows_per_warp=4, k_chunk=64, stages=4)),
]
CHILD = r'''
import json, sys, torch
sys.path.insert(0, ".")
import paper_2008_11849_b200 as srt
from synth import gen
cases = json.loads(sys.argv[1])
out = []
for (M, K, N), dt, kw in cases:
    tdt = torch.float16 if dt == "f16" else torch.float32
    w = gen.pruned_weights(M, K, 90, seed=1)
    try:
        p = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, **kw)
    except Exception as e:
        out.append(dict(us=float("nan"), tflops=str(e)[:40])); continue
    X = torch.rand(K, N, device="cuda", dtype=tdt); Y = torch.empty(M, N, device="cuda", dtype=tdt)
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); reps = 20
    with torch.cuda.stream(s):
        p.spmm(X, Y); torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for _ in range(reps): p.spmm(X, Y)
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    us = sorted(ts)[1]
    out.append(dict(shape=[M, K, N], dt=dt, cfg=kw, us=round(us, 2), tflops=round(2 * w.nnz * N / us / 1e6, 2)))
print(json.dumps(out))
'''
# optional first argument: a JSON file of cases [[[M, K, N], "f32", {opts}], ...]
if sys.argv[1].endswith(".json"):
    CASES = [(tuple(c[0]), c[1], c[2]) for c in json.load(open(sys.argv.pop(1)))]
res = {}
for lib in sys.argv[1:]:
    env = dict(os.environ, SPARSERT_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(CASES)], env=env, capture_output=True, text=True)
    if r.returncode:
        print(lib, "FAILED", r.stderr[-500:]); continue
    res[lib] = json.loads(r.stdout.strip().splitlines()[-1])
libs = list(res)
for i, (shape, dt, cfg) in enumerate(CASES):
    print(shape, dt, cfg, " | ".join(f"{os.path.basename(l)}: {res[l][i]['us']} us {res[l][i]['tflops']} TF" for l in libs))
