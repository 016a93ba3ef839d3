"""Warm graph-replay time of explicit tile configurations of one SpMM shape.
    python scripts/cfg_time.py M K N f32|f16 'warps=16,rows_per_warp=4;warps=8,...' """
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11849_b200 as srt
from synth import gen
M, K, N = map(int, sys.argv[1:4])
tdt = {"f16": torch.float16, "bf16": torch.bfloat16}.get(sys.argv[4], torch.float32)
w = gen.pruned_weights(M, K, 90, seed=1)
X = torch.rand(K, N, device="cuda", dtype=tdt); Y = torch.empty(M, N, device="cuda", dtype=tdt)
for cs in sys.argv[5].split(";"):
    kw = dict((k, int(v)) for k, v in (kv.split("=") for kv in cs.split(",") if kv))
    try:
        p = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, **kw)
    except Exception as e:
        print(kw, "ERR", str(e)[:60]); continue
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); reps = 30
    with torch.cuda.stream(s):
        p.spmm(X, Y); torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for _ in range(reps): p.spmm(X, Y)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    i = p.info
    print(f"{us:7.2f} us  {2*w.nnz*N/us/1e6:6.2f} TF  w{i['warps']} R{i['rows_per_warp']} kc{i['k_chunk']} st{i['stages']} gk{i['split_k']} ks{i['k_split']} panels{i['panels']} smem{i['smem_bytes']//1024}K", flush=True)
