import os, sys, itertools, numpy as np, torch
sys.path.insert(0, '.')
import paper_2008_11849_b200 as srt
from synth import gen
M, K, N = 2048, 512, 392
w = gen.int_weights(M, K, 90, seed=M + N, vmax=3)
X = torch.rand(K, N, device="cuda") * 2 - 1
Y = torch.empty(M, N, device="cuda")
st = torch.cuda.Stream()
only = os.environ.get("ONLY")
reps = int(os.environ.get("REPS", "17"))
for wp, R, kc, ks, gk in itertools.product([8, 16], [2, 4], [64, 128], [1, 2, 4, 8], [1, 2]):
    cfg = dict(warps=wp, rows_per_warp=R, k_chunk=kc, k_split=ks, split_k=gk)
    if only and only != f"{wp},{R},{kc},{ks},{gk}":
        continue
    p = srt.Plan.from_csr(w, dtype=torch.float32, n_hint=N, **cfg)
    with torch.cuda.stream(st):
        for _ in range(reps):
            p.spmm(X, Y)
    try:
        st.synchronize()
    except Exception as e:
        print("FAIL", cfg, p.info["stages"], e, flush=True)
        sys.exit(1)
    print("ok", cfg, p.info["stages"], flush=True)
