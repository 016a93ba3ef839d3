"""rel-L2 of the 3xTF32 tcgen05 executor (executor 4, fp32 plans) against a float64 product, as
a function of K (accumulation chain length), next to the CUDA-core fp32 executor.
    python scripts/tf32_err.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11849_b200 as srt
from synth import gen

dev = torch.device("cuda:0")
M, N = 768, 2048
for K in (256, 768, 1536, 3072, 6144):
    for p in (90, 50):
        w = gen.pruned_weights(M, K, p, seed=K + p)
        x = gen.uniform_x(K, N, seed=K + 1)
        Wd = torch.from_numpy(gen.to_dense(w)).to(dev)
        X = torch.from_numpy(x).to(dev)
        ref = Wd @ X.double()
        out = {}
        for name, kw in (("cuda-core", dict()), ("3xTF32", dict(executor=4)), ("3xTF32 cs2", dict(executor=4, x_multicast=2))):
            plan = srt.Plan.from_csr(w, dtype=torch.float32, n_hint=N, **kw)
            Y = plan.spmm(X)
            torch.cuda.synchronize()
            out[name] = float(torch.linalg.norm(Y.double() - ref) / torch.linalg.norm(ref))
        print(f"K={K:5d} p={p}: " + "  ".join(f"{k} {v:.3e}" for k, v in out.items()), flush=True)
