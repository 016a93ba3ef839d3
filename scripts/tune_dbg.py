import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2008_11849_b200 as srt
from synth import gen
M, K, N = 2048, 512, 392
for it in range(6):
    w = gen.int_weights(M, K, 90, seed=M + N, vmax=3)
    p = srt.Plan.from_csr(w, dtype=torch.float32, n_hint=N, tune=1)
    print("chosen", p.chosen_opts(), p.info["tuned_us"], flush=True)
    x = torch.ones(4, device="cuda"); torch.cuda.synchronize()
    print("ok", it, flush=True)
