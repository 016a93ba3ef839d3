"""Run every tuner-grid tile configuration of one SpMM shape on integer data and check it
bitwise against the exact product (debug aid: prints each config before running it).

    python scripts/cfg_sweep.py M K N [f16]
"""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11849_b200 as srt  # noqa: E402
from synth import gen  # noqa: E402

M, K, N = map(int, sys.argv[1:4])
f16 = "f16" in sys.argv[4:]
reps = int(os.environ.get("REPS", "1"))
seed = int(os.environ.get("SEED", "1"))
dt = torch.float16 if f16 else torch.float32
w = gen.int_weights(M, K, 90, seed=seed, vmax=2 if f16 else 3)
X = np.random.default_rng(0).integers(-3, 4, (K, N)).astype(np.float32)
ref = gen.to_dense(w, np.float64) @ X.astype(np.float64)
if f16:
    ref = ref.astype(np.float16).astype(np.float64)
Xd = torch.from_numpy(X).cuda().to(dt)
bad = 0
for wp, R, kc, ks, gk, cm in itertools.product([8, 16], [2, 4, 8], [64, 128], [1, 2, 4], [1, 2, 4], [1, 2, 4, 8]):
    if ks > 1 and cm > 1:
        continue
    cfg = dict(warps=wp, rows_per_warp=R, k_chunk=kc, k_split=ks, split_k=gk, x_multicast=cm)
    try:
        p = srt.Plan.from_csr(w, dtype=dt, n_hint=N, **cfg)
    except srt.SparseRTError as e:
        continue
    print(cfg, p.info["stages"], p.info["smem_bytes"] if "smem_bytes" in p.info else "", flush=True)
    Y = torch.full((M, N), float("nan"), dtype=dt, device="cuda")
    for _ in range(reps):
        p.spmm(Xd, Y)
    torch.cuda.synchronize()
    y = Y.double().cpu().numpy()
    if not np.array_equal(y, ref):
        bad += 1
        print("  MISMATCH", np.abs(y - ref).max(), flush=True)
print("bad", bad)
