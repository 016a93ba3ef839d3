"""Create one plan and launch it a few times (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2008_11849_b200 as srt  # noqa: E402
from synth import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=256)
ap.add_argument("--K", type=int, default=64)
ap.add_argument("--N", type=int, default=1568)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--opts", default="")
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
opts = dict((k, int(v)) for k, v in (kv.split("=") for kv in a.opts.split(",") if kv))
tdt = torch.float16 if a.dtype == "f16" else torch.float32
w = gen.pruned_weights(a.M, a.K, 90, seed=1)
p = srt.Plan.from_csr(w, dtype=tdt, n_hint=a.N, **opts)
x = torch.from_numpy(gen.uniform_x(a.K, a.N, seed=2)).cuda().to(tdt)
for _ in range(a.reps):
    p.spmm(x)
torch.cuda.synchronize()
print(p.info)
