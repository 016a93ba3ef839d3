"""Ablation of the plan source (the paper keeps A's values in the constant cache):
the plan-driven executor with its plan blocks staged into shared memory with every X chunk
(plan_source 0) vs the whole plan passed as a kernel parameter and read through the constant
cache (plan_source 1, plans <= 30 KB), on the small-plan layer shapes, same tile options (the
tuned staged configuration), cold L2 and warm.  JSON lines to --out.

    python scripts/plan_source_ablation.py --out gpurun_out/plan_source.jsonl
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import paper_2008_11849_b200 as srt  # noqa: E402
from synth import gen  # noqa: E402
from measure_table import Timer  # noqa: E402

SHAPES = [("tiny", 64, 64, 128), ("rn50_p1_b1", 64, 256, 3136), ("rn50_p1_b8", 64, 256, 25088),
          ("rn50_p2_b1", 256, 64, 3136), ("rn50_p2_b8", 256, 64, 25088), ("mbv1_p12_b1", 64, 32, 12544),
          ("mbv1_p12_b32", 64, 32, 401408), ("mbv1_p13_b1", 128, 64, 3136), ("mbv1_p13_b32", 128, 64, 100352),
          ("mbv1_p14_b8", 128, 128, 25088), ("effb0_96x16_b8", 96, 16, 100352), ("effb0_144x24_b8", 144, 24, 25088)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtypes", default="f32,f16")
    ap.add_argument("--sparsity", type=int, default=90)
    ap.add_argument("--out", default="gpurun_out/plan_source.jsonl")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    timer = Timer(dev)
    with open(args.out, "a") as f:
        for name, M, K, N in SHAPES:
            for dt in args.dtypes.split(","):
                tdt = torch.float16 if dt == "f16" else torch.float32
                w = gen.pruned_weights(M, K, args.sparsity, seed=gen.case_seed(name, args.sparsity))
                x = torch.from_numpy(gen.uniform_x(K, N, 3)).to(dev).to(tdt)
                y = torch.empty((M, N), dtype=tdt, device=dev)
                t = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, tune=1, executor=0, tc_min_density=-1)
                o = t.chosen_opts()
                t.close()
                o.update(split_k=1, k_split=1, x_multicast=1, x_source=0, executor=0, tc_min_density=-1)
                row = dict(name=name, dtype=dt, M=M, K=K, N=N, opts=o)
                for ps in (0, 1):
                    try:
                        p = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, plan_source=ps, **o)
                    except srt.SparseRTError as e:
                        row[f"ps{ps}"] = str(e)[:120]
                        continue
                    row[f"ps{ps}_cold_us"] = timer.cold(lambda: p.spmm(x, y))
                    row[f"ps{ps}_warm_us"] = timer.warm(lambda: p.spmm(x, y))
                    row["plan_bytes"] = p.info["plan_bytes"]
                    p.close()
                f.write(json.dumps(row) + "\n")
                f.flush()
                print(json.dumps(row), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
