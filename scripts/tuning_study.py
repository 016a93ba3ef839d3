"""Per-instance vs per-shape autotuning and the instance variance of E12
(P:304): for each shape, `--instances` differently-seeded magnitude-pruned W of the same
shape and sparsity (different sparsity patterns, like reused layers of one network):
  * heuristic: the inspector's default tile choice (no timing);
  * per-instance: tune=1 on every instance (< 100 timed candidates each);
  * per-shape: the options tuned on instance 0 applied to every other instance.
Cold-L2 median of 15 launches per instance and mode; JSON lines to --out.

    python scripts/tuning_study.py --out gpurun_out/tuning_study.jsonl
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import paper_2008_11849_b200 as srt  # noqa: E402
from synth import gen  # noqa: E402
from measure_table import Timer  # noqa: E402

SHAPES = [("rn50_p3_b8", "spmm", 128, 512, 784 * 8), ("rn50_p8_b8", "spmm", 2048, 512, 49 * 8),
          ("transformer_p11", "spmm", 512, 512, 256), ("mbv1_p20_b32", "spmm", 1024, 1024, 49 * 32),
          ("bert_3072x768_N2048", "spmm", 3072, 768, 2048), ("conv_128ch_28_b8", "conv", 128, 9 * 128, 8)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=5)
    ap.add_argument("--dtypes", default="f32,f16")
    ap.add_argument("--sparsity", type=int, default=90)
    ap.add_argument("--out", default="gpurun_out/tuning_study.jsonl")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    timer = Timer(dev)
    with open(args.out, "a") as f:
        for name, kind, M, K, N in SHAPES:
            for dt in args.dtypes.split(","):
                tdt = torch.float16 if dt == "f16" else torch.float32
                if kind == "spmm":
                    x = torch.from_numpy(gen.uniform_x(K, N, 7)).to(dev).to(tdt)
                    y = torch.empty((M, N), dtype=tdt, device=dev)
                    base = dict(n_hint=N, executor=2)
                    run = lambda p: p.spmm(x, y)  # noqa: E731
                else:
                    C, H, B = M, 28, N
                    x = torch.from_numpy(gen.relu_normal_x((C, B, H, H), 7)).to(dev).to(tdt)
                    y = torch.empty((M, B, H, H), dtype=tdt, device=dev)
                    base = dict(kind=srt.SPARSE_CONV3X3, c_in=C, h=H, w=H, n_hint=B)
                    run = lambda p: p.conv3x3(x, y)  # noqa: E731
                ws = [gen.pruned_weights(M, K, args.sparsity, seed=gen.case_seed(name, 1000 + i))
                      for i in range(args.instances)]
                res = {"heuristic": [], "per_instance": [], "per_shape": []}
                opts_i = []
                shape_opts = None
                for i, w in enumerate(ws):
                    p = srt.Plan.from_csr(w, dtype=tdt, **base)
                    res["heuristic"].append(timer.cold(lambda: run(p)))
                    p.close()
                    t = srt.Plan.from_csr(w, dtype=tdt, tune=1, **base)
                    o = t.chosen_opts()
                    t.close()
                    opts_i.append(o)
                    if i == 0:
                        shape_opts = o
                    p = srt.Plan.from_csr(w, dtype=tdt, **{**base, **o})
                    res["per_instance"].append(timer.cold(lambda: run(p)))
                    p.close()
                    p = srt.Plan.from_csr(w, dtype=tdt, **{**base, **shape_opts})
                    res["per_shape"].append(timer.cold(lambda: run(p)))
                    p.close()
                row = dict(name=name, dtype=dt, sparsity=args.sparsity, M=M, K=K, N=N, instances=args.instances,
                           us=res, mean={k: statistics.mean(v) for k, v in res.items()},
                           cv={k: statistics.pstdev(v) / statistics.mean(v) for k, v in res.items()},
                           per_shape_over_per_instance=statistics.mean(res["per_shape"]) / statistics.mean(res["per_instance"]),
                           heuristic_over_per_instance=statistics.mean(res["heuristic"]) / statistics.mean(res["per_instance"]),
                           distinct_tuned_configs=len({json.dumps(o, sort_keys=True) for o in opts_i}),
                           shape_opts=shape_opts)
                f.write(json.dumps(row) + "\n")
                f.flush()
                print(json.dumps({k: row[k] for k in ("name", "dtype", "mean", "cv", "per_shape_over_per_instance",
                                                      "heuristic_over_per_instance", "distinct_tuned_configs")}),
                      flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
