"""Tile-parameter sweep for one layer shape (the paper's offline autotuning grid).

    python scripts/sweep.py --M 3072 --K 768 --N 16384 --dtype f32 \
        --grid "rows_per_warp=4,8;stages=2,3;warps=4,8"

Every candidate is timed with CUDA events (median of --reps launches, L2 flushed before each)
and checked bitwise against the first candidate on integer data where the summation order
allows (candidates that only change the schedule, not k_chunk/split_k/k_split).
"""
import argparse
import itertools
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_11849_b200 as srt  # noqa: E402
from synth import gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, required=True)
    ap.add_argument("--K", type=int, required=True)
    ap.add_argument("--N", type=int, required=True)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--sparsity", type=int, default=90)
    ap.add_argument("--grid", default="")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--conv", default="", help="c_in,h,w,batch for a conv layer")
    ap.add_argument("--flush", default="write", choices=["none", "write", "writeread", "b2b"])
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    tdt = torch.float16 if args.dtype == "f16" else torch.float32
    axes = []
    for part in filter(None, args.grid.split(";")):
        k, vs = part.split("=")
        axes.append([(k, int(v)) for v in vs.split(",")])
    combos = [dict(c) for c in itertools.product(*axes)] if axes else [{}]
    w = gen.pruned_weights(args.M, args.K, args.sparsity, seed=1)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    if args.conv:
        cin, h, wd, b = map(int, args.conv.split(","))
        x = torch.from_numpy(gen.relu_normal_x((cin, b, h, wd), seed=2)).to(dev, tdt)
        kind = dict(kind=srt.SPARSE_CONV3X3, c_in=cin, h=h, w=wd, n_hint=b)
        N = b * h * wd
    else:
        x = torch.from_numpy(gen.uniform_x(args.K, args.N, seed=2)).to(dev, tdt)
        kind = dict(n_hint=args.N)
        N = args.N
    flops = 2 * w.nnz * N
    for c in [{}] + combos:
        try:
            plan = srt.Plan.from_csr(w, dtype=tdt, **kind, **c)
        except srt.SparseRTError as e:
            print(json.dumps({"opts": c, "error": str(e)}))
            continue
        fn = (lambda: plan.conv3x3(x)) if args.conv else (lambda: plan.spmm(x))
        for _ in range(3):
            fn()
        ms = []
        if args.flush == "b2b":  # back-to-back launches, warm L2: intrinsic kernel duration
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.zero_()
            e0.record()
            for _ in range(args.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = [e0.elapsed_time(e1) / args.reps]
        for _ in range(args.reps if args.flush != "b2b" else 0):
            if args.flush != "none":
                flush.zero_()
            if args.flush == "writeread":
                flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = statistics.median(ms)
        i = plan.info
        print(json.dumps({"opts": c or "default", "us": round(t * 1e3, 2), "gflops": round(flops / t / 1e6, 1),
                          "R": i["rows_per_warp"], "warps": i["warps"], "ks": i["k_split"], "gk": i["split_k"],
                          "kc": i["k_chunk"], "stages": i["stages"], "smem": i["smem_bytes"]}), flush=True)


if __name__ == "__main__":
    main()
