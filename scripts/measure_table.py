"""Per-shape measurement table: for every layer
shape of the BASELINE workloads at 90 % and 95 % sparsity, fp32 and fp16, the autotuned sparse
kernel (cold-L2 and warm), the same-shape dense baselines (fp32 SGEMM with TF32 off, fp16 and
bf16 tensor cores; cuDNN conv2d for the 3x3 convs), the roofline fraction, and a bitwise
integer-data parity check of the tuned plan.  One JSON line per case is appended to --out.

    python scripts/measure_table.py --groups rn50,mbv1,effnet,bert,transformer,conv,conv_t3 \
        --sparsity 90,95 --dtypes f32,f16 --out gpurun_out/table.jsonl
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: the parity check of each tuned plan)
import paper_2008_11849_b200 as srt  # noqa: E402
from synth import gen  # noqa: E402

EFFNET = [(16, 32, 12544), (96, 16, 12544), (24, 96, 3136), (144, 24, 3136), (24, 144, 3136),
          (40, 144, 784), (240, 40, 784), (40, 240, 784), (80, 240, 196), (480, 80, 196),
          (80, 480, 196), (112, 480, 196), (672, 112, 196), (112, 672, 196), (192, 672, 49),
          (1152, 192, 49), (192, 1152, 49), (320, 1152, 49), (1280, 320, 49)]


def cases(groups):
    out = []
    for g in groups:
        if g == "rn50":
            for b in (1, 8):
                for p in gen.RN50_1X1:
                    M, K, N = gen.TABLE1[p]
                    out.append(dict(group=g, name=f"rn50_p{p}_b{b}", kind="spmm", M=M, K=K, N=N * b))
        elif g == "mbv1":
            for b in (1, 2, 4, 8, 16, 32):
                for p in gen.MBV1_PW:
                    M, K, N = gen.TABLE1[p]
                    out.append(dict(group=g, name=f"mbv1_p{p}_b{b}", kind="spmm", M=M, K=K, N=N * b))
        elif g == "effnet":
            for b in (1, 8, 32):
                for M, K, N in EFFNET:
                    out.append(dict(group=g, name=f"effb0_{M}x{K}_b{b}", kind="spmm", M=M, K=K, N=N * b))
        elif g == "bert":
            for N in (128, 512, 2048, 8192, 16384):
                for M, K in gen.BERT_FC:
                    out.append(dict(group=g, name=f"bert_{M}x{K}_N{N}", kind="spmm", M=M, K=K, N=N))
        elif g == "transformer":
            for p in (9, 10, 11):
                M, K, N = gen.TABLE1[p]
                out.append(dict(group=g, name=f"transformer_p{p}", kind="spmm", M=M, K=K, N=N))
        elif g == "conv":
            out.append(dict(group=g, name="conv_256ch_14_b256", kind="conv", C=256, H=14, B=256))
        elif g == "conv_t3":
            for t, (H, C) in gen.TABLE3.items():
                out.append(dict(group=g, name=f"conv_t3_{C}ch_{H}_b1", kind="conv", C=C, H=H, B=1))
    return out


class Timer:
    def __init__(self, dev):
        self.dev = dev
        self.flush_w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        self.flush_r = torch.zeros(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        self.sink = torch.empty(1, dtype=torch.float32, device=dev)

    def flush(self):
        self.flush_w.zero_()
        torch.sum(self.flush_r, dim=0, out=self.sink[0])

    def cold(self, fn, reps=15):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            self.flush()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts)

    def warm(self, fn, reps=20):
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(reps):
                    fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / reps


def run_case(c, sp, dt, timer, peaks, args):
    dev = timer.dev
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dt]
    S = 4 if dt == "f32" else 2
    seed = gen.case_seed(c["name"], sp)
    if c["kind"] == "spmm":
        M, K, N = c["M"], c["K"], c["N"]
        w = gen.pruned_weights(M, K, sp, seed)
        x = torch.from_numpy(gen.uniform_x(K, N, seed + 1)).to(dev).to(tdt)
        y = torch.empty((M, N), dtype=tdt, device=dev)
        base = dict(n_hint=N, executor=2)
        mk = lambda ww, **kw: srt.Plan.from_csr(ww, dtype=tdt, device=0, **{**base, **kw})  # noqa: E731
        call = lambda p: p.spmm(x, y)  # noqa: E731
        Nn, Kx = N, K
    else:
        C, H, B = c["C"], c["H"], c["B"]
        M, K = C, 9 * C
        w = gen.pruned_weights(M, K, sp, seed)
        x = torch.from_numpy(gen.relu_normal_x((C, B, H, H), seed + 1)).to(dev).to(tdt)
        y = torch.empty((M, B, H, H), dtype=tdt, device=dev)
        base = dict(kind=srt.SPARSE_CONV3X3, c_in=C, h=H, w=H, n_hint=B)
        mk = lambda ww, **kw: srt.Plan.from_csr(ww, dtype=tdt, device=0, **{**base, **kw})  # noqa: E731
        call = lambda p: p.conv3x3(x, y)  # noqa: E731
        Nn, Kx = B * H * H, C
    t0 = time.perf_counter()
    tuned = mk(w, tune=1)
    opts = tuned.chosen_opts()
    tune_s = time.perf_counter() - t0
    tuned.close()
    plan = mk(w, **opts)
    t_cold = timer.cold(lambda: call(plan))
    t_warm = timer.warm(lambda: call(plan))
    info = plan.info
    # bitwise parity of the tuned plan on integer data (sampled outputs)
    wi = gen.int_weights(M, K, sp, seed, vmax=3 if dt == "f32" else 2)
    pi = mk(wi, **opts)
    vx = 3 if dt == "f32" else 4
    if c["kind"] == "spmm":
        xi = gen.int_x(K, N, seed + 5, vmax=vx)
        yi = pi.spmm(torch.from_numpy(xi).to(dev).to(tdt))
        ids = np.unique(np.r_[0, N - 1, np.random.default_rng(seed).integers(0, N, 24)])
        ref = oracle.spmm(M, K, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), xi[:, ids].astype(np.float64))
    else:
        xi = gen.int_x(C * B * H, H, seed + 5, vmax=vx).reshape(C, B, H, H)
        yi = pi.conv3x3(torch.from_numpy(xi).to(dev).to(tdt))
        ids = np.unique(np.r_[0, B - 1])
        ref = oracle.conv3x3(M, wi.row_ptr, wi.col_idx, wi.values.astype(np.float64), xi[:, ids].astype(np.float64))
    torch.cuda.synchronize()
    ref = torch.from_numpy(ref.astype(np.float32)).to(tdt).double().numpy()
    exact = bool(np.array_equal(yi[:, torch.from_numpy(ids).to(dev)].double().cpu().numpy(), ref))
    pi.close()
    # dense baselines (W densified, zeros included), same cold-L2 protocol
    dense = {}
    Wd = torch.from_numpy(gen.to_dense(w, np.float32)).to(dev)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    for label, ddt in (("fp32_sgemm", torch.float32), ("fp16_tc", torch.float16), ("bf16_tc", torch.bfloat16)):
        Wdd = Wd.to(ddt)
        if c["kind"] == "spmm":
            xd = x.to(ddt)
            fn = lambda: torch.matmul(Wdd, xd)  # noqa: E731
        else:
            xd = x.to(ddt).permute(1, 0, 2, 3).contiguous()
            Wc = Wdd.reshape(M, c["C"], 3, 3)
            fn = lambda: F.conv2d(xd, Wc, padding=1)  # noqa: E731
        dense[label] = timer.cold(fn)
    flops = 2 * w.nnz * Nn
    alu = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6
    by = S * (Kx * Nn + M * Nn) + info["plan_bytes"]
    t_roof = max(flops / alu, by / (peaks["hbm_gbs"] * 1e9))
    row = dict(group=c["group"], name=c["name"], kind=c["kind"], M=M, K=K, N=Nn, sparsity=sp, dtype=dt,
               nnz=w.nnz, us_cold=t_cold, us_warm=t_warm, gflops_cold=flops / t_cold / 1e3,
               roof_us=t_roof * 1e6, roof_frac=t_roof * 1e6 / t_cold,
               bound="alu" if flops / alu >= by / (peaks["hbm_gbs"] * 1e9) else "hbm",
               dense_us=dense, speedup={k: v / t_cold for k, v in dense.items()},
               executor=info["executor"], conv_kernel=info.get("conv_kernel"), opts=opts,
               tune_s=round(tune_s, 2), exact=exact)
    plan.close()
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", default="rn50,mbv1,bert,transformer,conv,conv_t3,effnet")
    ap.add_argument("--sparsity", default="90,95")
    ap.add_argument("--dtypes", default="f32,f16")
    ap.add_argument("--out", default="gpurun_out/table.jsonl")
    ap.add_argument("--budget-s", type=float, default=3000.0)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    timer = Timer(dev)
    d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peaks = dict(hbm_gbs=float(d.get("hbm_gbs", 6650.0)), sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)))
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    t_start = time.time()
    with open(args.out, "a") as f:
        for c in cases(args.groups.split(",")):
            for sp in map(int, args.sparsity.split(",")):
                for dt in args.dtypes.split(","):
                    if time.time() - t_start > args.budget_s:
                        print("budget exhausted", flush=True)
                        return 0
                    try:
                        row = run_case(c, sp, dt, timer, peaks, args)
                    except Exception as e:  # record and keep going
                        row = dict(group=c["group"], name=c["name"], sparsity=sp, dtype=dt, error=str(e)[:200])
                    f.write(json.dumps(row) + "\n")
                    f.flush()
                    print(json.dumps({k: row.get(k) for k in ("name", "sparsity", "dtype", "us_cold", "roof_frac",
                                                               "speedup", "exact", "error")}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
