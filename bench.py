#!/usr/bin/env python
"""Benchmark of the B200 SparseRT hot path (effective GFLOP/s = 2*nnz*N / t).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload rn50_b8] [--dtype f32]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...     # the CPU oracle arm (rank 0 only)

A "step" is one pass of the executor over one batch of synthetic input for every layer of
the workload (the plans are built once, offline, like the paper's inspector; their
build time is reported in config.plan_build_ms).  Default workload (BASELINE.json
configs[1]): the eight ResNet-50 1x1 layers of PAPER.md Table 1, 90% sparsity,
batch 8 per GPU, fp32 (the paper's precision).  L2 is flushed (256 MiB write + 256 MiB read)
before every timed step, outside the timed events, so every layer reads cold HBM.

Multi-GPU: one process per GPU, each with a replicated plan and its own batch (weak
scaling for the layer workloads: no collective on the data path); the conv workload
(configs[4]) shards the fixed batch of 256 images over ranks (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import gen  # noqa: E402

METRIC = "effective GFLOP/s (2·nnz·N) and speedup vs dense GEMM at 90/95% sparsity"


# ----------------------------------------------------------------------------- workloads

def workload_layers(name: str, sparsity: int, world: int):
    """Returns (layers, scaling, description).  layer = dict(kind, M, K, N | conv geometry)."""
    if name in ("rn50_b8", "rn50_b1"):
        b = 8 if name == "rn50_b8" else 1
        layers = [dict(kind="spmm", name=f"rn50_p{p}", M=gen.TABLE1[p][0], K=gen.TABLE1[p][1],
                       N=gen.TABLE1[p][2] * b) for p in gen.RN50_1X1]
        return layers, "weak", f"ResNet-50 1x1 layers (Table 1 p1-p8), batch {b} per GPU"
    if name == "mbv1_b32":
        layers = [dict(kind="spmm", name=f"mbv1_p{p}", M=gen.TABLE1[p][0], K=gen.TABLE1[p][1],
                       N=gen.TABLE1[p][2] * 32) for p in gen.MBV1_PW]
        return layers, "weak", "MobileNetV1 pointwise layers (Table 1 p12-p20), batch 32 per GPU"
    if name == "bert":
        layers = [dict(kind="spmm", name=f"bert_{M}x{K}", M=M, K=K, N=32 * 512) for M, K in gen.BERT_FC]
        return layers, "weak", "BERT-base FFN layers, N = 32 x 512 per GPU"
    if name == "conv":
        B = 256
        if B % world:
            raise SystemExit("conv workload: world size must divide 256")
        return ([dict(kind="conv", name="rn50_conv3x3_256ch_14", M=256, K=9 * 256, c_in=256,
                      H=14, W=14, B=B // world)], "strong",
                "ResNet-50 3x3 conv 256ch 14x14, batch 256 sharded over GPUs")
    if name == "tiny":
        return [dict(kind="spmm", name="tiny", M=64, K=64, N=128)], "weak", "tiny 64x64x128"
    raise SystemExit(f"unknown workload {name}")


def layer_N(L):
    return L["N"] if L["kind"] == "spmm" else L["B"] * L["H"] * L["W"]


def make_inputs(L, sparsity, rank):
    seed = gen.case_seed(L["name"], sparsity)
    w = gen.pruned_weights(L["M"], L["K"], sparsity, seed=seed)
    if L["kind"] == "spmm":
        x = gen.uniform_x(L["K"], L["N"], seed=seed + 1 + 1000 * rank)
    else:
        x = gen.relu_normal_x((L["c_in"], L["B"], L["H"], L["W"]), seed=seed + 1 + 1000 * rank)
    return w, x


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- peaks

def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=float(d["hbm_gbs"]), sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)),
                    bf16_tflops=float(d.get("bf16_tflops", 2250.0)), source="measured")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, bf16_tflops=2250.0, source="fallback")


def alu_peak_gflops(sm_mhz: float) -> float:
    # 148 SMs x 128 FP32 lanes x 2 flop/FMA x clock
    return 148 * 128 * 2 * sm_mhz * 1e-3


# ----------------------------------------------------------------------------- reference arm

def _samples_for(layers, ins, cols):
    samples = []
    for (w, x), Lx in zip(ins, layers):
        if Lx["kind"] == "spmm":
            n = min(cols, Lx["N"])
            samples.append(("spmm", w, np.ascontiguousarray(x[:, :n]).astype(np.float64), n))
        else:
            hw = Lx["H"] * Lx["W"]
            nb = max(1, min(Lx["B"], cols // hw))
            samples.append(("conv", w, np.ascontiguousarray(x[:, :nb]).astype(np.float64), nb * hw))
    return samples


def oracle_step_sample(layers, sparsity, per_step_s: float, rank: int):
    """Bounded sample: the first n columns (whole images for conv) of every layer, n sized by
    a calibration run so that one oracle step takes about per_step_s seconds."""
    ins = [make_inputs(L, sparsity, rank) for L in layers]
    cols = 32 if layers[0]["kind"] == "spmm" else layers[0]["H"] * layers[0]["W"]
    for _ in range(4):
        samples = _samples_for(layers, ins, cols)
        t0 = time.perf_counter()
        run_oracle_step(samples)
        dt = time.perf_counter() - t0
        if dt > 0.5 * per_step_s or all(s[3] >= layer_N(L) for s, L in zip(samples, layers)):
            break
        cols = int(cols * min(64.0, max(2.0, per_step_s / max(dt, 1e-4))))
    cols = max(1, int(cols * min(1.0, per_step_s / max(dt, 1e-4))))
    return _samples_for(layers, ins, cols)


def run_oracle_step(samples):
    import oracle
    flops = 0
    for kind, w, x, n in samples:
        if kind == "spmm":
            oracle.spmm(w.M, w.K, w.row_ptr, w.col_idx, w.values.astype(np.float64), x)
        else:
            oracle.conv3x3(w.M, w.row_ptr, w.col_idx, w.values.astype(np.float64), x)
        flops += 2 * w.nnz * n
    return flops


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    layers, scaling, desc = workload_layers(args.workload, args.sparsity, 1)
    budget = float(os.environ.get("SPARSERT_REF_BUDGET_S", "120"))
    per_step = max(0.05, min(2.0, budget / max(1, args.steps + args.warmup)))
    samples = oracle_step_sample(layers, args.sparsity, per_step, rank)
    for _ in range(args.warmup):
        run_oracle_step(samples)
    t0 = time.perf_counter()
    flops = 0
    for _ in range(args.steps):
        flops += run_oracle_step(samples)
    dt = time.perf_counter() - t0
    value = flops / dt / 1e9
    cores = oracle.default_threads()
    sample_desc = "; ".join(f"{L['name']}: first {n} of {layer_N(L)} columns"
                            for L, (_, _, _, n) in zip(layers, samples))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / max(1, args.steps) * 1e3, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "description": desc, "sparsity_pct": args.sparsity,
                   "oracle": "oracle/oracle.c (dense-expanded m-k-n triple loop, double, OpenMP)"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": sample_desc},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="rn50_b8",
                    choices=["rn50_b8", "rn50_b1", "mbv1_b32", "bert", "conv", "tiny"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "f16", "bf16"])
    ap.add_argument("--sparsity", type=int, default=90)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip e2e/dense/cpu legs (for ncu runs)")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--executor", type=int, default=2, choices=[0, 1, 2],
                    help="SpMM executor: 0 plan-driven, 1 JIT code generator (the paper's method), "
                         "2 auto")
    ap.add_argument("--retune", action="store_true", help="re-run the autotuner even if "
                    "profiles/tuned_<workload>.json exists")
    ap.add_argument("--no-tune", action="store_true",
                    help="skip the offline autotuner (P:259-263); use the heuristic tile choice")
    args = ap.parse_args()
    if args.warmup < 3 and not args.quick:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist
    import paper_2008_11849_b200 as srt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16}.get(args.dtype, torch.float32)
    S = 2 if args.dtype in ("f16", "bf16") else 4

    layers, scaling, desc = workload_layers(args.workload, args.sparsity, world)
    plans, xs, ys, host = [], [], [], []
    build_ms, chosen, tuned_us = [], [], []
    tuned_path = os.path.join(ROOT, "profiles",
                              f"tuned_{args.workload}_{args.dtype}_s{args.sparsity}_x{args.executor}.json")
    saved = None
    if not args.no_tune and not args.retune and os.path.exists(tuned_path):
        saved = json.load(open(tuned_path))
    retuned = {}
    for L in layers:
        w, x = make_inputs(L, args.sparsity, rank)
        if L["kind"] == "spmm":
            base = dict(n_hint=L["N"], executor=args.executor)
        else:
            base = dict(kind=srt.SPARSE_CONV3X3, c_in=L["c_in"], h=L["H"], w=L["W"], n_hint=L["B"])
        if args.no_tune:
            p = srt.Plan.from_csr(w, dtype=tdt, device=local, **base)
        else:
            # offline autotuning: the configuration chosen by tune=1 is stored in
            # profiles/tuned_<workload>.json and reused (deterministic, same plans under ncu);
            # --retune re-runs the timed search on rank 0.  Every rank then builds the chosen
            # configuration explicitly, so the replicated plans are identical (digests).
            opts = [saved.get(L["name"]) if saved else None]
            if opts[0] is None and rank == 0:
                tuned = srt.Plan.from_csr(w, dtype=tdt, device=local, tune=1, **base)
                opts = [tuned.chosen_opts()]
                tuned_us.append(round(tuned.info["tuned_us"], 2))
                tuned.close()
                retuned[L["name"]] = opts[0]
            if world > 1:
                dist.broadcast_object_list(opts, src=0)
            chosen.append(opts[0])
            kw = dict(base)
            kw.update(opts[0])
            p = srt.Plan.from_csr(w, dtype=tdt, device=local, **kw)
        build_ms.append(round(p.info["build_ms"] + p.info["jit_compile_ms"], 1))
        X = torch.from_numpy(x).to(dev).to(tdt).contiguous()
        if L["kind"] == "spmm":
            Y = torch.empty((L["M"], L["N"]), dtype=tdt, device=dev)
        else:
            Y = torch.empty((L["M"], L["B"], L["H"], L["W"]), dtype=tdt, device=dev)
        plans.append((p, w))
        xs.append(X)
        ys.append(Y)
        host.append(x)
    if retuned and rank == 0 and not saved:
        os.makedirs(os.path.dirname(tuned_path), exist_ok=True)
        with open(tuned_path, "w") as f:
            json.dump(retuned, f, indent=1)
    stream = torch.cuda.current_stream(dev)
    digests = [int(p.info["digest"]) for p, _ in plans]
    replicas_equal = True
    if world > 1:
        allds = [None] * world
        dist.all_gather_object(allds, digests)
        replicas_equal = all(d == allds[0] for d in allds)

    def call(i, X=None, Y=None, stream=stream):
        p, _ = plans[i]
        if layers[i]["kind"] == "spmm":
            p.spmm(xs[i] if X is None else X, ys[i] if Y is None else Y, stream=stream)
        else:
            p.conv3x3(xs[i] if X is None else X, ys[i] if Y is None else Y, stream=stream)

    # L2 flush: write a 256 MiB buffer (evicts everything), then read a second 256 MiB buffer
    # so the write-back of the dirty flush lines also happens here, outside the timed events,
    # and the timed step starts from a cold and clean L2 (HBM-honest inputs, no write-back of
    # flush data charged to the first kernels)
    flush_w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_r = torch.zeros(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.empty(1, dtype=torch.float32, device=dev)

    class _Flush:
        @staticmethod
        def zero_():
            flush_w.zero_()
            torch.sum(flush_r, dim=0, out=flush_sink[0])

    flush = _Flush()
    nl = len(layers)
    flops_step = sum(2 * plans[i][1].nnz * layer_N(layers[i]) for i in range(nl))

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        flush.zero_()
        for i in range(nl):
            call(i)
    torch.cuda.synchronize()

    # One step = the nl executor launches, captured once in a CUDA graph (launch-bound layers
    # would otherwise time the host).  The step graph has events only at its two ends, so
    # consecutive kernels chain directly (programmatic dependent launch overlaps one layer's
    # prologue with the previous layer's tail); the `value` is timed on it.  A second graph of
    # the same launches with an event between every two kernels is replayed for the same
    # number of steps to measure each kernel's duration (roofline, per-layer breakdown).
    graph = graph_l = None
    gev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(nl + 1)]
    sev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(2)]
    if not args.eager:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            cur = torch.cuda.current_stream(dev)
            sev[0].record(cur)
            for i in range(nl):
                call(i, stream=cur)
            sev[1].record(cur)
        graph_l = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_l):
            cur = torch.cuda.current_stream(dev)
            gev[0].record(cur)
            for i in range(nl):
                call(i, stream=cur)
                gev[i + 1].record(cur)
        for _ in range(max(1, args.warmup // 2)):
            flush.zero_()
            graph.replay()
            flush.zero_()
            graph_l.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, layer_acc = [], [0.0] * nl
    if graph is not None:
        for s in range(args.steps):
            flush.zero_()
            torch.cuda.nvtx.range_push("timed")  # ncu --nvtx-include "timed/" selects these
            graph.replay()
            torch.cuda.nvtx.range_pop()
            torch.cuda.synchronize()
            step_ms.append(sev[0].elapsed_time(sev[1]))
        for s in range(args.steps):
            flush.zero_()
            graph_l.replay()
            torch.cuda.synchronize()
            for i in range(nl):
                layer_acc[i] += gev[i].elapsed_time(gev[i + 1])
    else:
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)] for _ in range(args.steps)]
        for s in range(args.steps):
            flush.zero_()
            torch.cuda.nvtx.range_push("timed")
            ev[s][0].record(stream)
            for i in range(nl):
                call(i)
                ev[s][i + 1].record(stream)
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        step_ms = [ev[s][0].elapsed_time(ev[s][nl]) for s in range(args.steps)]
        for s in range(args.steps):
            for i in range(nl):
                layer_acc[i] += ev[s][i].elapsed_time(ev[s][i + 1])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    layer_ms = [v / args.steps for v in layer_acc]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max = float(t.item())
    value = flops_step * world * args.steps / (total_ms_max * 1e-3) / 1e9
    # kernels per layer call: the executor, + the device repack of an X whose row stride is
    # not 16-byte aligned (N = 49 ...), + the tensor-core sub-block kernel when the plan has
    # dense tiles; TMA-fed conv: the input pre-pass + the conv kernel
    def kernels_per_call(i):
        info = plans[i][0].info
        if layers[i]["kind"] != "spmm":
            return 2 if info["conv_kernel"] == 2 else 1
        X = xs[i]
        unaligned = (X.data_ptr() % 16) != 0 or (X.stride(0) * X.element_size()) % 16 != 0
        return 1 + int(unaligned) + int(info["tc_tiles"] > 0)

    launches = args.steps * sum(kernels_per_call(i) for i in range(nl))

    # ---------------- roofline of the dominant kernel (longest layer)
    peaks = load_peaks()
    alu = alu_peak_gflops(peaks["sm_max_mhz"])
    per_layer = []
    for i, L in enumerate(layers):
        p, w = plans[i]
        N = layer_N(L)
        x_bytes = S * (L["K"] if L["kind"] == "spmm" else L["c_in"]) * N
        y_bytes = S * L["M"] * N
        alg_bytes = x_bytes + y_bytes + p.info["plan_bytes"]
        flops = 2 * w.nnz * N
        t_fma = flops / (alu * 1e9)
        t_hbm = alg_bytes / (peaks["hbm_gbs"] * 1e9)
        bound = "alu" if t_fma >= t_hbm else "hbm"
        sec = layer_ms[i] * 1e-3
        per_layer.append(dict(name=L["name"], M=L["M"], K=L["K"], N=N, nnz=w.nnz, ms=layer_ms[i],
                              gflops=flops / sec / 1e9, bound=bound,
                              roof_frac=max(t_fma, t_hbm) / sec, alg_bytes=alg_bytes))
    dom = max(range(nl), key=lambda i: layer_ms[i])
    d = per_layer[dom]
    sec = d["ms"] * 1e-3
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}_{args.dtype}_s{args.sparsity}.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath)).get(d["name"])
        traffic = t and t.get("traffic_bytes_per_launch")
    pinfo = plans[dom][0].info
    if pinfo.get("executor") == 3:
        # condensed-panel tensor cores (DESIGN.md kernel 5b): a dense fp16 contraction of the
        # panels' column unions; executed flops = 2 * 16 * 16 * N per k16 step, against the
        # measured dense bf16 peak (fp16 runs at the same tensor rate)
        tc_flops = 2 * 16 * 16 * d["N"] * pinfo["tc_panel_steps"]
        roof = {"bound": "tensor", "achieved": tc_flops / sec / 1e12, "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "useful_tflops": 2 * d["nnz"] * d["N"] / sec / 1e12,
                "executed_flops_per_launch": tc_flops}
    elif d["bound"] == "hbm":
        roof = {"bound": "hbm", "achieved": d["alg_bytes"] / sec / 1e9, "peak": peaks["hbm_gbs"],
                "unit": "GB/s"}
    else:
        roof = {"bound": "alu", "achieved": 2 * d["nnz"] * d["N"] / sec / 1e12,
                "peak": alu / 1e3, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = traffic
    roof["kernel"] = d["name"]
    roof["peak_source"] = peaks["source"] if roof["bound"] == "hbm" else \
        ("MEASURED_PEAKS.json bf16_tflops (dense tcgen05 cuBLAS; this kernel issues mma.sync)"
         if roof["bound"] == "tensor" else
         "derived: 148 SM x 128 FP32 lanes x 2 x sm_max_mhz (MEASURED_PEAKS.json)")
    roof["alg_bytes_per_launch"] = d["alg_bytes"]
    roof["flops_per_launch"] = 2 * d["nnz"] * d["N"]
    # Design ceilings of the CUDA-core executor, context for `frac`: one shared-
    # memory X load per lane-FMA caps it at 25% (fp32) / 50% (fp16) of the FMA peak, and every
    # row panel re-reads its X tiles from L2 (measured L2 -> SM streaming: 4.7 TB/s).
    pi = plans[dom][0].info
    Ld = layers[dom]
    xb = S * (Ld["K"] if Ld["kind"] == "spmm" else Ld["c_in"]) * d["N"]
    t_smem = 2 * d["nnz"] * d["N"] / (alu * 1e9 * (0.5 if S == 2 else 0.25))
    t_l2 = pi["panels"] * xb / 4.7e12
    t_ceil = max(t_smem, t_l2, max(d["alg_bytes"] / (peaks["hbm_gbs"] * 1e9), 0.0))
    roof["design_ceiling"] = {"smem_fma_frac_max": 0.5 if S == 2 else 0.25,
                              "t_smem_us": t_smem * 1e6, "t_l2_reread_us": t_l2 * 1e6,
                              "frac_of_design_ceiling": t_ceil / (d["ms"] * 1e-3)}

    # ---------------- optional gather of Y over ranks: off the data path, NCCL
    # all-gather (NVLink / NVSwitch) of every layer's output slab, timed separately
    gather = None
    if world > 1 and not args.quick:
        outs = [torch.empty((world,) + tuple(y.shape), dtype=y.dtype, device=dev) for y in ys]
        for _ in range(2):
            for y, o in zip(ys, outs):
                dist.all_gather_into_tensor(o, y.contiguous())
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        g0.record(stream)
        for _ in range(reps):
            for y, o in zip(ys, outs):
                dist.all_gather_into_tensor(o, y.contiguous())
        g1.record(stream)
        torch.cuda.synchronize()
        tg = torch.tensor([g0.elapsed_time(g1) / reps], dtype=torch.float64, device=dev)
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        gather = {"ms_per_step": float(tg.item()), "bytes_per_rank": sum(y.numel() * S for y in ys),
                  "collective": "all_gather_into_tensor (NCCL), not part of the timed step"}
        del outs

    # ---------------- e2e through the public API with host buffers
    e2e = None
    if not (args.no_e2e or args.quick):
        hx = [torch.from_numpy(h).to(tdt).pin_memory() for h in host]
        hy = [torch.empty(tuple(y.shape), dtype=tdt).pin_memory() for y in ys]
        h2d = sum(h.numel() * S for h in hx)
        d2h = sum(y.numel() * S for y in hy)
        n_e2e = max(3, min(args.steps, 50))
        # Three streams: copy-in (pinned host -> device), compute (the executors), copy-out
        # (device -> pinned host), chained per layer with events, so the H2D of the next layer,
        # the current layer's kernel and the D2H of the previous layer overlap (PCIe is full
        # duplex).  Every step still copies all of its inputs in and all of its results out.
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(nl)]
        ev_done = [torch.cuda.Event() for _ in range(nl)]
        ev_out = [torch.cuda.Event() for _ in range(nl)]

        def e2e_step(first):
            for i in range(nl):
                if not first:
                    s_in.wait_event(ev_done[i])  # previous step's kernel i has read xs[i]
                with torch.cuda.stream(s_in):
                    xs[i].copy_(hx[i], non_blocking=True)
                    ev_in[i].record(s_in)
                stream.wait_event(ev_in[i])
                if not first:
                    stream.wait_event(ev_out[i])  # previous step's ys[i] is on the host
                call(i)
                ev_done[i].record(stream)
                s_out.wait_event(ev_done[i])
                with torch.cuda.stream(s_out):
                    hy[i].copy_(ys[i], non_blocking=True)
                    ev_out[i].record(s_out)

        for s in range(2):
            e2e_step(s == 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_in)
        stream.wait_event(e0)
        s_out.wait_event(e0)
        for s in range(n_e2e):
            e2e_step(s == 0)
        s_out.wait_stream(stream)
        s_out.wait_stream(s_in)
        e1.record(s_out)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": flops_step * world * n_e2e / (float(te.item()) * 1e-3) / 1e9,
               "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "steps": n_e2e, "pipeline": "H2D / kernels / D2H on three streams, per-layer events"}

    # ---------------- dense GEMM context (same shapes, W densified, cold L2)
    dense = None
    if not (args.no_dense or args.quick) and rank == 0:
        dense = {}
        prev_tf32 = torch.backends.cuda.matmul.allow_tf32
        prev_cudnn_tf32 = torch.backends.cudnn.allow_tf32
        torch.backends.cudnn.benchmark = True
        # fp32 dense context = true fp32 (SGEMM / fp32 cuDNN conv, TF32 off), the paper's
        # cuBLAS / cuDNN fp32 baselines; fp16 = tensor cores
        ctx = [("fp32_sgemm", torch.float32, False), ("fp16_tc", torch.float16, False)]
        if args.dtype == "bf16":
            ctx.append(("bf16_tc", torch.bfloat16, False))
        for label, ddt, tf32 in ctx:
            torch.backends.cuda.matmul.allow_tf32 = tf32
            torch.backends.cudnn.allow_tf32 = tf32
            tot = 0.0
            for i, L in enumerate(layers):
                w = plans[i][1]
                Wd = torch.from_numpy(gen.to_dense(w, np.float32)).to(dev, ddt)
                if L["kind"] == "spmm":
                    Xd = xs[i].to(ddt)
                    fn = lambda: torch.matmul(Wd, Xd)
                else:
                    import torch.nn.functional as F
                    Xn = xs[i].to(ddt).permute(1, 0, 2, 3).contiguous()
                    Wc = Wd.reshape(L["M"], L["c_in"], 3, 3)
                    fn = lambda: F.conv2d(Xn, Wc, padding=1)
                for _ in range(3):
                    fn()
                reps = 10
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ms = []
                for _ in range(reps):
                    flush.zero_()
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                tot += statistics.median(ms)
            sparse_step = statistics.median(step_ms)
            dense[label] = {"ms_per_step": tot, "speedup_of_sparse": tot / sparse_step}
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
        torch.backends.cudnn.allow_tf32 = prev_cudnn_tf32

    # ---------------- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if not (args.no_cpu_baseline or args.quick) and rank == 0 and world == 1:
        import oracle
        samples = oracle_step_sample(layers, args.sparsity, 10.0, rank)
        t0 = time.perf_counter()
        fl = run_oracle_step(samples)
        dt = time.perf_counter() - t0
        cpu = {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": oracle.default_threads(),
               "kind": "oracle",
               "sample": "; ".join(f"{L['name']}: first {n} of {layer_N(L)} columns"
                                   for L, (_, _, _, n) in zip(layers, samples)),
               "seconds": dt}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"{args.workload}_s{args.sparsity}_{args.dtype}",
                       "description": desc, "sparsity_pct": args.sparsity,
                       "layers": [f"{L['M']}x{L['K']}xN{layer_N(L)}" for L in layers],
                       "l2": "flushed before every timed step, outside the events: 256 MiB write, then a 256 MiB read (cold, clean L2; inputs > L2 not needed)",
                       "launch": "eager" if args.eager else "cuda-graph replay of the step",
                       "layer_times": "eager, events between launches" if args.eager else
                       "second graph of the same launches with an event between kernels, replayed "
                       "for the same number of steps (the step graph has events only at its ends)",
                       "plan_build_ms": build_ms,
                       "executor": {0: "plan-driven", 1: "jit", 2: "auto"}[args.executor],
                       "tuned": None if args.no_tune else chosen,
                       "tuned_us": None if args.no_tune else tuned_us,
                       "tuned_from": None if args.no_tune else (
                           os.path.relpath(tuned_path, ROOT) if saved else "timed search in this run"),
                       "parallelism": f"N-sharded x{world}, replicated plan, no collective",
                       "replica_digests_equal": replicas_equal},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "layers": per_layer, "dense_baseline": dense, "gather": gather,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
