#!/usr/bin/env python
"""Benchmark of the B200 SparseRT hot path (effective GFLOP/s = 2*nnz*N / t).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload conv] [--dtype f32]
    python bench.py --impl reference ...     # the CPU oracle arm (rank 0 only)
    python bench.py --plan-only --gpus 2     # launcher + sharding + replicated plans, no GPU

A "step" is one pass of the executor over one batch of synthetic input for every layer of
the workload (the plans are built once, offline, like the paper's inspector; their
build time is reported in config.plan_build_ms).  Default workload: BASELINE.json
configs[4], the ResNet-50 sparse 3x3 conv (256 channels, 14x14) at batch 256 and 90%
sparsity in fp32 (the paper's precision) -- the largest configuration BASELINE names
that fits one GPU and the one it shards over 1/2/4/8 GPUs.  The same JSON line carries a
`secondary` block with the BERT-base FFN layers at N = 32 x 512 (configs[3]) in fp32 and
fp16 and the same conv in fp16, timed the same way.  L2 is flushed (256 MiB write + 256 MiB read) before every timed
step, outside the timed events, so every layer reads cold HBM.

After timing, every timed plan is checked against the CPU oracle (`parity`): the timed
outputs on sampled columns / images (rel-L2 within the north-star tolerance), and the same
plan options on integer data at the full timed size (bitwise on the samples).  A failed check
marks the line `parity_checked: false` and exits 1.

Multi-GPU (`--gpus N`): one process per GPU.  Without WORLD_SIZE in the environment the
script re-launches itself under `torch.distributed.run` with N local ranks (and fails if
fewer than N GPUs are visible).  The conv workload shards the fixed batch of 256 images over
the ranks by whole images (strong scaling); the layer workloads give every rank
its own batch (weak scaling).  Plans are replicated (digests compared), no collective on the
data path; NCCL (communicator log on stderr) carries only barriers and the max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
CONV_BATCH = 256
TOL = {"f32": 1e-5, "f16": 1e-2, "bf16": 1e-2}  # north-star rel-L2 gates


# ----------------------------------------------------------------------------- workloads

def workload_layers(name: str, world: int, rank: int):
    """Returns (layers, scaling, description).  layer = dict(kind, M, K, N | conv geometry);
    conv layers carry the rank's image range [b0, b1) of the global batch."""
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
        from paper_2008_11849_b200.shard import shard_columns
        b0, b1 = shard_columns(CONV_BATCH, world, rank)
        if b1 <= b0:
            raise SystemExit(f"conv workload: {world} ranks for {CONV_BATCH} images")
        return ([dict(kind="conv", name="rn50_conv3x3_256ch_14", M=256, K=9 * 256, c_in=256,
                      H=14, W=14, B=b1 - b0, b0=b0, b1=b1)], "strong",
                f"ResNet-50 3x3 conv 256ch 14x14, batch {CONV_BATCH} sharded over GPUs by whole images")
    if name == "tiny":
        return [dict(kind="spmm", name="tiny", M=64, K=64, N=128)], "weak", "tiny 64x64x128"
    raise SystemExit(f"unknown workload {name}")


def layer_N(L):
    return L["N"] if L["kind"] == "spmm" else L["B"] * L["H"] * L["W"]


def make_inputs(L, sparsity, rank, integer=False, f16=False):
    """Seeded synthetic inputs (synth/gen.py recipe).  Conv: the rank's images of ONE global
    256-image batch (so the shards concatenate to the unsharded problem).  integer=True: the
    exact-mode data of SURVEY 8(c) at the same positions (every partial sum an exact integer)."""
    seed = gen.case_seed(L["name"], sparsity)
    vw, vx = (2, 4) if f16 else (3, 3)
    w = gen.int_weights(L["M"], L["K"], sparsity, seed, vmax=vw) if integer else \
        gen.pruned_weights(L["M"], L["K"], sparsity, seed=seed)
    if L["kind"] == "spmm":
        xs = seed + 1 + 1000 * rank + (555 if integer else 0)
        x = gen.int_x(L["K"], L["N"], xs, vmax=vx) if integer else gen.uniform_x(L["K"], L["N"], seed=xs)
    else:
        rng = np.random.default_rng(seed + 1 + (555 if integer else 0))
        shape = (L["c_in"], CONV_BATCH, L["H"], L["W"])
        if integer:
            full = rng.integers(-vx, vx + 1, size=shape).astype(np.float32)
        else:
            full = np.maximum(rng.standard_normal(shape), 0.0).astype(np.float32)
        x = np.ascontiguousarray(full[:, L["b0"]:L["b1"]])
    return w, x


def tuned_path(workload, dtype, sparsity, executor):
    return os.path.join(ROOT, "profiles", f"tuned_{workload}_{dtype}_s{sparsity}_x{executor}.json")


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
    layers, scaling, desc = workload_layers(args.workload, 1, 0)
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
        "config": {"workload": f"{args.workload}_s{args.sparsity}_{args.dtype}", "description": desc,
                   "sparsity_pct": args.sparsity,
                   "oracle": "oracle/oracle.c (dense-expanded m-k-n triple loop / direct 7-loop "
                             "conv, double, OpenMP)"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": sample_desc},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- launcher

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_relaunch(args, visible_gpus) -> int | None:
    """--gpus N without a torch.distributed environment: re-launch this script under
    torch.distributed.run with N local ranks (one process per GPU).  Returns the exit code of
    the launched job, or None when this process is already the right rank."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        if int(world_env) != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}", file=sys.stderr)
            return 2
        return None
    if args.gpus <= 1:
        return None
    if visible_gpus is not None and visible_gpus < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {visible_gpus} GPU(s) are visible",
              file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


def plan_only_arm(args):
    """The multi-rank host logic without a GPU: every rank builds host-only plans of the
    workload (the tuned options when present), takes its shard, and the ranks compare plan
    digests over gloo.  Rank 0 prints one JSON line."""
    import torch.distributed as dist
    import paper_2008_11849_b200 as srt
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    layers, scaling, desc = workload_layers(args.workload, world, rank)
    tp = tuned_path(args.workload, args.dtype, args.sparsity, args.executor)
    saved = json.load(open(tp)) if os.path.exists(tp) else {}
    import torch
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16}.get(args.dtype, torch.float32)
    mine = []
    for L in layers:
        w, _ = make_inputs(L, args.sparsity, rank) if L["kind"] == "spmm" else \
            (gen.pruned_weights(L["M"], L["K"], args.sparsity, gen.case_seed(L["name"], args.sparsity)), None)
        kw = dict(n_hint=L["N"]) if L["kind"] == "spmm" else \
            dict(kind=srt.SPARSE_CONV3X3, c_in=L["c_in"], h=L["H"], w=L["W"], n_hint=L["B"])
        kw.update(saved.get(L["name"], {}))
        p = srt.Plan.from_csr(w, dtype=tdt, device=srt.SPARSE_DEVICE_HOST_ONLY, **kw)
        mine.append(dict(name=L["name"], digest=int(p.info["digest"]), N=layer_N(L),
                         images=[L.get("b0"), L.get("b1")] if L["kind"] == "conv" else None))
        p.close()
    allr = [None] * world
    if world > 1:
        dist.all_gather_object(allr, mine)
    else:
        allr = [mine]
    if rank == 0:
        eq = all([d["digest"] for d in r] == [d["digest"] for d in allr[0]] for r in allr)
        print(json.dumps({"plan_only": True, "n_ranks": world, "workload": args.workload,
                          "scaling": scaling, "replica_digests_equal": eq,
                          "ranks": [[{k: v for k, v in d.items() if k != "digest"} for d in r]
                                    for r in allr]}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- GPU arm

class Run:
    """One workload on this rank: plans (tuned options), device buffers, timing, roofline,
    parity.  Every computation goes through the C ABI (paper_2008_11849_b200.sparsert)."""

    def __init__(self, ctx, workload, dtype, sparsity, args):
        self.ctx, self.workload, self.dtype, self.sparsity, self.args = ctx, workload, dtype, sparsity, args
        torch, srt = ctx["torch"], ctx["srt"]
        self.tdt = {"f16": torch.float16, "bf16": torch.bfloat16}.get(dtype, torch.float32)
        self.S = 2 if dtype in ("f16", "bf16") else 4
        self.layers, self.scaling, self.desc = workload_layers(workload, ctx["world"], ctx["rank"])
        self.plans, self.ws, self.xs, self.ys, self.host, self.kws = [], [], [], [], [], []
        self.build_ms, self.chosen, self.tuned_us = [], [], []
        tp = tuned_path(workload, dtype, sparsity, args.executor)
        self.tuned_path = tp
        saved = None
        if not args.no_tune and not args.retune and os.path.exists(tp):
            saved = json.load(open(tp))
        self.saved = saved
        retuned = {}
        dev, local, dist = ctx["dev"], ctx["local"], ctx["dist"]
        for L in self.layers:
            w, x = make_inputs(L, sparsity, ctx["rank"])
            if L["kind"] == "spmm":
                base = dict(n_hint=L["N"], executor=args.executor)
            else:
                base = dict(kind=srt.SPARSE_CONV3X3, c_in=L["c_in"], h=L["H"], w=L["W"], n_hint=L["B"])
            kw = dict(base)
            if not args.no_tune:
                # offline autotuning: the configuration chosen by tune=1 is stored in
                # profiles/tuned_<workload>.json and reused (deterministic, same plans under ncu);
                # --retune re-runs the timed search on rank 0.  Every rank then builds the chosen
                # configuration explicitly, so the replicated plans are identical (digests).
                opts = [saved.get(L["name"]) if saved else None]
                if opts[0] is None and ctx["rank"] == 0:
                    tuned = srt.Plan.from_csr(w, dtype=self.tdt, device=local, tune=1, **base)
                    opts = [tuned.chosen_opts()]
                    self.tuned_us.append(round(tuned.info["tuned_us"], 2))
                    tuned.close()
                    retuned[L["name"]] = opts[0]
                if ctx["world"] > 1:
                    dist.broadcast_object_list(opts, src=0)
                self.chosen.append(opts[0])
                kw.update(opts[0])
            p = srt.Plan.from_csr(w, dtype=self.tdt, device=local, **kw)
            self.kws.append(kw)
            self.build_ms.append(round(p.info["build_ms"] + p.info["jit_compile_ms"], 1))
            X = torch.from_numpy(x).to(dev).to(self.tdt).contiguous()
            if L["kind"] == "spmm":
                Y = torch.empty((L["M"], L["N"]), dtype=self.tdt, device=dev)
            else:
                Y = torch.empty((L["M"], L["B"], L["H"], L["W"]), dtype=self.tdt, device=dev)
            self.plans.append(p)
            self.ws.append(w)
            self.xs.append(X)
            self.ys.append(Y)
            self.host.append(x)
        if retuned and ctx["rank"] == 0 and not saved:
            os.makedirs(os.path.dirname(tp), exist_ok=True)
            with open(tp, "w") as f:
                json.dump(retuned, f, indent=1)
        self.digests = [int(p.info["digest"]) for p in self.plans]
        self.replicas_equal = True
        if ctx["world"] > 1:
            allds = [None] * ctx["world"]
            dist.all_gather_object(allds, self.digests)
            self.replicas_equal = all(d == allds[0] for d in allds)
        self.nl = len(self.layers)
        self.flops_step = sum(2 * self.ws[i].nnz * layer_N(self.layers[i]) for i in range(self.nl))

    def call(self, i, X=None, Y=None, stream=None):
        stream = stream or self.ctx["stream"]
        p = self.plans[i]
        if self.layers[i]["kind"] == "spmm":
            p.spmm(self.xs[i] if X is None else X, self.ys[i] if Y is None else Y, stream=stream)
        else:
            p.conv3x3(self.xs[i] if X is None else X, self.ys[i] if Y is None else Y, stream=stream)

    # ---------------------------------------------------------------- timing
    def time(self, steps, warmup, eager=False):
        """One step = the nl executor launches, captured once in a CUDA graph (launch-bound
        layers would otherwise time the host).  The step graph has events only at its two
        ends, so consecutive kernels chain directly (programmatic dependent launch overlaps one
        layer's prologue with the previous layer's tail); the `value` is timed on it.  A second
        graph of the same launches with an event between every two kernels is replayed for the
        same number of steps to measure each kernel's duration (roofline, per-layer times)."""
        torch, dist, dev, flush = self.ctx["torch"], self.ctx["dist"], self.ctx["dev"], self.ctx["flush"]
        nl, world = self.nl, self.ctx["world"]
        for _ in range(warmup):
            flush()
            for i in range(nl):
                self.call(i)
        torch.cuda.synchronize()
        graph = graph_l = None
        gev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(nl + 1)]
        sev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(2)]
        if not eager:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                cur = torch.cuda.current_stream(dev)
                sev[0].record(cur)
                for i in range(nl):
                    self.call(i, stream=cur)
                sev[1].record(cur)
            graph_l = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph_l):
                cur = torch.cuda.current_stream(dev)
                gev[0].record(cur)
                for i in range(nl):
                    self.call(i, stream=cur)
                    gev[i + 1].record(cur)
            for _ in range(max(1, warmup // 2)):
                flush()
                graph.replay()
                flush()
                graph_l.replay()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        step_ms, layer_acc = [], [0.0] * nl
        if graph is not None:
            for s in range(steps):
                flush()
                torch.cuda.nvtx.range_push("timed")  # ncu --nvtx-include "timed/" selects these
                graph.replay()
                torch.cuda.nvtx.range_pop()
                torch.cuda.synchronize()
                step_ms.append(sev[0].elapsed_time(sev[1]))
            for s in range(steps):
                flush()
                graph_l.replay()
                torch.cuda.synchronize()
                for i in range(nl):
                    layer_acc[i] += gev[i].elapsed_time(gev[i + 1])
        else:
            stream = self.ctx["stream"]
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)] for _ in range(steps)]
            for s in range(steps):
                flush()
                torch.cuda.nvtx.range_push("timed")
                ev[s][0].record(stream)
                for i in range(nl):
                    self.call(i)
                    ev[s][i + 1].record(stream)
                torch.cuda.nvtx.range_pop()
            torch.cuda.synchronize()
            step_ms = [ev[s][0].elapsed_time(ev[s][nl]) for s in range(steps)]
            for s in range(steps):
                for i in range(nl):
                    layer_acc[i] += ev[s][i].elapsed_time(ev[s][i + 1])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        self.graphs = (graph, graph_l)
        self.step_ms = step_ms
        self.layer_ms = [v / steps for v in layer_acc]
        total_ms = sum(step_ms)
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        self.total_ms_max = float(t.item())
        self.steps = steps
        self.value = self.flops_step * world * steps / (self.total_ms_max * 1e-3) / 1e9
        self.launches = steps * sum(self.kernels_per_call(i) for i in range(nl))
        return self.value

    def kernels_per_call(self, i):
        """Kernels one layer call launches: the executor, + the device repack of an X whose row
        stride is not 16-byte aligned (N = 49 ...), + the tensor-core sub-block kernel when the
        plan has dense tiles; conv: the conv kernel (+ the input pre-pass of conv_kernel 2)."""
        info = self.plans[i].info
        if self.layers[i]["kind"] != "spmm":
            return 2 if info["conv_kernel"] in (2, 4, 5) else 1  # pre-pass + conv kernel
        X = self.xs[i]
        unaligned = (X.data_ptr() % 16) != 0 or (X.stride(0) * X.element_size()) % 16 != 0
        return 1 + int(unaligned) + int(info["tc_tiles"] > 0)

    # ---------------------------------------------------------------- roofline
    def roofline(self):
        """Roofline of the dominant kernel (longest layer): algorithmic flops 2*nnz*N and bytes
        (X read once + Y written once + the plan) per launch over its measured duration."""
        peaks = load_peaks()
        alu = alu_peak_gflops(peaks["sm_max_mhz"])
        S = self.S
        per_layer = []
        for i, L in enumerate(self.layers):
            p, w = self.plans[i], self.ws[i]
            N = layer_N(L)
            x_bytes = S * (L["K"] if L["kind"] == "spmm" else L["c_in"]) * N
            y_bytes = S * L["M"] * N
            alg_bytes = x_bytes + y_bytes + p.info["plan_bytes"]
            flops = 2 * w.nnz * N
            t_fma = flops / (alu * 1e9)
            t_hbm = alg_bytes / (peaks["hbm_gbs"] * 1e9)
            sec = self.layer_ms[i] * 1e-3
            per_layer.append(dict(name=L["name"], M=L["M"], K=L["K"], N=N, nnz=w.nnz, ms=self.layer_ms[i],
                                  gflops=flops / sec / 1e9, bound="alu" if t_fma >= t_hbm else "hbm",
                                  roof_frac=max(t_fma, t_hbm) / sec, alg_bytes=alg_bytes))
        dom = max(range(self.nl), key=lambda i: self.layer_ms[i])
        d = per_layer[dom]
        sec = d["ms"] * 1e-3
        traffic = None
        tpath = os.path.join(ROOT, "profiles", f"traffic_{self.workload}_{self.dtype}_s{self.sparsity}.json")
        if os.path.exists(tpath):
            t = json.load(open(tpath)).get(d["name"])
            traffic = t and t.get("traffic_bytes_per_launch")
        pinfo = self.plans[dom].info
        if pinfo.get("executor") in (3, 4):
            # tensor cores: executor 3 = condensed panels (DESIGN.md kernel 5b), a dense 16-bit
            # contraction of the panels' column unions, 2 * 16 * 16 * N flops per k16 step;
            # executor 4 = W's nonzero 128 x 64 blocks on tcgen05 (kernel 5d), 2 * 128 * 64 * N
            # flops per block; against the measured dense bf16 peak (fp16 runs at the same rate)
            # (x_multicast row blocks per union entry); fp32 plans run 3xTF32 (three K8 MMAs per
            # 128 x 32 block) against the TF32 peak = the measured bf16 peak x the nominal 1/2
            tf = S == 4 and pinfo["executor"] == 4
            per = 2 * 16 * 16 if pinfo["executor"] == 3 else \
                (3 * 2 * 128 * 32 if tf else 2 * 128 * 64) * max(1, pinfo.get("x_multicast", 1))
            cols = d["N"]
            Ld = self.layers[dom]
            im2col = os.environ.get("SRT_CONV_IM2COL", "1") != "0" and (Ld.get("c_in", 0) * S) % 16 == 0
            if Ld["kind"] == "conv" and not im2col:  # the MMA runs over the interleaved span
                g = pinfo["conv_images_per_tile"]
                cols = -(-Ld["B"] // g) * (Ld["H"] + 2) * g * Ld["W"]
            # (im2col TMA, the default: the MMA runs over the B H W output pixels only)
            tc_flops = per * cols * pinfo["tc_panel_steps"]
            roof = {"bound": "tensor", "achieved": tc_flops / sec / 1e12,
                    "peak": peaks["bf16_tflops"] * (0.5 if tf else 1.0),
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
            (("MEASURED_PEAKS.json bf16_tflops (dense tcgen05 cuBLAS)" +
              (" x 1/2 (TF32 nominal ratio)" if S == 4 else "")) if roof["bound"] == "tensor" else
             "derived: 148 SM x 128 FP32 lanes x 2 x sm_max_mhz (MEASURED_PEAKS.json)")
        roof["alg_bytes_per_launch"] = d["alg_bytes"]
        roof["flops_per_launch"] = 2 * d["nnz"] * d["N"]
        roof["launch_us"] = d["ms"] * 1e3
        # Design ceiling of the CUDA-core executor, context for `frac`: one
        # shared-memory X load per lane-FMA caps it at 25% (fp32) / 50% (16-bit) of the FMA peak
        t_smem = 2 * d["nnz"] * d["N"] / (alu * 1e9 * (0.5 if S == 2 else 0.25))
        roof["design_ceiling"] = {"smem_fma_frac_max": 0.5 if S == 2 else 0.25,
                                  "t_smem_us": t_smem * 1e6,
                                  "frac_of_design_ceiling": max(t_smem, d["alg_bytes"] / (peaks["hbm_gbs"] * 1e9))
                                  / sec}
        self.per_layer = per_layer
        return roof

    # ---------------------------------------------------------------- parity
    def parity(self, n_cols=64, n_images=6):
        """Check the timed plans against the CPU oracle (test infrastructure, oracle/):
        (1) the timed outputs (the synthetic real-valued inputs of the timed region) on sampled
            columns / images: rel-L2 within the north-star tolerance (fp32 1e-5, 16-bit 1e-2);
        (2) the SAME plan options on integer data (SURVEY 8(c) exact mode) at the full timed
            size and launch configuration: sampled outputs bitwise equal to the oracle's exact
            result (rounded RN-even once for 16-bit outputs)."""
        import oracle
        torch, dev, srt = self.ctx["torch"], self.ctx["dev"], self.ctx["srt"]
        torch.cuda.synchronize()
        f16 = self.dtype != "f32"
        rng = np.random.default_rng(12345 + self.ctx["rank"])

        def widen(a):  # the exact values the device consumes, as float64
            return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(self.tdt).double().numpy()

        def sample_ids(L):
            if L["kind"] == "spmm":
                N = L["N"]
                ids = {0, N - 1, max(0, N - 2)} | set(rng.choice(N, size=min(N, n_cols), replace=False).tolist())
            else:
                B = L["B"]
                ids = {0, B - 1} | set(rng.choice(B, size=min(B, n_images), replace=False).tolist())
            return np.array(sorted(ids))

        def ref_of(L, w, x, ids):
            if L["kind"] == "spmm":
                return oracle.spmm(w.M, w.K, w.row_ptr, w.col_idx, widen(w.values), widen(x[:, ids]))
            return oracle.conv3x3(w.M, w.row_ptr, w.col_idx, widen(w.values), widen(x[:, ids]))

        def take(Y, L, ids):
            t = Y[:, torch.from_numpy(ids).to(dev)] if L["kind"] == "spmm" else Y[:, torch.from_numpy(ids).to(dev)]
            return t.double().cpu().numpy()

        out = {"real_rel_l2": {}, "exact_bitwise": {}, "tol": TOL[self.dtype]}
        ok = True
        for i, L in enumerate(self.layers):
            ids = sample_ids(L)
            ref = ref_of(L, self.ws[i], self.host[i], ids)
            err = oracle.rel_l2(take(self.ys[i], L, ids), ref)
            out["real_rel_l2"][L["name"]] = err
            ok &= bool(err <= TOL[self.dtype])
            # integer data through a plan with the timed options
            wi, xi = make_inputs(L, self.sparsity, self.ctx["rank"], integer=True, f16=f16)
            pi = srt.Plan.from_csr(wi, dtype=self.tdt, device=self.ctx["local"], **self.kws[i])
            Xi = torch.from_numpy(xi).to(dev).to(self.tdt).contiguous()
            Yi = torch.full_like(self.ys[i], float("nan"))
            if L["kind"] == "spmm":
                pi.spmm(Xi, Yi, stream=self.ctx["stream"])
            else:
                pi.conv3x3(Xi, Yi, stream=self.ctx["stream"])
            torch.cuda.synchronize()
            refi = widen(ref_of(L, wi, xi, ids).astype(np.float32)) if f16 else ref_of(L, wi, xi, ids)
            eq = bool(np.array_equal(take(Yi, L, ids), refi))
            out["exact_bitwise"][L["name"]] = eq
            ok &= eq
            pi.close()
            del Xi, Yi
        out["sample"] = (f"{n_cols}+3 columns per SpMM layer / {n_images}+2 images per conv layer, "
                         "seeded; integer-data plans built with the timed options")
        flag = torch.tensor([1.0 if ok else 0.0], device=dev)
        if self.ctx["world"] > 1:
            self.ctx["dist"].all_reduce(flag, op=self.ctx["dist"].ReduceOp.MIN)
        out["ok"] = bool(flag.item() == 1.0)
        self.parity_result = out
        return out

    # ---------------------------------------------------------------- dense context
    def dense(self):
        """Same-shape dense GEMM / cuDNN conv (W densified), cold L2, context only: fp32 SGEMM
        (TF32 off, the paper's cuBLAS fp32 baseline P:275) and fp16 tensor cores."""
        torch, dev, flush, stream = self.ctx["torch"], self.ctx["dev"], self.ctx["flush"], self.ctx["stream"]
        out = {}
        prev_tf32 = torch.backends.cuda.matmul.allow_tf32
        prev_cudnn_tf32 = torch.backends.cudnn.allow_tf32
        torch.backends.cudnn.benchmark = True
        ctx = [("fp32_sgemm", torch.float32), ("fp16_tc", torch.float16)]
        if self.dtype == "bf16":
            ctx.append(("bf16_tc", torch.bfloat16))
        import torch.nn.functional as F
        for label, ddt in ctx:
            torch.backends.cuda.matmul.allow_tf32 = False
            torch.backends.cudnn.allow_tf32 = False
            tot = 0.0
            for i, L in enumerate(self.layers):
                Wd = torch.from_numpy(gen.to_dense(self.ws[i], np.float32)).to(dev, ddt)
                if L["kind"] == "spmm":
                    Xd = self.xs[i].to(ddt)
                    fn = lambda: torch.matmul(Wd, Xd)  # noqa: E731
                else:
                    Xn = self.xs[i].to(ddt).permute(1, 0, 2, 3).contiguous()
                    Wc = Wd.reshape(L["M"], L["c_in"], 3, 3)
                    fn = lambda: F.conv2d(Xn, Wc, padding=1)  # noqa: E731
                for _ in range(3):
                    fn()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ms = []
                for _ in range(10):
                    flush()
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                tot += statistics.median(ms)
            out[label] = {"ms_per_step": tot, "speedup_of_sparse": tot / statistics.median(self.step_ms)}
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
        torch.backends.cudnn.allow_tf32 = prev_cudnn_tf32
        return out

    # ---------------------------------------------------------------- e2e
    def e2e(self):
        """The same metric end to end through the public API with HOST buffers: every step
        copies its inputs pinned host -> device and its results device -> pinned host.  Three
        streams (copy-in, compute, copy-out) chained per layer with events, so the H2D of the
        next layer, the current layer's kernel and the D2H of the previous layer overlap."""
        torch, dev, dist, stream = self.ctx["torch"], self.ctx["dev"], self.ctx["dist"], self.ctx["stream"]
        nl, S = self.nl, self.S
        hx = [torch.from_numpy(h).to(self.tdt).pin_memory() for h in self.host]
        hy = [torch.empty(tuple(y.shape), dtype=self.tdt).pin_memory() for y in self.ys]
        h2d = sum(h.numel() * S for h in hx)
        d2h = sum(y.numel() * S for y in hy)
        n_e2e = max(3, min(self.steps, 50))
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(nl)]
        ev_done = [torch.cuda.Event() for _ in range(nl)]
        ev_out = [torch.cuda.Event() for _ in range(nl)]

        def e2e_step(first):
            for i in range(nl):
                if not first:
                    s_in.wait_event(ev_done[i])  # previous step's kernel i has read xs[i]
                with torch.cuda.stream(s_in):
                    self.xs[i].copy_(hx[i], non_blocking=True)
                    ev_in[i].record(s_in)
                stream.wait_event(ev_in[i])
                if not first:
                    stream.wait_event(ev_out[i])  # previous step's ys[i] is on the host
                self.call(i)
                ev_done[i].record(stream)
                s_out.wait_event(ev_done[i])
                with torch.cuda.stream(s_out):
                    hy[i].copy_(self.ys[i], non_blocking=True)
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
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if self.ctx["world"] > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return {"value": self.flops_step * self.ctx["world"] * n_e2e / (float(te.item()) * 1e-3) / 1e9,
                "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": n_e2e, "pipeline": "H2D / kernels / D2H on three streams, per-layer events"}

    def gather(self):
        """Optional gather of Y over ranks: off the data path, NCCL all-gather
        (NVLink / NVSwitch) of every layer's output slab, timed separately."""
        torch, dev, dist, stream = self.ctx["torch"], self.ctx["dev"], self.ctx["dist"], self.ctx["stream"]
        world = self.ctx["world"]
        outs = [torch.empty((world,) + tuple(y.shape), dtype=y.dtype, device=dev) for y in self.ys]
        for _ in range(2):
            for y, o in zip(self.ys, outs):
                dist.all_gather_into_tensor(o, y.contiguous())
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        g0.record(stream)
        for _ in range(reps):
            for y, o in zip(self.ys, outs):
                dist.all_gather_into_tensor(o, y.contiguous())
        g1.record(stream)
        torch.cuda.synchronize()
        tg = torch.tensor([g0.elapsed_time(g1) / reps], dtype=torch.float64, device=dev)
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        return {"ms_per_step": float(tg.item()), "bytes_per_rank": sum(y.numel() * self.S for y in self.ys),
                "collective": "all_gather_into_tensor (NCCL), not part of the timed step"}

    def cpu_baseline(self):
        import oracle
        samples = oracle_step_sample(self.layers, self.sparsity, 10.0, self.ctx["rank"])
        t0 = time.perf_counter()
        fl = run_oracle_step(samples)
        dt = time.perf_counter() - t0
        return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": oracle.default_threads(),
                "kind": "oracle",
                "sample": "; ".join(f"{L['name']}: first {n} of {layer_N(L)} columns"
                                    for L, (_, _, _, n) in zip(self.layers, samples)),
                "seconds": dt}

    def config(self):
        a = self.args
        return {"workload": f"{self.workload}_s{self.sparsity}_{self.dtype}",
                "description": self.desc, "sparsity_pct": self.sparsity,
                "layers": [f"{L['M']}x{L['K']}xN{layer_N(L)}" for L in self.layers],
                "images": [[L["b0"], L["b1"]] for L in self.layers if L["kind"] == "conv"] or None,
                "l2": "flushed before every timed step, outside the events: 256 MiB write, then a "
                      "256 MiB read (cold, clean L2)",
                "launch": "eager" if a.eager else "cuda-graph replay of the step",
                "layer_times": "eager, events between launches" if a.eager else
                "second graph of the same launches with an event between kernels, replayed "
                "for the same number of steps (the step graph has events only at its ends)",
                "plan_build_ms": self.build_ms,
                "tuned": None if a.no_tune else self.chosen,
                "tuned_us": None if a.no_tune else self.tuned_us,
                "tuned_from": None if a.no_tune else (
                    os.path.relpath(self.tuned_path, ROOT) if self.saved else "timed search in this run"),
                "parallelism": f"N-sharded x{self.ctx['world']}, replicated plan, no collective",
                "replica_digests_equal": self.replicas_equal}

    def close(self):
        for p in self.plans:
            p.close()
        self.plans = []


def parse_secondary(spec: str, world: int):
    if spec == "auto":
        spec = "bert:f32:90,bert:f16:90,conv:f16:90,conv:f32:95" if world == 1 else ""
    out = []
    for item in filter(None, spec.split(",")):
        wl, dt, sp = item.split(":")
        out.append((wl, dt, int(sp)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="conv",
                    choices=["conv", "bert", "rn50_b8", "rn50_b1", "mbv1_b32", "tiny"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "f16", "bf16"])
    ap.add_argument("--sparsity", type=int, default=90)
    ap.add_argument("--secondary", default="auto",
                    help="extra workloads timed the same way, 'wl:dtype:sparsity,...'; 'auto' = "
                         "BERT FFN fp32 and fp16 and the C5 conv in fp16 at 90%%, the C5 conv fp32 at 95%% on 1 GPU, none on "
                         "N > 1; '' = none")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-timing oracle check")
    ap.add_argument("--quick", action="store_true",
                    help="skip e2e/dense/cpu/parity legs and secondaries (for ncu runs)")
    ap.add_argument("--plan-only", action="store_true",
                    help="no GPU: host-only plans, sharding and replica digests over gloo")
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
    if args.plan_only:
        rc = maybe_relaunch(args, None)
        return plan_only_arm(args) if rc is None else rc

    import torch
    rc = maybe_relaunch(args, torch.cuda.device_count())
    if rc is not None:
        return rc
    if not torch.cuda.is_available():
        print("bench.py: no CUDA device (the GPU arm has no CPU fallback)", file=sys.stderr)
        return 2
    import torch.distributed as dist
    import paper_2008_11849_b200 as srt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    nccl = None
    if world > 1:
        # NCCL's communicator log (ranks, NVLink / NVLS transport) goes to stderr, never stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        nccl = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                "version": ".".join(map(str, torch.cuda.nccl.version())),
                "log": "NCCL_DEBUG=INFO (INIT) on stderr"}
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)

    # L2 flush: write a 256 MiB buffer (evicts everything), then read a second 256 MiB buffer
    # so the write-back of the dirty flush lines also happens here, outside the timed events,
    # and the timed step starts from a cold and clean L2
    flush_w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_r = torch.zeros(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.empty(1, dtype=torch.float32, device=dev)

    def flush():
        flush_w.zero_()
        torch.sum(flush_r, dim=0, out=flush_sink[0])

    ctx = dict(torch=torch, dist=dist, srt=srt, dev=dev, local=local, rank=rank, world=world,
               stream=stream, flush=flush)
    full = not args.quick

    sampler = ClockSampler(local)
    sampler.start()
    run = Run(ctx, args.workload, args.dtype, args.sparsity, args)
    run.time(args.steps, args.warmup, eager=args.eager)
    clocks = sampler.stop()
    roof = run.roofline()
    parity = run.parity() if full and not args.no_parity else None
    gather = run.gather() if world > 1 and full else None
    e2e = run.e2e() if full and not args.no_e2e else None
    dense = run.dense() if full and not args.no_dense and rank == 0 else None
    cpu = run.cpu_baseline() if full and not args.no_cpu_baseline and rank == 0 and world == 1 else None
    line_cfg = run.config()
    per_layer, value, launches = run.per_layer, run.value, run.launches
    ms_per_step, scaling = run.total_ms_max / args.steps, run.scaling
    run.close()

    secondary = []
    for wl, dt, sp in (parse_secondary(args.secondary, world) if full else []):
        r2 = Run(ctx, wl, dt, sp, args)
        r2.time(args.steps, args.warmup, eager=args.eager)
        rf = r2.roofline()
        par = r2.parity() if not args.no_parity else None
        dn = r2.dense() if not args.no_dense and rank == 0 else None
        secondary.append({"workload": f"{wl}_s{sp}_{dt}", "metric": METRIC, "value": r2.value,
                          "unit": "GFLOP/s", "ms_per_step": r2.total_ms_max / args.steps,
                          "dtype": dt, "scaling": r2.scaling, "gpu_launches": r2.launches,
                          "roofline": rf, "parity": par,
                          "parity_checked": None if par is None else par["ok"],
                          "dense_baseline": dn, "layers": r2.per_layer, "config": r2.config()})
        r2.close()

    checked = [parity] + [s["parity"] for s in secondary]
    parity_ok = all(p["ok"] for p in checked if p is not None)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (magnitude-pruned He-normal W, seeded; DESIGN.md input recipe)",
            "config": line_cfg, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks,
            "parity_checked": None if parity is None else parity_ok, "parity": parity,
            "layers": per_layer, "dense_baseline": dense, "gather": gather, "nccl": nccl,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if parity_ok else 1


if __name__ == "__main__":
    sys.exit(main())
