"""Ablations on B200 (the paper's P:385-387 experiments): autotuning vs the
heuristic and vs round-1 defaults, LPT load balancing vs natural row order (uniform and
Zipf-skewed rows), JIT vs plan-driven executor, TMEM vs shared-memory X source, X multicast.
Each variant: median of 15 cold-L2 launches (256 MiB write + 256 MiB read before each), CUDA
events.  Writes profiles/r01_v6_ablation.json.

    python scripts/ablation.py [out.json]
"""
import json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11849_b200 as srt
from synth import gen

dev = torch.device("cuda:0")
fw = torch.empty(64 << 20, device=dev)
fr = torch.zeros(64 << 20, device=dev)
sink = torch.empty(1, device=dev)


def cold_us(plan, X, Y, reps=15):
    ts = []
    for _ in range(reps + 2):
        fw.zero_()
        torch.sum(fr, dim=0, out=sink[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.spmm(X, Y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts[2:])


CASES = [("bert_3072x768_N16384", 3072, 768, 16384, "f32"),
         ("rn50_p8_2048x512_N392", 2048, 512, 392, "f32"),
         ("mbv1_p20_1024x1024_N1568", 1024, 1024, 1568, "f16")]
out = {}
for name, M, K, N, dt in CASES:
    tdt = torch.float16 if dt == "f16" else torch.float32
    X = torch.rand(K, N, device=dev, dtype=tdt)
    Y = torch.empty(M, N, device=dev, dtype=tdt)
    for pattern in ("uniform", "zipf"):
        w = gen.pruned_weights(M, K, 90, seed=7) if pattern == "uniform" else \
            gen.stress_pattern("zipf", M, K, seed=7)
        res = {}
        tuned = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, tune=1)
        topt = tuned.chosen_opts()
        res["tuned"] = cold_us(tuned, X, Y)
        res["tuned_opts"] = topt
        res["heuristic_default"] = cold_us(srt.Plan.from_csr(w, dtype=tdt, n_hint=N), X, Y)
        res["round1_defaults_w8_R4_kc64_st2"] = cold_us(srt.Plan.from_csr(
            w, dtype=tdt, n_hint=N, warps=8, rows_per_warp=4, k_chunk=64, stages=2), X, Y)
        po = {k: v for k, v in topt.items() if k not in ("executor", "jit_rows", "jit_warps")}
        po["executor"] = 0
        res["plan_driven_tuned_opts_lpt"] = cold_us(srt.Plan.from_csr(w, dtype=tdt, n_hint=N, **po), X, Y)
        res["plan_driven_tuned_opts_natural_rows"] = cold_us(srt.Plan.from_csr(
            w, dtype=tdt, n_hint=N, **dict(po, row_order=1)), X, Y)
        pl = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, **dict(po, row_order=1))
        res["natural_rows_panel_nnz_min_max"] = [pl.info["min_panel_nnz"], pl.info["max_panel_nnz"]]
        pl = srt.Plan.from_csr(w, dtype=tdt, n_hint=N, **po)
        res["lpt_panel_nnz_min_max"] = [pl.info["min_panel_nnz"], pl.info["max_panel_nnz"]]
        if pattern == "uniform":
            if M * K <= 2048 * 1024:
                try:
                    res["jit_executor"] = cold_us(srt.Plan.from_csr(w, dtype=tdt, n_hint=N, executor=1), X, Y)
                except srt.SparseRTError as e:
                    res["jit_executor"] = str(e)[:80]
            base = dict(warps=16, rows_per_warp=4, k_chunk=56)
            res["x_source_smem_w16_R4_kc56"] = cold_us(srt.Plan.from_csr(w, dtype=tdt, n_hint=N, **base), X, Y)
            res["x_source_tmem_w16_R4_kc56"] = cold_us(srt.Plan.from_csr(
                w, dtype=tdt, n_hint=N, x_source=1, **base), X, Y)
            for cm in (1, 2, 4):
                try:
                    res[f"x_multicast_{cm}_w16_R4_kc64"] = cold_us(srt.Plan.from_csr(
                        w, dtype=tdt, n_hint=N, warps=16, rows_per_warp=4, k_chunk=64, x_multicast=cm), X, Y)
                except srt.SparseRTError as e:
                    res[f"x_multicast_{cm}_w16_R4_kc64"] = str(e)[:80]
        out[f"{name}_{dt}_{pattern}"] = res
        print(name, dt, pattern, json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}), flush=True)
path = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_v6_ablation.json"
json.dump({"method": "median of 15 cold-L2 single launches (CUDA events), us", "results": out},
          open(path, "w"), indent=1)
