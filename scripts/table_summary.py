"""Summarise scripts/measure_table.py output (JSON lines) into a markdown table with the
north-star geomeans: speedup of the sparse kernel over the same-shape dense GEMM (fp16 / bf16
tensor cores, fp32 SGEMM with TF32 off) at 90 % and 95 % sparsity, and the roofline fraction.

    python scripts/table_summary.py profiles/r02_table.jsonl > profiles/r02_table.md
"""
import collections
import json
import math
import sys


def gmean(v):
    v = [x for x in v if x and x > 0]
    return math.exp(sum(math.log(x) for x in v) / len(v)) if v else float("nan")


rows = [json.loads(ln) for f in sys.argv[1:] for ln in open(f) if ln.strip()]
ok = [r for r in rows if "error" not in r]
bad = [r for r in rows if "error" in r]
print("# Per-shape measurement table (B200, 1 GPU, cold L2)\n")
print("Sparse = autotuned plan (P:259-263), cold-L2 median of 15 launches; dense = torch.matmul / "
      "cuDNN conv2d on the densified W (context only; fp32 with TF32 off).  `frac` = roofline "
      "fraction (slower of FFMA peak on 2 nnz N and HBM bytes of X + Y + plan, MEASURED_PEAKS.json).  "
      "`exact` = the tuned plan on integer data is bitwise equal to the oracle on sampled outputs.\n")
print(f"{len(ok)} cases measured, {len(bad)} errors, "
      f"{sum(1 for r in ok if r.get('exact'))} / {len(ok)} exact.\n")
print("## Geomeans\n")
print("| group | sparsity | dtype | cases | sparse GFLOP/s (gm) | frac (gm) | vs fp32 SGEMM | vs fp16 TC | vs bf16 TC |")
print("|---|---|---|---|---|---|---|---|---|")
grp = collections.defaultdict(list)
for r in ok:
    grp[(r["group"], r["sparsity"], r["dtype"])].append(r)
for (g, sp, dt), rs in sorted(grp.items()):
    print(f"| {g} | {sp} | {dt} | {len(rs)} | {gmean([r['gflops_cold'] for r in rs]):.0f} | "
          f"{gmean([r['roof_frac'] for r in rs]):.3f} | {gmean([r['speedup']['fp32_sgemm'] for r in rs]):.2f}x | "
          f"{gmean([r['speedup']['fp16_tc'] for r in rs]):.2f}x | {gmean([r['speedup']['bf16_tc'] for r in rs]):.2f}x |")
print("\n## North-star summary (RN50 / MobileNetV1 / BERT layer shapes)\n")
print("| sparsity | dtype | cases | vs dense fp16 TC (target >= 3x) | vs dense bf16 TC | vs fp32 SGEMM | frac (gm) | cases >= 0.6 of roofline |")
print("|---|---|---|---|---|---|---|---|")
for sp in (90, 95):
    for dt in ("f32", "f16"):
        rs = [r for r in ok if r["group"] in ("rn50", "mbv1", "bert") and r["sparsity"] == sp and r["dtype"] == dt]
        if not rs:
            continue
        print(f"| {sp} | {dt} | {len(rs)} | {gmean([r['speedup']['fp16_tc'] for r in rs]):.2f}x | "
              f"{gmean([r['speedup']['bf16_tc'] for r in rs]):.2f}x | {gmean([r['speedup']['fp32_sgemm'] for r in rs]):.2f}x | "
              f"{gmean([r['roof_frac'] for r in rs]):.3f} | {sum(1 for r in rs if r['roof_frac'] >= 0.6)} |")
print("\n## All cases\n")
print("| case | M x K x N | sp | dt | us cold | us warm | GFLOP/s | bound | frac | vs SGEMM | vs fp16 TC | exec | exact |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in ok:
    ex = {0: "plan", 1: "jit", 3: "tc-panels"}.get(r["executor"], str(r["executor"]))
    if r["kind"] == "conv":
        ex = f"conv{r['conv_kernel']}"
    print(f"| {r['name']} | {r['M']}x{r['K']}x{r['N']} | {r['sparsity']} | {r['dtype']} | {r['us_cold']:.1f} | "
          f"{r['us_warm']:.1f} | {r['gflops_cold']:.0f} | {r['bound']} | {r['roof_frac']:.3f} | "
          f"{r['speedup']['fp32_sgemm']:.2f}x | {r['speedup']['fp16_tc']:.2f}x | {ex} | {r['exact']} |")
for r in bad:
    print(f"| {r['name']} | error: {r['error'][:80]} | {r['sparsity']} | {r['dtype']} |")
