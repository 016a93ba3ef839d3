"""Print the autotuner's cold-L2 timing of every candidate for a few layer shapes.
    SPARSERT_TUNE_DEBUG=1 python scripts/tune_landscape.py"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11849_b200 as srt
from synth import gen
shapes = [(64, 256, 25088), (256, 1024, 1568), (512, 2048, 392), (2048, 512, 392)]
if len(sys.argv) > 1:
    shapes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]]
for dt in (torch.float32,):
    for M, K, N in shapes:
        print(f"=== {M}x{K} N={N} {dt}", file=sys.stderr, flush=True)
        p = srt.Plan.from_csr(gen.pruned_weights(M, K, 90, seed=1), dtype=dt, n_hint=N, tune=1)
        print("chosen", p.chosen_opts(), p.info["tuned_us"], file=sys.stderr, flush=True)
