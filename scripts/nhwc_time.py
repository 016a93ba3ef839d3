"""Warm graph-replayed time of the C5 conv (256 ch, 14x14, batch 256, 90 %) through the
channels-last entry point sparse_conv3x3_nhwc vs the CNHW one, for explicit options.
    python scripts/nhwc_time.py f32|f16 'conv_kernel=5,cta_pair=1;...'"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11849_b200 as srt
from synth import gen
tdt = torch.float16 if sys.argv[1] == "f16" else torch.float32
w = gen.pruned_weights(256, 2304, 90, seed=1)
x = torch.from_numpy(gen.relu_normal_x((256, 256, 14, 14), seed=2)).cuda().to(tdt)
xn = x.permute(1, 2, 3, 0).contiguous()
for cs in sys.argv[2].split(";"):
    kw = dict((k, int(v)) for k, v in (kv.split("=") for kv in cs.split(",") if kv))
    p = srt.Plan.from_csr(w, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=256, h=14, w=14, n_hint=256, **kw)
    for name, fn, inp in (("cnhw", p.conv3x3, x), ("nhwc", p.conv3x3_nhwc, xn)):
        fn(inp); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); reps = 10
        with torch.cuda.stream(s):
            fn(inp); torch.cuda.synchronize()
            with torch.cuda.graph(g):
                for _ in range(reps): fn(inp)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        print(f"{name} {us:8.1f} us {2 * w.nnz * 256 * 196 / us / 1e6:6.2f} TF  {kw}", flush=True)
