"""One conv layer launch (for ncu): python scripts/conv_one.py f32|f16 'opts'"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11849_b200 as srt
from synth import gen
tdt = torch.float16 if sys.argv[1] == "f16" else torch.float32
opts = dict((k, int(v)) for k, v in (kv.split("=") for kv in sys.argv[2].split(",") if kv)) if len(sys.argv) > 2 else {}
w = gen.pruned_weights(256, 2304, 90, seed=1)
x = torch.from_numpy(gen.relu_normal_x((256, 256, 14, 14), seed=2)).cuda().to(tdt)
p = srt.Plan.from_csr(w, dtype=tdt, kind=srt.SPARSE_CONV3X3, c_in=256, h=14, w=14, n_hint=256, **opts)
for _ in range(3):
    y = p.conv3x3(x)
torch.cuda.synchronize()
print(p.info)
