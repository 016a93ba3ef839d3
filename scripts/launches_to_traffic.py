"""Turn an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv, restricted to the bench's timed NVTX range) into
profiles/traffic_<workload>_<dtype>_s<sparsity>.json: per layer, the mean DRAM bytes per
launch (read + write) and the ncu duration, plus each layer's share of the step.

    python scripts/launches_to_traffic.py LAUNCHES.csv WORKLOAD DTYPE SPARSITY OUT.json
"""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

path, wl, dt, sp, out = sys.argv[1:6]
layers, _, _ = bench.workload_layers(wl, int(sp), 1)
names = [L["name"] for L in layers]
rows = [r for r in csv.reader(open(path)) if r]
hdr = next(r for r in rows if "Metric Name" in r)
idx = {h: i for i, h in enumerate(hdr)}
per = collections.OrderedDict()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    kid = int(r[idx["ID"]])
    name = r[idx["Kernel Name"]]
    if "spmm" not in name and "conv3x3" not in name and "srt_jit" not in name:
        continue
    d = per.setdefault(kid, {"kernel": name})
    val = float(r[idx["Metric Value"]].replace(",", ""))
    unit = r[idx["Metric Unit"]]
    m = r[idx["Metric Name"]]
    if m.startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[m] = val * scale
    elif m == "gpu__time_duration.sum":
        scale = {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        d["us"] = val * scale
launches = list(per.values())
res = {}
for i, L in enumerate(names):
    mine = launches[i::len(names)]
    if not mine:
        continue
    res[L] = {
        "traffic_bytes_per_launch": sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                                        for m in mine) / len(mine),
        "ncu_us_per_launch": sum(m.get("us", 0) for m in mine) / len(mine),
        "launches": len(mine),
        "kernel": mine[0]["kernel"][:80],
    }
tot = sum(v["ncu_us_per_launch"] for v in res.values()) or 1
for v in res.values():
    v["share_of_step"] = v["ncu_us_per_launch"] / tot
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
