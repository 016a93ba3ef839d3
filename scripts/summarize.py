"""Print a compact table of bench JSON lines (files given on the command line)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f"== {f}: unreadable ({e})")
        continue
    r = d.get("roofline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    dense = d.get("dense_baseline") or {}
    print(f"== {f}: {d['value']:.1f} GFLOP/s  {d['ms_per_step']*1e3:.1f} us/step  e2e {e2e and round(e2e,1)}  "
          f"roof {r.get('bound')} frac {r.get('frac', 0):.3f} ({r.get('kernel')})  clocks {d.get('clocks', {}).get('sm_mhz')}")
    if dense:
        print("   dense: " + ", ".join(f"{k} {v['ms_per_step']*1e3:.1f}us x{v['speedup_of_sparse']:.2f}" for k, v in dense.items()))
    for L in d.get("layers", []):
        print(f"   {L['name']:<24} {L['M']:>5}x{L['K']:<5} N={L['N']:<6} {L['ms']*1e3:8.2f} us {L['gflops']:9.1f} GF/s {L['bound']} {L['roof_frac']:.3f}")
