"""One-line summary (plus per-layer lines) of bench JSON files."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    dense = {k: round(v["speedup_of_sparse"], 2) for k, v in (d.get("dense_baseline") or {}).items()}
    print(f"{f}: value={d['value']:.0f} ms={d['ms_per_step']:.4f} frac={r.get('frac', 0):.3f} "
          f"({r.get('bound')} {r.get('kernel')}) e2e={e2e} dense={dense}")
    tuned = (d.get("config") or {}).get("tuned") or []
    for i, L in enumerate(d.get("layers", [])):
        t = tuned[i] if i < len(tuned) else {}
        print(f"   {L['name']:24s} {L['ms']*1e3:8.1f} us {L['gflops']:8.0f} GF/s {L['bound']} {L['roof_frac']:.3f} {t}")
