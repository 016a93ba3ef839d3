"""Print the SASS of an ncu report with per-instruction executed counts and stall samples.

    python scripts/sass_hot.py REPORT.ncu-rep [min_count]
"""
import csv, subprocess, sys
rep = sys.argv[1]
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
i = {h: k for k, h in enumerate(hdr)}
tot = 0
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    n = int(r[i["Instructions Executed"]] or 0)
    tot += n
    if n >= mn:
        print(f"{n:9d} {r[i['Warp Stall Sampling (All Samples)']]:>6s}  {r[i['Source']].strip()}")
print("total warp instructions", tot)
