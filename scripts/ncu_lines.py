"""Attribute ncu per-instruction counts (source page, SASS) to CUDA source lines using
nvdisasm -g line info.  Usage: ncu_lines.py REPORT.ncu-rep CUBIN FUNCTION_MANGLED [kernel_idx]"""
import collections
import csv
import re
import subprocess
import sys

rep, cubin, fn = sys.argv[1:4]
kidx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
off2line = {}
cur = None
inside = False
for ln in dis.splitlines():
    if re.match(r"^\s*\.section\s+\.text\.", ln):
        inside = (".text." + fn + ",") in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        off2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, blk = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        blk = []
        blocks.append(blk)
        continue
    if blk is not None:
        blk.append(r)
b = blocks[kidx]
hdr = b[0]
idx = {h: i for i, h in enumerate(hdr)}
data = b[1:]
base = int(data[0][idx["Address"]], 16)
agg = collections.Counter()
stall = collections.Counter()
tot = 0
for x in data:
    n = int(x[idx["Instructions Executed"]] or 0)
    s = int(x[idx["Warp Stall Sampling (All Samples)"]] or 0)
    off = int(x[idx["Address"]], 16) - base
    key = off2line.get(off, ("?", 0))
    agg[key] += n
    stall[key] += s
    tot += n
stot = sum(stall.values()) or 1
print("total warp-instructions", tot)
for key, n in agg.most_common(30):
    print("%5.1f%% instr %5.1f%% stall  %s:%d" % (100 * n / tot, 100 * stall[key] / stot, key[0], key[1]))
