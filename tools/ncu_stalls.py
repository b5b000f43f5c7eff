#!/usr/bin/env python
"""Per-loop stall breakdown of an ncu report's SASS page: the hottest straight-line groups (as in
ncu_sass_summary.py) with the share of each warp-stall reason among their samples.
  python tools/ncu_stalls.py gpurun_out/me_box_full.ncu-rep [n_groups]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
ie = h.index("Instructions Executed")
sc = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
def num(x):
    try: return float(x)
    except ValueError: return 0.0
groups = []
for i, r in enumerate(data):
    c = num(r[ie])
    if groups and groups[-1]["c"] == c and c > 0: g = groups[-1]
    else:
        g = {"c": c, "i": i, "n": 0, "st": collections.Counter()}; groups.append(g)
    g["n"] += 1
    for j in sc: g["st"][h[j][6:]] += num(r[j])
groups.sort(key=lambda g: -g["c"] * g["n"])
for g in groups[:int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
    tot = sum(g["st"].values()) or 1
    print(f"at {g['i']} n {g['n']} cnt {g['c']:.0f}: " + ", ".join(f"{k} {v/tot*100:.0f}%" for k, v in g["st"].most_common(8)))
