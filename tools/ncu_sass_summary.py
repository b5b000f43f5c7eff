#!/usr/bin/env python
"""Summarise an ncu report's SASS source page: hottest straight-line groups (by executed
instructions), their stall samples and shared-memory wavefronts, and the opcode mix of each.
  python tools/ncu_sass_summary.py gpurun_out/me_box_full.ncu-rep [n_groups]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    ng = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[1], rows[2:]
    ie, src = h.index("Instructions Executed"), h.index("Source")
    smp, wf = h.index("Warp Stall Sampling (All Samples)"), h.index("L1 Wavefronts Shared")

    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(num(r[ie]) for r in data)
    tots = sum(num(r[smp]) for r in data) or 1
    totw = sum(num(r[wf]) for r in data) or 1
    print(f"warp instructions {tot:.4g}  shared wavefronts {totw:.4g}")
    groups = []
    for i, r in enumerate(data):
        c = num(r[ie])
        if groups and groups[-1]["c"] == c and c > 0:
            g = groups[-1]
        else:
            g = {"c": c, "i": i, "n": 0, "s": 0.0, "w": 0.0, "ops": collections.Counter()}
            groups.append(g)
        g["n"] += 1
        g["s"] += num(r[smp])
        g["w"] += num(r[wf])
        op = r[src].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1]
        g["ops"][op.split()[0] if op else "?"] += 1
    groups.sort(key=lambda g: -g["c"] * g["n"])
    for g in groups[:ng]:
        print(f"count {g['c']:>12.0f} at {g['i']:5d} n {g['n']:4d}  instr {g['c'] * g['n'] / tot * 100:5.1f}%  "
              f"stalls {g['s'] / tots * 100:5.1f}%  smem {g['w'] / totw * 100:5.1f}%")
        print("     ", ", ".join(f"{k} {v}" for k, v in g["ops"].most_common(12)))


if __name__ == "__main__":
    main()
