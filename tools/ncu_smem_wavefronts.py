#!/usr/bin/env python
"""Per-instruction shared-memory wavefronts vs their ideal count from an ncu source-page CSV
(ncu -i REP --page source --csv --print-source sass > x.csv): python tools/ncu_smem_wavefronts.py x.csv [N]."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
ix = {n: h.index(n) for n in ["Address","Source","Instructions Executed","L1 Wavefronts Shared","L1 Wavefronts Shared Ideal","Warp Stall Sampling (All Samples)"]}
def num(x):
    try: return float(x)
    except: return 0.0
tot = sum(num(r[ix["L1 Wavefronts Shared"]]) for r in data)
toti = sum(num(r[ix["L1 Wavefronts Shared Ideal"]]) for r in data)
totI = sum(num(r[ix["Instructions Executed"]]) for r in data)
print("total wavefronts %.4g ideal %.4g instr %.4g" % (tot, toti, totI))
lst = sorted(data, key=lambda r: -num(r[ix["L1 Wavefronts Shared"]]))
for r in lst[:int(sys.argv[2]) if len(sys.argv)>2 else 40]:
    w = num(r[ix["L1 Wavefronts Shared"]]); wi = num(r[ix["L1 Wavefronts Shared Ideal"]])
    print("%8s %-52s ex %10.0f wf %10.0f ideal %10.0f x%.2f" % (r[ix["Address"]], r[ix["Source"]][:52], num(r[ix["Instructions Executed"]]), w, wi, w/max(wi,1)))
