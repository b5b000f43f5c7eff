#!/usr/bin/env python
"""Per-kernel totals and shares from an ncu launch list (--metrics gpu__time_duration.sum --csv).
  python tools/launch_shares.py gpurun_out/launches.csv "<command>" > profiles/launches_rNN.json"""
import collections
import csv
import json
import sys

OURS = ("box_kernel", "epilogue_kernel", "certify_scan_kernel", "certify_fix_kernel", "project_kernel", "finalize_kernel",
        "nnc_kernel", "revgrid", "rme_decide")


def main():
    path = sys.argv[1]
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        key = next((o for o in OURS if o in name), "other: " + name[:48])
        v = float(r["Metric Value"])
        unit = r.get("Metric Unit", "")
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v
        tot[key][0] += 1
        tot[key][1] += ms
    ours = sum(v[1] for k, v in tot.items() if not k.startswith("other"))
    out = {"command": sys.argv[2] if len(sys.argv) > 2 else None,
           "note": "cold-cache, serialised launches under ncu: compare kernel SHARES of the step, not absolute times",
           "per_kernel": {k: {"launches": n, "total_ms": round(ms, 4),
                              "share_of_ours": None if k.startswith("other") else round(ms / ours, 4)}
                          for k, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
