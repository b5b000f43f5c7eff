#!/usr/bin/env python
"""traffic_digest.py -- per-kernel DRAM bytes of the bench's steady-state loop from an ncu capture
taken with --cache-control none (caches NOT flushed between kernels, so L2 reuse between me_box, certify
and the epilogue counts as reuse) and --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum.  The last `steps` steps are the timed ones (the first are warm-up).
  python tools/traffic_digest.py gpurun_out/traffic_c4.csv 4 3 > profiles/me_box_traffic_c4.json"""
import collections
import csv
import io
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))


def main():
    path, cfg, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    import synth
    c = synth.CONFIGS[cfg]
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    launches = collections.OrderedDict()
    for r in rows:
        key = int(r["ID"])
        name = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
        d = launches.setdefault(key, {"kernel": name})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    seq = list(launches.values())
    # one epilogue launch per step; float references launch me_box as two grids (border, interior)
    n_epi = sum(1 for x in seq if x["kernel"] == "epilogue_kernel")
    n_box = n_epi
    per_step = len(seq) // n_epi
    timed = seq[-steps * per_step:]
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0])
    for x in timed:
        a = agg[x["kernel"]]
        a[0] += x.get("dram__bytes_read.sum", 0.0)
        a[1] += x.get("dram__bytes_write.sum", 0.0)
        a[2] += x.get("gpu__time_duration.sum", 0.0)
        a[3] += 1
    px = c.w * c.h
    esz = 4 if c.ref_f32 else 1
    alg_in = px * (2 + 3 * esz)                         # cur + mask + three references, once
    out = {"config": c.name, "capture": path, "how": "ncu --cache-control none --clock-control none, bench.py steady "
           f"state (last {steps} steps of {n_box}); DRAM bytes per launch (read + write)",
           "algorithmic_input_bytes_per_me_box_launch": alg_in,
           "kernels": {}}
    for k, (rd, wr, t, n) in agg.items():
        out["kernels"][k] = {"launches": n, "dram_read_per_launch": rd / n, "dram_write_per_launch": wr / n,
                             "dram_bytes_per_launch": (rd + wr) / n, "duration_per_launch": t / n}
    bx = out["kernels"].get("box_kernel")
    if bx:   # per me_box call (qs_me_search_refs): every box grid of one step
        per_call = bx["dram_bytes_per_launch"] * bx["launches"] / steps
        out["box_grids_per_call"] = bx["launches"] / steps
        out["dram_bytes_per_launch"] = per_call
        out["me_box_traffic_over_algorithmic_inputs"] = per_call / alg_in
    tot = sum(v["dram_bytes_per_launch"] * v["launches"] for v in out["kernels"].values()) / steps
    out["dram_bytes_per_step_all_kernels"] = tot
    out["per_step_over_algorithmic_inputs_plus_pr_planes"] = tot / (alg_in + 2 * px * esz + 5 * px)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
