#!/usr/bin/env python
"""Digest of an ncu --set full capture (one kernel launch) as JSON: the numbers DESIGN.md and
bench.py's roofline cite (duration, issue, pipes, shared wavefronts, DRAM bytes, stalls).
  python tools/ncu_digest.py gpurun_out/me_box_full.ncu-rep > profiles/ncu_me_box_rNN.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic",
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    vals = dict(zip(h, zip(v, u)))
    d = {"report": rep, "kernel": vals.get("Kernel Name", ("", ""))[0]}
    for k in KEYS:
        if k in vals:
            d[k] = {"value": vals[k][0], "unit": vals[k][1]}
    stalls = {k.split("issue_stalled_")[1].split("_per_issue")[0]: float(vals[k][0])
              for k in vals if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
    d["stalls_per_issue"] = {k: round(x, 3) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1]) if x > 0.01}
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
