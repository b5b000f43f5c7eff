# Copy the round's GPU evidence from gpurun_out/ into profiles/ (run here, after tools/gpu_profile_round.sh).
set -e
R=${1:-r01}
cp gpurun_out/bench.json profiles/bench_$R.json
cp gpurun_out/bench_ref.json profiles/bench_ref_$R.json
cp gpurun_out/launches.csv profiles/launches_$R.csv
python tools/launch_shares.py gpurun_out/launches.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare" > profiles/launches_$R.json
python tools/ncu_digest.py gpurun_out/me_box_full.ncu-rep > profiles/ncu_me_box_$R.json
python tools/ncu_digest.py gpurun_out/epi_full.ncu-rep > profiles/ncu_epilogue_$R.json
python tools/ncu_sass_summary.py gpurun_out/me_box_full.ncu-rep 12 > profiles/ncu_me_box_${R}_sass.txt
python tools/ncu_sass_summary.py gpurun_out/epi_full.ncu-rep 12 > profiles/ncu_epilogue_${R}_sass.txt
python - <<PY
import json
d = json.load(open("profiles/ncu_me_box_$R.json"))
def b(x):
    u = x["unit"]; v = float(x["value"])
    return int(v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u])
t = {"kernel": "box_kernel<8,false,false,false> (me_box, config-4 launch of qs_me_search_refs: 1920x1080, S=24, three f32 references)",
     "source": "ncu --set full --clock-control none on tools/one_pair.py --refs (config 4, t=3, d=1..3); digest profiles/ncu_me_box_$R.json",
     "dram_bytes_read": b(d["dram__bytes_read.sum"]), "dram_bytes_write": b(d["dram__bytes_write.sum"]),
     "algorithmic_input_bytes": 4147200 + 3 * 8294400,
     "note": "inputs: cur u8 2.07 MB + mask u8 2.07 MB + 3 x ref f32 8.29 MB = 29.0 MB; the rest is the 3 x 16.6 MB key planes (8 B/pixel) read back by the 64-bit atomicMin merges after the memset; writes stay in L2 (126 MB)."}
t["dram_bytes_per_launch"] = t["dram_bytes_read"] + t["dram_bytes_write"]
json.dump(t, open("profiles/me_box_traffic.json", "w"), indent=1)
print("traffic", t["dram_bytes_per_launch"])
PY
