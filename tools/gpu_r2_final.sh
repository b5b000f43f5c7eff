# round-2 measurement: full GPU suite, smoke, bench lines for every config, the reference arm,
# CC variants, the launch list of the bench command, clocks
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err; echo "ref rc=$?"
for C in 1 2 3; do timeout 900 python bench.py --config $C --steps 10 --frames 12 > gpurun_out/bench_c$C.json 2> gpurun_out/bench_c$C.err; echo "bench c$C rc=$?"; done
timeout 1200 python bench.py --config 5 --steps 5 --frames 10 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
timeout 1200 python bench.py --config 5 --sequences --steps 5 --frames 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_seq.json 2> gpurun_out/bench_c5_seq.err; echo "bench c5 seq rc=$?"
timeout 1200 python bench.py --variants --steps 5 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_variants.json 2> gpurun_out/bench_variants.err; echo "variants rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
python - <<'PY'
import json
for n in ("c4","c1","c2","c3","c5","c5_seq","variants","ref_c4"):
    try:
        d=json.load(open(f"gpurun_out/bench_{n}.json"))
        print(n, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"), ((d.get("cpu_baseline") or {}).get("all_cores") or {}).get("value"))
    except Exception as e:
        print(n, "ERR", e)
PY
