# Round-2 (second session) measurement: full GPU suite, smoke, bench lines for every config, the
# reference arm, CC variants, the launch list of the bench command, ncu captures + steady-state traffic.
mkdir -p gpurun_out/final
O=gpurun_out/final
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err; echo "ref rc=$?"
for C in 1 2 3; do timeout 900 python bench.py --config $C --steps 10 --frames 12 > $O/bench_c$C.json 2> $O/bench_c$C.err; echo "bench c$C rc=$?"; done
timeout 1200 python bench.py --config 5 --steps 5 --frames 10 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"
timeout 1200 python bench.py --config 5 --sequences --steps 5 --frames 10 --no-cpu-baseline --no-e2e > $O/bench_c5_seq.json 2> $O/bench_c5_seq.err; echo "bench c5 seq rc=$?"
timeout 1200 python bench.py --variants --steps 5 --no-cpu-baseline --no-e2e --no-compare > $O/bench_variants.json 2> $O/bench_variants.err; echo "variants rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:epilogue -s 1 -c 1 -o $O/epi_full -f python tools/one_pair.py --refs --reps 2 > $O/ncu_epi.log 2>&1; echo "ncu epi rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:box_kernel -s 1 -c 1 -o $O/box_full -f python tools/one_pair.py --refs --reps 2 > $O/ncu_box.log 2>&1; echo "ncu box rc=$?"
python - <<'PY'
import json
for n in ("c4","c1","c2","c3","c5","c5_seq","variants","ref_c4"):
    try:
        d=json.load(open(f"gpurun_out/final/bench_{n}.json"))
        print(n, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("kernel_ms_per_step"))
    except Exception as e:
        print(n, "ERR", e)
PY
