# Round-2 third-session measurement: full GPU suite, smoke, bench lines for every config, the reference
# arm, CC variants, torchrun N=1, the launch list, ncu full captures (c4 border / interior me_box grids,
# epilogue; c3 / c5 me_box for the pipe roofline), steady-state DRAM traffic per config.
O=gpurun_out/final3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt; nvidia-smi -q -d CLOCK | grep -A3 "Max Clocks" >> $O/host.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
QS_SPLIT=0 timeout 1200 python bench.py --no-cpu-baseline > $O/bench_c4_split0.json 2> $O/bench_c4_split0.err; echo "bench c4 split0 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4_torchrun1.json 2> $O/bench_c4_torchrun1.err; echo "torchrun rc=$?"
for C in 1 2 3; do timeout 900 python bench.py --config $C --steps 10 --frames 12 > $O/bench_c$C.json 2> $O/bench_c$C.err; echo "bench c$C rc=$?"; done
timeout 1200 python bench.py --config 5 --steps 5 --frames 10 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"
timeout 1200 python bench.py --config 5 --sequences --steps 5 --frames 10 --no-cpu-baseline --no-e2e > $O/bench_c5_seq.json 2> $O/bench_c5_seq.err; echo "bench c5 seq rc=$?"
timeout 1200 python bench.py --variants --steps 5 --no-cpu-baseline --no-e2e --no-compare > $O/bench_variants.json 2> $O/bench_variants.err; echo "variants rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
for C in 4 3 5; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
    -k regex:"box_kernel|epilogue|certify" --csv --log-file $O/traffic_c$C.csv \
    python bench.py --config $C --steps 3 --warmup 3 --frames 16 --no-e2e --no-cpu-baseline --no-compare > $O/ncu_traffic_c$C.log 2>&1; echo "traffic c$C rc=$?"
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:box_kernel -s 2 -c 2 -o $O/box_full -f python tools/one_pair.py --refs --reps 2 > $O/ncu_box.log 2>&1; echo "ncu box rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:epilogue -s 1 -c 1 -o $O/epi_full -f python tools/one_pair.py --refs --reps 2 > $O/ncu_epi.log 2>&1; echo "ncu epi rc=$?"
for C in 3 5; do
timeout 1200 ncu --set full --clock-control none -k regex:box_kernel -s 1 -c 1 -o $O/box_full_c$C -f python tools/one_pair.py --config $C --refs --reps 2 > $O/ncu_box_c$C.log 2>&1; echo "ncu box c$C rc=$?"
done
python - <<'PY'
import json
for n in ("c4","c4_split0","c4_torchrun1","c1","c2","c3","c5","c5_seq","variants","ref_c4"):
    try:
        d=json.loads(open(f"gpurun_out/final3/bench_{n}.json").read().strip().split("\n")[-1])
        print(n, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("kernel_ms_per_step"))
    except Exception as e:
        print(n, "ERR", e)
PY
