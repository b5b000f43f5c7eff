# Round-2 fifth session, second call: default bench line with roofline.second (epilogue), then the ncu
# launch list of the same command (after the bench has exited 0 without ncu).
O=gpurun_out/r02e
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_b.log 2>&1 || { echo build failed; tail $O/build_b.log; exit 1; }
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
python -c "import json; d=json.load(open('$O/bench_c4.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('second'), d.get('e2e',{}).get('value'))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/launch_shares.py $O/launches.csv "python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare" > $O/launches.json; tail -c 600 $O/launches.json
timeout 600 python bench.py --config 5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --config 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"
