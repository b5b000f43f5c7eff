# Round-2 fifth session: re-validate HEAD on a fresh box (tests, smoke, default bench line).
O=gpurun_out/r02e
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
python -c "import json; d=json.load(open('$O/bench_c4.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('e2e',{}).get('value'), d.get('kernel_ms_per_step'))"
