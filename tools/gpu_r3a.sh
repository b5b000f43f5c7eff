# Session re-entry check of HEAD: full GPU suite, smoke, default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_a.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_a.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_a.log
timeout 900 python bench.py > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo "bench rc=$?"; cat gpurun_out/bench_a.json | head -c 1500
