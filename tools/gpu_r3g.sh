mkdir -p gpurun_out/r3g
timeout 1500 python -m pytest tests -m gpu -x -q -k "variants or row_bands or smoke or adjacent or projection_only" > gpurun_out/r3g/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3g/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3g/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3g/bench_c4.json 2> gpurun_out/r3g/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r3g/bench_c4.json
