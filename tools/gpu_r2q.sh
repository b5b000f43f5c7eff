mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['kernel_ms_per_step'], d['gpu_launches'], d['clocks'])"
