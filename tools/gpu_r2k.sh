mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "f32 or quad or adjacent or projection or refs" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d['certify'])"
