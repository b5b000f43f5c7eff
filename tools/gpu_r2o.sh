mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -k "f32 or config4 or quad or adjacent or projection or refs" > gpurun_out/pytest_f.log 2>&1; echo "pytest f rc=$?"; tail -3 gpurun_out/pytest_f.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_o_c4.json 2> gpurun_out/bench_o_c4.err; python -c "import json; d=json.load(open('gpurun_out/bench_o_c4.json')); print('c4', d['value'], d['ms_per_step'], d['kernel_ms_per_step']['me_box'], d['kernel_ms_per_step']['epilogue'], d['certify'])"
