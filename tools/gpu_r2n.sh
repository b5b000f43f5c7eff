mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -k "not f32 and not config4" > gpurun_out/pytest_u8.log 2>&1; echo "pytest u8 rc=$?"; tail -3 gpurun_out/pytest_u8.log
for C in 3 5; do timeout 900 python bench.py --config $C --steps 6 --frames 12 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_n_c$C.json 2> gpurun_out/bench_n_c$C.err; python -c "import json; d=json.load(open('gpurun_out/bench_n_c$C.json')); print('c$C', d['value'], d['ms_per_step'], d['kernel_ms_per_step']['me_box'], d['kernel_ms_per_step']['epilogue'])"; done
