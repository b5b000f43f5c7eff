# integer u8 interior body: parity (u8 tests) and the timing comparison against the fp32 body
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "not f32 and not config4" > gpurun_out/pytest_u8.log 2>&1; echo "pytest u8 rc=$?"; tail -5 gpurun_out/pytest_u8.log
for C in 3 5; do
  for B in int float; do
    QS_U8_BODY=$B timeout 900 python bench.py --config $C --steps 5 --warmup 3 --frames 12 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_c${C}_$B.json 2> gpurun_out/bench_c${C}_$B.err; echo "bench c$C $B rc=$?"
    python -c "import json; d=json.load(open('gpurun_out/bench_c${C}_$B.json')); print('c$C $B', d['value'], d['ms_per_step'], d['kernel_ms_per_step'])"
  done
done
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['kernel_ms_per_step'])"
