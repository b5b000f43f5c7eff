mkdir -p gpurun_out
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)
import ctypes
" 
for M in 0 96; do timeout 900 python bench.py --steps 10 --l2-persist-mb $M --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_l2_$M.json 2> gpurun_out/bench_l2_$M.err; python -c "import json; d=json.load(open('gpurun_out/bench_l2_$M.json')); print('l2 $M', d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d['config']['l2_persist_bytes'])"; done
for M in 0 96; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
    -k regex:"box_kernel|epilogue|certify" --csv --log-file gpurun_out/traffic_l2_$M.csv \
    python bench.py --steps 3 --warmup 3 --frames 16 --l2-persist-mb $M --no-e2e --no-cpu-baseline --no-compare > gpurun_out/ncu_traffic_l2_$M.log 2>&1; echo "traffic $M rc=$?"
done
timeout 900 python -m pytest tests -m gpu -q -x -k "refs or projection or adjacent" > gpurun_out/pytest_l2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_l2.log
