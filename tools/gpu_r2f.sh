# TMA staging: parity + timing; projection-only bench; new tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "variants or projection_only or adjacent or smoke or f32_me_bit_exact or quad_tiles" > gpurun_out/pytest_new.log 2>&1; echo "pytest new rc=$?"; tail -4 gpurun_out/pytest_new.log
QS_TMA=1 timeout 1500 python -m pytest tests -m gpu -q -k "f32 and not full_frame and not row_bands" > gpurun_out/pytest_tma.log 2>&1; echo "pytest tma rc=$?"; tail -4 gpurun_out/pytest_tma.log
for T in 0 1; do
QS_TMA=$T timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_c4_tma$T.json 2> gpurun_out/bench_c4_tma$T.err; python -c "import json; d=json.load(open('gpurun_out/bench_c4_tma$T.json')); print('tma$T', d['value'], d['ms_per_step'], d['kernel_ms_per_step'])"
done
QS_TMA=1 timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:box_kernel -s 1 -c 1 python tools/one_pair.py --refs --reps 2 > gpurun_out/ncu_tma1.log 2>&1; tail -8 gpurun_out/ncu_tma1.log
QS_TMA=0 timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:box_kernel -s 1 -c 1 python tools/one_pair.py --refs --reps 2 > gpurun_out/ncu_tma0.log 2>&1; tail -8 gpurun_out/ncu_tma0.log
