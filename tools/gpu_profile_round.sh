# Round measurement: full bench line (ours + reference arm), launch list of the bench command,
# full ncu captures of the two dominant kernels, clocks.  Outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
kill $SMI
cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:box_kernel -s 1 -c 1 -o gpurun_out/me_box_full -f python tools/one_pair.py --refs --reps 2 > gpurun_out/ncu_box.log 2>&1; echo "ncu box rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:epilogue -s 1 -c 1 -o gpurun_out/epi_full -f python tools/one_pair.py --refs --reps 2 > gpurun_out/ncu_epi.log 2>&1; echo "ncu epi rc=$?"
