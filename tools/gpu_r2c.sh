# profiling round: launch list of the bench, ncu full captures (me_box, epilogue), DRAM traffic with
# --cache-control none in the bench's steady-state loop for configs 4, 3, 5; memcheck
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
for C in 4 3 5; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
    -k regex:"box_kernel|epilogue|certify" --csv --log-file gpurun_out/traffic_c$C.csv \
    python bench.py --config $C --steps 3 --warmup 3 --frames 16 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/ncu_traffic_c$C.log 2>&1; echo "traffic c$C rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:box_kernel -s 1 -c 1 -o gpurun_out/me_box_full -f python tools/one_pair.py --refs --reps 2 > gpurun_out/ncu_box.log 2>&1; echo "ncu box rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:epilogue -s 1 -c 1 -o gpurun_out/epi_full -f python tools/one_pair.py --refs --reps 2 > gpurun_out/ncu_epi.log 2>&1; echo "ncu epi rc=$?"
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_case.py > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/memcheck.log
