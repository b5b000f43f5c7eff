# ncu source-level captures of the epilogue and me_box (one three-reference launch each, config 4)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:epilogue -s 1 -c 1 -o gpurun_out/epi_r3 -f python tools/one_pair.py --refs --reps 2 > gpurun_out/ncu_epi_r3.log 2>&1; echo "ncu epi rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:box_kernel -s 1 -c 1 -o gpurun_out/box_r3 -f python tools/one_pair.py --refs --reps 2 > gpurun_out/ncu_box_r3.log 2>&1; echo "ncu box rc=$?"
ls -la gpurun_out/*.ncu-rep
