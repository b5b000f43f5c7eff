# ncu capture of the dominant kernels on one config-4 pair (tools/one_pair.py), plus ALU issue peaks.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/alu_peaks tools/alu_peaks.cu && ./gpurun_out/alu_peaks > gpurun_out/alu_peaks.txt 2>&1
timeout 300 python tools/one_pair.py --reps 3 > gpurun_out/one_pair.txt 2>&1; echo "one_pair rc=$?"
cat gpurun_out/one_pair.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:box_kernel -s 1 -c 1 -o gpurun_out/me_box_full -f python tools/one_pair.py --reps 2 > gpurun_out/ncu_box.log 2>&1; echo "ncu box rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:epilogue -s 1 -c 1 -o gpurun_out/epi_full -f python tools/one_pair.py --reps 2 > gpurun_out/ncu_epi.log 2>&1; echo "ncu epi rc=$?"
