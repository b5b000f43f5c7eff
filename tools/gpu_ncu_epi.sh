mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:epilogue -s 1 -c 1 -o gpurun_out/epi_full -f python tools/one_pair.py --reps 2 > gpurun_out/ncu_epi.log 2>&1; echo "ncu epi rc=$?"
