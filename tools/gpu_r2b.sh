# float parity subset + bench + ALU peaks
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/alu_peaks tools/alu_peaks.cu && ./gpurun_out/alu_peaks 1965 gpurun_out/alu_peaks.json > gpurun_out/alu_peaks.txt 2>&1; cat gpurun_out/alu_peaks.txt
timeout 1500 python -m pytest tests -m gpu -q -x -k "f32 or config4 or quad or adjacent or smoke or refs" > gpurun_out/pytest_f32.log 2>&1; echo "pytest f32 rc=$?"; tail -5 gpurun_out/pytest_f32.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms_per_step'], d['gpu_launches'], d['certify'])"
