# Round 2: bbox ref staging in the epilogue -- full GPU suite + per-config bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_s.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_s.log
for C in 3 5 4; do timeout 900 python bench.py --config $C --steps 5 --frames 10 --no-cpu-baseline --no-compare > /tmp/b.json 2>/dev/null; python -c "import json; d=json.load(open('/tmp/b.json')); print('c$C', d['value'], d['kernel_ms_per_step'])"; done
