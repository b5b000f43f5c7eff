# Round-2 third session: full GPU suite on the default build (float me_box split into border / interior
# kernels), A/B timing against QS_SPLIT=0, bench config 4, and launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3c_build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3c_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3c_pytest.log
for i in 1 2 3; do
  echo "c4 split:"; timeout 300 python tools/one_pair.py --config 4 --refs --reps 10 | grep -E "me_box|epilogue|certify"
  echo "c4 single:"; QS_SPLIT=0 timeout 300 python tools/one_pair.py --config 4 --refs --reps 10 | grep -E "me_box|epilogue|certify"
done
timeout 600 python bench.py > gpurun_out/r3c_bench_c4.json 2> gpurun_out/r3c_bench_c4.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r3c_bench_c4.json
