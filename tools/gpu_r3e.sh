# uint8 border support runs (split kernels for uint8 SAD): GPU parity of the uint8 paths, then alternating
# me_box timings (QS_SPLIT=0: one kernel) for configs 3, 5, 2 and 4.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3e_build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -k "u8 or config1 or config2 or fullsize or row_bands or refs or quad or fuzz or staging or adjacent or projection" > gpurun_out/r3e_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3e_pytest.log
for c in 3 5 2 4; do
  for i in 1 2 3; do
    echo "c$c split:"; timeout 300 python tools/one_pair.py --config $c --refs --reps 10 | grep -E "me_box"
    echo "c$c single:"; QS_SPLIT=0 timeout 300 python tools/one_pair.py --config $c --refs --reps 10 | grep -E "me_box"
  done
done
