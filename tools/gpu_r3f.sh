# uint8 border support runs in the single me_box kernel (expbuild/libqs_u8runs.so) against the product build.
mkdir -p gpurun_out
EXP=$PWD/expbuild/libqs_u8runs.so
QS_LIBQS=$EXP timeout 1500 python -m pytest tests -m gpu -x -q -k "u8 or config1 or config2 or fullsize_u8 or row_bands or refs or quad or fuzz or staging or adjacent or projection" > gpurun_out/r3f_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3f_pytest.log
for c in 3 5 2; do
  for i in 1 2 3; do
    echo "c$c base:"; timeout 300 python tools/one_pair.py --config $c --refs --reps 10 | grep -E "me_box"
    echo "c$c u8runs:"; QS_LIBQS=$EXP timeout 300 python tools/one_pair.py --config $c --refs --reps 10 | grep -E "me_box"
  done
done
