# A/B/n: parity subset on each experimental build, then alternating one-launch timings (config 4, 3 refs)
#   bash tools/gpu_abn.sh "pytest -k expression" NAME1 NAME2 ...
mkdir -p gpurun_out
K=$1; shift
for N in "$@"; do
  QS_LIBQS=$PWD/expbuild/libqs_$N.so timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/ab_${N}_pytest.log 2>&1; echo "pytest($N) rc=$?"; tail -1 gpurun_out/ab_${N}_pytest.log
done
for i in 1 2 3; do
  echo "base:"; timeout 300 python tools/one_pair.py --refs --reps 10 | grep -E "me_box|epilogue"
  for N in "$@"; do echo "$N:"; QS_LIBQS=$PWD/expbuild/libqs_$N.so timeout 300 python tools/one_pair.py --refs --reps 10 | grep -E "me_box|epilogue"; done
done
