# A/B/C: bash tools/gpu_ab3.sh NAME1 NAME2 -- parity subset on NAME1, then alternating one-pair timings.
mkdir -p gpurun_out
K="quad or f32_me_bit_exact or refs_u8 or bench_launch_sampled or exact_ties"
for N in $1 $2; do
QS_LIBQS=$PWD/expbuild/libqs_$N.so timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/ab_${N}_pytest.log 2>&1; echo "pytest($N) rc=$?"; tail -1 gpurun_out/ab_${N}_pytest.log
done
for i in 1 2 3; do
  echo "base:"; timeout 300 python tools/one_pair.py --refs --reps 10 | grep -E "me_box|certify"
  for N in $1 $2; do echo "$N:"; QS_LIBQS=$PWD/expbuild/libqs_$N.so timeout 300 python tools/one_pair.py --refs --reps 10 | grep -E "me_box|certify"; done
done
