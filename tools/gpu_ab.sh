# A/B of an experimental build against the product build on one box:
#   bash tools/gpu_ab.sh NAME [pytest -k expression]
# parity subset on expbuild/libqs_NAME.so, then alternating one-pair timings (config 4, three references).
mkdir -p gpurun_out
EXP=$PWD/expbuild/libqs_$1.so
K=${2:-"quad or f32_me_bit_exact or refs_u8 or bench_launch_sampled or exact_ties"}
QS_LIBQS=$EXP timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/ab_$1_pytest.log 2>&1; echo "pytest($1) rc=$?"; tail -2 gpurun_out/ab_$1_pytest.log
for i in 1 2 3; do
  echo "base:"; timeout 300 python tools/one_pair.py --refs --reps 10 ${3:-} | grep -E "me_box|epilogue|certify"
  echo "$1:"; QS_LIBQS=$EXP timeout 300 python tools/one_pair.py --refs --reps 10 ${3:-} | grep -E "me_box|epilogue|certify"
done
