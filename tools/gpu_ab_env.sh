# A/B of an environment switch of the product build on one box:
#   bash tools/gpu_ab_env.sh NAME "VAR=VAL ..." [configs] [pytest -k expression]
# builds libqs.so, runs the GPU parity subset with the switch on, then alternating me_box / epilogue
# timings (qs_me_search_refs, three references) per config with the switch off (base) and on.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_$1_build.log 2>&1 || { echo build failed; tail gpurun_out/ab_$1_build.log; exit 1; }
K=${4:-"quad or f32_me_bit_exact or refs_u8 or bench_launch_sampled or exact_ties or row_bands or adjacent"}
env $2 timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/ab_$1_pytest.log 2>&1; echo "pytest($1) rc=$?"; tail -2 gpurun_out/ab_$1_pytest.log
for c in ${3:-4}; do
  for i in 1 2 3; do
    echo "c$c base:"; timeout 300 python tools/one_pair.py --config $c --refs --reps 10 | grep -E "me_box|epilogue|certify"
    echo "c$c $1:"; env $2 timeout 300 python tools/one_pair.py --config $c --refs --reps 10 | grep -E "me_box|epilogue|certify"
  done
done
