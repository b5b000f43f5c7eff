# measurement: the interior grid's per-CTA quarter-mask check (expbuild/libqs_nomask.so skips it)
EXP=$PWD/expbuild/libqs_nomask.so
for i in 1 2 3; do
  echo "c4 base:"; timeout 300 python tools/one_pair.py --config 4 --refs --reps 10 | grep -E "me_box"
  echo "c4 nomask:"; QS_LIBQS=$EXP timeout 300 python tools/one_pair.py --config 4 --refs --reps 10 | grep -E "me_box"
done
