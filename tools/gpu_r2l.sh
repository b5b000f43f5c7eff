for r in 1 2; do for L in expbuild/libqs_orig.so expbuild/libqs_grouped.so; do
  echo "lib=$L"; QS_LIBQS=$PWD/$L timeout 300 python tools/one_pair.py --config 4 --refs --reps 5 2>&1 | grep -E "me_box"
done; done
