for L in "" expbuild/libqs_skipborder.so expbuild/libqs_skipinterior.so; do
  for C in 4 5; do
    echo "lib=${L:-product} config=$C"; QS_LIBQS=${L:+$PWD/$L} timeout 300 python tools/one_pair.py --config $C --refs --reps 3 2>&1 | grep -E "me_box|epilogue"
  done
done
