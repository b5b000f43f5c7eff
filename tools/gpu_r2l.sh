QS_LIBQS=$PWD/expbuild/libqs_sts.so timeout 900 python -m pytest tests -m gpu -q -x -k "f32_me_bit_exact or quad_tiles or exact_ties or quad_interior or variants" 2>&1 | tail -2
for r in 1 2; do for L in base sts; do
  echo "lib=$L"; QS_LIBQS=$PWD/expbuild/libqs_$L.so timeout 300 python tools/one_pair.py --config 4 --refs --reps 5 2>&1 | grep -E "me_box"
done; done
