# Build a measurement variant of libqs.so: bash tools/build_exp.sh NAME "-DMACRO=V ..."
#   -> expbuild/libqs_NAME.so (load with QS_LIBQS=$PWD/expbuild/libqs_NAME.so); not part of the product
set -e
mkdir -p expbuild
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -Xptxas -v $2 -o expbuild/libqs_$1.so paper_2203_09200_b200/csrc/*.cu > expbuild/build_$1.log 2>&1 || { grep -i error expbuild/build_$1.log | head; exit 1; }
echo built expbuild/libqs_$1.so
