# Build an experiment variant of libqs.so: bash tools/build_exp.sh N  ->  exp/libqs_expN.so (-DQS_EXP=N)
set -e
mkdir -p exp
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -Xptxas -v -DQS_EXP=$1 -o exp/libqs_exp$1.so paper_2203_09200_b200/csrc/*.cu > exp/build_exp$1.log 2>&1 || { grep -i error exp/build_exp$1.log | head; exit 1; }
grep -A1 "box_kernelILi8ELb0ELb0ELb0" exp/build_exp$1.log | grep -o "Used [0-9]* registers.*" | head -2
