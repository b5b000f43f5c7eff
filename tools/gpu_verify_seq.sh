# Sequence-scale verification on one B200: bash tools/gpu_verify_seq.sh [configs]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/verify_build.log 2>&1
nproc > gpurun_out/verify_host.txt; lscpu | grep "Model name" >> gpurun_out/verify_host.txt
QS_VERIFY_SEQ=${1:-1,2,3,4,5} QS_VERIFY_OUT=gpurun_out/verify_seq.json timeout 3000 \
  python -m pytest tests/test_sequence_verify.py -m gpu -q -rA > gpurun_out/verify_seq_pytest.log 2>&1
echo "verify rc=$?"; tail -5 gpurun_out/verify_seq_pytest.log
