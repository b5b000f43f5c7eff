mkdir -p gpurun_out
for S in 24 6 9 16; do for M in sad ssd; do QS_TMA=1 QS_LIBQS=libqs_checked.so timeout 120 python tools/tma_debug.py $S $M 2>&1 | tail -1; done; done
QS_TMA=1 timeout 1500 python -m pytest tests -m gpu -q -k "f32 and not full_frame and not row_bands" > gpurun_out/pytest_tma.log 2>&1; echo "pytest tma rc=$?"; tail -3 gpurun_out/pytest_tma.log
timeout 1500 python -m pytest tests -m gpu -q -k "variants or config5" > gpurun_out/pytest_c5.log 2>&1; echo "pytest variants/c5 rc=$?"; tail -3 gpurun_out/pytest_c5.log
