# u8 integer body parity + checked-build run of the GPU suite
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "not f32 and not config4" > gpurun_out/pytest_u8.log 2>&1; echo "pytest u8 rc=$?"; tail -5 gpurun_out/pytest_u8.log
QS_LIBQS=libqs_checked.so timeout 2400 python -m pytest tests -m gpu -q -k "not full_frame" > gpurun_out/pytest_checked.log 2>&1; echo "pytest checked rc=$?"; tail -5 gpurun_out/pytest_checked.log
QS_LIBQS=libqs_checked.so timeout 600 python tools/sanitize_case.py > gpurun_out/checked_cases.log 2>&1; echo "checked cases rc=$?"; tail -4 gpurun_out/checked_cases.log
