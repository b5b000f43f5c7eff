# Bounds-checked build (sanitizer substitute) on HEAD's kernels: the GPU suite and the every-entry-point cases.
O=gpurun_out/r02d
mkdir -p $O
QS_LIBQS=libqs_checked.so timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu_checked.log 2>&1; echo "checked pytest rc=$?"; tail -2 $O/pytest_gpu_checked.log
QS_LIBQS=libqs_checked.so timeout 600 python tools/sanitize_case.py > $O/checked_cases.log 2>&1; echo "checked cases rc=$?"; tail -5 $O/checked_cases.log
