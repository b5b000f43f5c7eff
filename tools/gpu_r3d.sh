mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3d_build.log 2>&1 || { echo build failed; exit 1; }
QS_SPLIT=2 timeout 900 python -m pytest tests -m gpu -x -q -k "f32 or config4" > gpurun_out/r3d_pytest.log 2>&1; echo "pytest(split=2) rc=$?"; tail -1 gpurun_out/r3d_pytest.log
for i in 1 2 3; do
  for m in 0 1 2; do echo "c4 split=$m:"; QS_SPLIT=$m timeout 300 python tools/one_pair.py --config 4 --refs --reps 10 | grep -E "me_box"; done
done
