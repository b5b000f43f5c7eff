# Functional check of bench.py's N > 1 code path on one GPU (gloo backend, ranks share the GPU):
# row bands + halo exchange, max over ranks, rank 0's JSON line.  Not a scaling measurement.
O=gpurun_out/r02d
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_b.log 2>&1 || { echo build failed; exit 1; }
for N in 2 4; do
QS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N \
  bench.py --gpus $N --steps 3 --warmup 3 > $O/bench_gloo_n$N.json 2> $O/bench_gloo_n$N.err; echo "gloo N=$N rc=$?"; tail -c 600 $O/bench_gloo_n$N.json; echo
done
QS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --config 5 --sequences --steps 2 --warmup 3 --frames 8 > $O/bench_gloo_c5seq_n2.json 2> $O/bench_gloo_c5seq_n2.err; echo "gloo c5 seq rc=$?"; tail -c 300 $O/bench_gloo_c5seq_n2.json
