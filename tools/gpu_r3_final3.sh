# Round-2 third-session measurement (artefacts kept small: ncu reports are digested on the box, in /tmp).
O=gpurun_out/final4
T=/tmp/ncu_r3
mkdir -p $O $T
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
QS_SPLIT=0 timeout 1200 python bench.py --no-cpu-baseline > $O/bench_c4_split0.json 2> $O/bench_c4_split0.err; echo "bench c4 split0 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4_torchrun1.json 2> $O/bench_c4_torchrun1.err; echo "torchrun rc=$?"
for C in 1 2 3; do timeout 900 python bench.py --config $C --steps 10 --frames 12 > $O/bench_c$C.json 2> $O/bench_c$C.err; echo "bench c$C rc=$?"; done
timeout 1200 python bench.py --config 5 --steps 5 --frames 10 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"
timeout 1200 python bench.py --config 5 --sequences --steps 5 --frames 10 --no-cpu-baseline --no-e2e > $O/bench_c5_seq.json 2> $O/bench_c5_seq.err; echo "bench c5 seq rc=$?"
timeout 1200 python bench.py --variants --steps 5 --no-cpu-baseline --no-e2e --no-compare > $O/bench_variants.json 2> $O/bench_variants.err; echo "variants rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare > $T/ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/launch_shares.py $O/launches.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compare" > $O/launches.json
for C in 4 3 5; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
    -k regex:"box_kernel|epilogue|certify" --csv --log-file $O/traffic_c$C.csv \
    python bench.py --config $C --steps 3 --warmup 3 --frames 16 --no-e2e --no-cpu-baseline --no-compare > $T/ncu_traffic_c$C.log 2>&1; echo "traffic c$C rc=$?"
python tools/traffic_digest.py $O/traffic_c$C.csv $C 3 > $O/me_box_traffic_c$C.json
done
cap() {  # name, config, skip, kernel regex
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$4 -s $3 -c 1 -o $T/$1 -f python tools/one_pair.py --config $2 --refs --reps 2 > $T/$1.log 2>&1; echo "ncu $1 rc=$?"
  python tools/ncu_digest.py $T/$1.ncu-rep > $O/ncu_$1.json
  python tools/ncu_sass_summary.py $T/$1.ncu-rep 12 > $O/ncu_$1_sass.txt
}
cap box_border_c4 4 2 box_kernel
cap box_interior_c4 4 3 box_kernel
cap epilogue_c4 4 1 epilogue
cap box_c3 3 1 box_kernel
cap box_c5 5 1 box_kernel
du -sh $O
