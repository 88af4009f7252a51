# round-2 bench lines for every BASELINE config (c2 headline with CPU baselines + extras, the reference arm,
# c3, c4 strong-scaling shape at N=1, c5 per-GPU shard) and a gloo plan-only N=2 run
export PYTHONUNBUFFERED=1
D=gpurun_out/${TAG:-r02h}; mkdir -p $D
nproc > $D/nproc.txt
timeout -s KILL 600 python bench.py > $D/bench_c2.log 2>&1; echo "c2 rc=$?"; tail -c 600 $D/bench_c2.log; echo
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 1 > $D/ref_c2.log 2>&1; echo "ref rc=$?"; tail -c 300 $D/ref_c2.log; echo
timeout -s KILL 400 python bench.py --workload c3 --no-cpu-baseline > $D/bench_c3.log 2>&1; echo "c3 rc=$?"; tail -c 300 $D/bench_c3.log; echo
timeout -s KILL 600 python bench.py --workload c4 --steps 5 --warmup 3 > $D/bench_c4.log 2>&1; echo "c4 rc=$?"; tail -c 600 $D/bench_c4.log; echo
timeout -s KILL 1200 python bench.py --workload c5 --steps 2 --warmup 3 --cpu-seconds 0.5 > $D/bench_c5.log 2>&1; echo "c5 rc=$?"; tail -c 600 $D/bench_c5.log; echo
