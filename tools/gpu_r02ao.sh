#!/bin/bash
# final ncu launch lists (gpu__time_duration per launch) of the default bench (c2) and of c5
export PYTHONUNBUFFERED=1
cd /root/repo
T=gpurun_out/r02ao; mkdir -p $T
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $T/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-graph --no-parity \
  > $T/bench_c2_under_ncu.log 2>&1; echo "c2 rc=$?"
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $T/launches_c5.csv python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline --no-extras --no-graph --no-parity \
  > $T/bench_c5_under_ncu.log 2>&1; echo "c5 rc=$?"
ls -la $T
