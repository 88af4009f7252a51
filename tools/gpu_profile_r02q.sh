#!/bin/bash
# final round-2 ncu evidence: c2 launch list, full captures of the kernels changed late in the round
export PYTHONUNBUFFERED=1
cd "$(dirname "$0")/.."
T=gpurun_out/r02q; mkdir -p $T
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $T/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --no-graph --no-parity \
  > $T/bench_under_ncu.log 2>&1
cap() {  # name regex skip count script args...
  name=$1; rx=$2; sk=$3; c=$4; shift 4
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:$rx -s $sk -c $c \
    -o $T/$name python "$@" > $T/ncu_$name.log 2>&1
}
cap grid_L10 gtp_grid_tc 2 1 tools/profile_kernel.py --kind gtp_grid --L 10
cap grid_L1_small gtp_small 2 1 tools/profile_kernel.py --kind gtp_grid --L 1
cap cgtp_L6 cgtp_tc 2 1 tools/profile_kernel.py --kind cgtp --L 6
cap mtp_L7_simt mtp_kernel 2 1 tools/profile_kernel.py --kind mtp --L 7
cap cgtp_bwd_L6 cgtp_bwd 4 2 tools/profile_cgtp_bwd.py 6
timeout -s KILL 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100000 python tools/sanitize_small.py > $T/racecheck_full.log 2>&1
echo "racecheck rc=$?"; tail -2 $T/racecheck_full.log
ls -la $T
