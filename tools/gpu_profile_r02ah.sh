#!/bin/bash
# final ncu captures of the separable row-quad kernel (grid L = 16, 11; Fourier L = 16) + sanitizers
export PYTHONUNBUFFERED=1
cd /root/repo
T=gpurun_out/r02ah; mkdir -p $T
cap() { name=$1; shift
  timeout -s KILL 500 ncu --set full --clock-control none --import-source on -k regex:grid_quad -s 2 -c 1 \
    -o $T/$name python tools/profile_kernel.py "$@" > $T/ncu_$name.log 2>&1; echo "$name rc=$?"; }
cap quad_grid_L16 --kind gtp_grid --L 16 --batch 65536
cap quad_grid_L11 --kind gtp_grid --L 11 --batch 65536
cap quad_fourier_L16 --kind gtp_fourier --L 16 --batch 65536
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > $T/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 $T/memcheck.log
timeout -s KILL 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_small.py > $T/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 $T/racecheck.log
