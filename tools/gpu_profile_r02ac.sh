#!/bin/bash
export PYTHONUNBUFFERED=1
cd /root/repo
T=gpurun_out/r02ac; mkdir -p $T
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:cgtp_tc -s 1 -c 1 \
    -o $T/cgtp_L16 python tools/profile_kernel.py --kind cgtp --L 16 --batch 2048 --reps 2 > $T/ncu16.log 2>&1
echo rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:cgtp_tc -s 1 -c 1 \
    -o $T/cgtp_L10 python tools/profile_kernel.py --kind cgtp --L 10 --batch 16384 --reps 2 > $T/ncu10.log 2>&1
echo rc=$?
