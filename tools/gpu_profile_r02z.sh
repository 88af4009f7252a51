#!/bin/bash
export PYTHONUNBUFFERED=1
cd /root/repo
T=gpurun_out/r02z; mkdir -p $T
timeout -s KILL 500 ncu --set full --clock-control none --import-source on -k regex:grid_quad -s 2 -c 1 \
    -o $T/quad_L16_v2 python tools/profile_kernel.py --kind gtp_grid --L 16 --batch 65536 > $T/ncu.log 2>&1
echo rc=$?
