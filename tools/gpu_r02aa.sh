#!/bin/bash
# row-quad kernel vs tcgen05 at L = 8..12 (threshold), + ncu of L = 16
cd /root/repo
D=gpurun_out/r02aa; mkdir -p $D
timeout 300 python tools/grid_quad_timing.py 8,9,10,11,12 simt,auto gtp_grid > $D/thr.jsonl 2>&1
timeout 300 python tools/grid_quad_timing.py 8,9,10,11,12 sep,auto gtp_fourier >> $D/thr.jsonl 2>&1
cat $D/thr.jsonl
timeout -s KILL 500 ncu --set full --clock-control none --import-source on -k regex:grid_quad -s 2 -c 1 \
    -o $D/quad_L16_v4 python tools/profile_kernel.py --kind gtp_grid --L 16 --batch 65536 > $D/ncu.log 2>&1
echo ncu rc=$?
