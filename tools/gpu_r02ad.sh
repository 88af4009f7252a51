#!/bin/bash
# grid / Fourier backward: tcgen05 degree groups (auto) vs the swapped-operand forward on the row-quad kernel
cd /root/repo
D=gpurun_out/r02ad; mkdir -p $D
for P in auto simt; do
  timeout 600 python tools/bwd_timing.py --kinds gtp_grid --Ls 4,6,8,10,11,12,13,14,16 --path $P
done > $D/bwd_paths.jsonl 2>&1
cat $D/bwd_paths.jsonl
