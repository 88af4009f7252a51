#!/bin/bash
# MTP SIMT: 256-thread blocks (two per SM) vs 512 (one)
cd /root/repo
D=gpurun_out/r02ag; mkdir -p $D
for N in 512 256 512 256; do echo "NT=$N"; TPO_MTP_NT=$N timeout 300 python tools/mtp_simt_timing.py; done > $D/mtp_nt.txt 2>&1; cat $D/mtp_nt.txt
for N in 512 256; do TPO_MTP_NT=$N timeout 300 python tools/c5_sweep.py 7,9,12,14,16 mtp 2>&1 | cut -c1-120 | sed "s/^/NT=$N /"; done
TPO_MTP_NT=256 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -k "mtp" -x -q 2>&1 | tail -2
