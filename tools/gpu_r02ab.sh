#!/bin/bash
# MTP SIMT: 8-deep term prefetch A/B; MTP parity
cd /root/repo
D=gpurun_out/r02ab; mkdir -p $D
for P in 0 1 0 1; do echo "PF8=$P"; TPO_MTP_PF8=$P timeout 300 python tools/mtp_simt_timing.py; done > $D/mtp_pf8.txt 2>&1
cat $D/mtp_pf8.txt
TPO_MTP_PF8=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -k "mtp" -x -q 2>&1 | tail -2
