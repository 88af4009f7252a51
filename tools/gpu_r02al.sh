#!/bin/bash
# MTP SIMT: extract grouped by order (default) vs per-output term lists (TPO_MTP_XG=0)
cd /root/repo
for X in 0 1 0 1; do echo "XG=$X"; TPO_MTP_XG=$X timeout 300 python tools/mtp_simt_timing.py; done 2>&1
for X in 0 1; do TPO_MTP_XG=$X timeout 300 python tools/c5_sweep.py 7,9,12,14,16 mtp 2>&1 | cut -c1-100 | sed "s/^/XG=$X /"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py tests/test_gpu_backward.py tests/test_gpu_stages.py -k "mtp" -x -q 2>&1 | tail -2
