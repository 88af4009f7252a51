#!/bin/bash
# MTP SIMT with the k-split matmul: timing + parity; separable unequal-degree tests
cd /root/repo
D=gpurun_out/r02ae; mkdir -p $D
timeout 300 python tools/mtp_simt_timing.py > $D/mtp_ksplit.txt 2>&1; cat $D/mtp_ksplit.txt
timeout 300 python tools/c5_sweep.py 7,8,9,10,11,12,13,14,15,16 mtp > $D/mtp_c5.jsonl 2>&1; cut -c1-160 $D/mtp_c5.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py tests/test_gpu_backward.py -k "mtp or separable_auto" -x -q 2>&1 | tail -2
