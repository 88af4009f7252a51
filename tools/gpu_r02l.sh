#!/bin/bash
# CGTP backward on tcgen05: parity + timing vs the SIMT kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02l
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q -k cgtp 2>&1 | tail -15
echo "== tc"
timeout 300 python tools/bwd_timing.py --kinds cgtp --Ls 3,4,5,6 | tee gpurun_out/r02l/bwd_tc.jsonl
echo "== simt"
TPO_CGTP_BWD_TC=0 timeout 300 python tools/bwd_timing.py --kinds cgtp --Ls 3,4,5,6 | tee gpurun_out/r02l/bwd_simt.jsonl
