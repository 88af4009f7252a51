#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q -k cgtp 2>&1 | tail -2
for i in 1 2; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgtp_bwd_tc --csv python tools/profile_cgtp_bwd.py 6 2>&1 | grep -o '"gpu__time_duration.sum","[^"]*","[^"]*"' | tail -1; done
timeout 300 python tools/bwd_timing.py --kinds cgtp --Ls 4,6,7
