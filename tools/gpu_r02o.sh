#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q -k cgtp 2>&1 | tail -3
timeout 300 python tools/bwd_timing.py --kinds cgtp --Ls 3,4,5,6
TPO_CGTP_BWD_PROF=1 timeout 120 python tools/profile_cgtp_bwd.py 6 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgtp_bwd --csv python tools/profile_cgtp_bwd.py 6 2>/dev/null | grep -o '"gpu__time_duration.sum","[^"]*","[^"]*"' | tail -2
TPO_CGTP_BWD_PROF=1 timeout 120 python tools/profile_cgtp_bwd.py 6 2>&1 | tail -1
