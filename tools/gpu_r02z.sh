#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q -k cgtp 2>&1 | tail -2
TPO_VERBOSE=1 timeout 600 python tools/bwd_timing.py --kinds cgtp --Ls 3,4,5,6,7 2>&1 | grep -v "^\[tpo\] [^c]"
