#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q -k cgtp 2>&1 | tail -3
timeout 600 python tools/bwd_timing.py --kinds cgtp --Ls 6,7,8
