#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/ -x -q -m gpu -k "mtp" 2>&1 | tail -2
timeout 600 python tools/bwd_timing.py --kinds mtp --Ls 2,3,4,5,6
