#!/bin/bash
cd "$(dirname "$0")/.."
for sl in 30 36 40 45; do for k in gtp_grid gtp_fourier; do for L in 11 12; do echo "seg=$sl $k L=$L $(TPO_GRID_SEG_SLICES=$sl timeout 60 python tools/grid_time.py $k $L 2>&1 | grep -o '"ms": [0-9.]*')"; done; done; done
for sl in 36 40 45; do TPO_GRID_SEG_SLICES=$sl timeout 600 python -m pytest tests/test_gpu_parity_scale.py -q -x -k "adversarial and gtp and (11 or 12)" 2>&1 | tail -1; done
