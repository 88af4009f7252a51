#!/bin/bash
# row-quad separable grid kernel: parity, then timing against the old SIMT kernel and tcgen05
cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "grid_simt" -x -q 2>&1 | tail -5
timeout 300 python tools/grid_quad_timing.py > gpurun_out/gq_new.jsonl 2>&1; cat gpurun_out/gq_new.jsonl
TPO_GRID_SIMT_OLD=1 timeout 300 python tools/grid_quad_timing.py 12,14,15,16 simt > gpurun_out/gq_old.jsonl 2>&1; cat gpurun_out/gq_old.jsonl
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_parity_scale.py -k "simt or (adversarial and grid) or strict" -x -q 2>&1 | tail -5
