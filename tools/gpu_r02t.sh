#!/bin/bash
# separable Fourier kernel + row-quad thread count: parity, timing
cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "simt or separable or fourier" -x -q 2>&1 | tail -5
timeout 300 python tools/grid_quad_timing.py 8,10,11,12,13,14,15,16 sep,auto gtp_fourier > gpurun_out/gq_fourier.jsonl 2>&1; cat gpurun_out/gq_fourier.jsonl
timeout 300 python tools/grid_quad_timing.py 10,12,13,14,15,16 simt gtp_grid > gpurun_out/gq_grid2.jsonl 2>&1; cat gpurun_out/gq_grid2.jsonl
timeout 1200 python -m pytest tests/test_gpu_backward.py tests/test_gpu_parity_scale.py -k "simt or separable or adversarial or strict or high_L or degree_groups" -x -q 2>&1 | tail -5
