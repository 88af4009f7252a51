#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_parity.py -x -q -k "small or bench_config or adversarial" 2>&1 | tail -3
timeout 300 python tools/grid_small_paths.py 2>&1 | head -2
