export PYTHONUNBUFFERED=1
TPO_GRID_VERBOSE=1 timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 300 -p no:cacheprovider -k "tcgen05" 2>&1 | grep -E "passed|failed|FAILED|L=12|G=1225|G=1250" | tail -8
TPO_GRID_VERBOSE=1 timeout -s KILL 300 python tools/c5_sweep.py 11,12 gtp_grid,gtp_fourier 2>&1 | tail -8
