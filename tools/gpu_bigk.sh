export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -q -rf --timeout 300 -p no:cacheprovider -k "tcgen05 or weighted or fourier or equivar or backward" 2>&1 | tail -4
timeout -s KILL 300 python tools/c5_sweep.py 10,11 gtp_grid,gtp_fourier 2>&1 | tail -12
