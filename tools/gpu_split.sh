export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 300 -p no:cacheprovider -k "degree_groups or simt or fourier or equivar" 2>&1 | tail -4
timeout -s KILL 600 python tools/c5_sweep.py 13,14,15 gtp_grid,gtp_fourier 2>&1 | tail -6
