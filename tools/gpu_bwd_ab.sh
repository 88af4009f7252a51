export PYTHONUNBUFFERED=1
timeout -s KILL 500 python -m pytest tests/test_gpu_backward.py -q -rf --timeout 300 -p no:cacheprovider 2>&1 | tail -2
python tools/bwd_timing.py --kinds mtp,gtp_grid --Ls 1,2,4,6,8,10
