export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 500 -p no:cacheprovider -k "degree_groups" 2>&1 | grep -E "^FAILED|AssertionError|passed|failed" | head -12
for Y in 1 0; do echo "ywhole=$Y"; TPO_GTP_SPLIT_YWHOLE=$Y TPO_GRID_VERBOSE=1 timeout -s KILL 900 python tools/c5_sweep.py 13,14,15 gtp_grid,gtp_fourier 2>&1 | grep -E "^\{|split" | grep -v "^\[tpo\] gtp_fourier" | tail -12; done
