export PYTHONUNBUFFERED=1
TPO_VERBOSE=1 timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 300 -p no:cacheprovider -k "cgtp" 2>&1 | grep -v "^\[tpo\] cgtp tcgen05 L=([0-9]," | tail -12
timeout -s KILL 600 python tools/c5_sweep.py 10,11,12,13,14,15,16 cgtp 2>&1 | tail -8
