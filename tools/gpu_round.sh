# one GPU session: kernel parity/timing sweep, pytest -m gpu, smoke, bench
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
python tools/gpu_debug.py grid 2>&1 | tee gpurun_out/debug_grid.log
timeout -s KILL 700 python -m pytest tests -m gpu -q -rf --timeout 240 --timeout-method=thread -p no:cacheprovider \
    2>&1 | tee gpurun_out/pytest_gpu.log | tail -40
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout -s KILL 400 python bench.py --steps 5 --warmup 3 2>&1 | tee gpurun_out/bench.log | tail -3
