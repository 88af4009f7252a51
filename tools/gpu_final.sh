# end-of-round GPU session: full parity suite, smoke, bench, backward + C5 sweeps
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/r01i
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 -p no:cacheprovider > gpurun_out/r01i/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r01i/pytest_gpu.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout -s KILL 400 python bench.py --steps 5 --warmup 3 > gpurun_out/r01i/bench.log 2>&1; tail -c 300 gpurun_out/r01i/bench.log
timeout -s KILL 300 python tools/bwd_timing.py > gpurun_out/r01i/bwd_timing.jsonl 2>&1
timeout -s KILL 900 python tools/c5_sweep.py > gpurun_out/r01i/c5_sweep.jsonl 2>&1
tail -3 gpurun_out/r01i/c5_sweep.jsonl
