# full parity suite + smoke + bench (no sweeps)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/r01l
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 500 -p no:cacheprovider > gpurun_out/r01l/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r01l/pytest_gpu.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 400 python bench.py --steps 5 --warmup 3 > gpurun_out/r01l/bench.log 2>&1; tail -c 200 gpurun_out/r01l/bench.log
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01l/ref.log 2>&1; tail -c 400 gpurun_out/r01l/ref.log
