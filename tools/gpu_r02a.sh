# round 2: full parity suite (incl. bench-scale + adversarial precision), smoke, short bench
export PYTHONUNBUFFERED=1
D=gpurun_out/r02a; mkdir -p $D
timeout -s KILL 1200 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > $D/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" $D/pytest_gpu.log | tail -30
cp gpurun_out/precision_table.json $D/ 2>/dev/null
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 400 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > $D/bench.log 2>&1; tail -c 1500 $D/bench.log
