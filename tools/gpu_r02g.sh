# full GPU suite (round 2 state) + smoke + short bench
export PYTHONUNBUFFERED=1
D=gpurun_out/${TAG:-r02g}; mkdir -p $D
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > $D/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "^FAILED|^E  |passed|failed" $D/pytest_gpu.log | head -40
cp gpurun_out/precision_table.json gpurun_out/equivariance_large.json $D/ 2>/dev/null
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
