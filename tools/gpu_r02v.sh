#!/bin/bash
# full GPU suite + smoke + c5 bench + sanitizers after the separable kernels
export PYTHONUNBUFFERED=1
cd /root/repo
D=gpurun_out/r02v; mkdir -p $D
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > $D/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" $D/pytest_gpu.log | tail -5
cp gpurun_out/precision_table.json $D/ 2>/dev/null
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 900 python bench.py --workload c5 --steps 2 --warmup 3 > $D/bench_c5.log 2>&1
tail -1 $D/bench_c5.log > $D/bench_c5.json; echo "c5: $(head -c 600 $D/bench_c5.json)"
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > $D/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 $D/memcheck.log
timeout -s KILL 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_small.py > $D/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 $D/racecheck.log
