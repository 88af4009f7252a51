#!/bin/bash
# round-2 GPU session: full parity suite, smoke, every bench workload (+ reference arm), backward table
export PYTHONUNBUFFERED=1
cd "$(dirname "$0")/.."
D=gpurun_out/${TAG:-r02f}; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv | tee $D/nvsmi.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > $D/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" $D/pytest_gpu.log | tail -5
cp gpurun_out/precision_table.json gpurun_out/equivariance_large.json $D/ 2>/dev/null
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for w in c2 c3 c4 c5; do
  steps=20; warm=5; [ $w = c5 ] && steps=2 && warm=3; [ $w = c4 ] && steps=5 && warm=3
  timeout -s KILL 900 python bench.py --workload $w --steps $steps --warmup $warm > $D/bench_$w.log 2>&1
  tail -1 $D/bench_$w.log > $D/bench_$w.json; echo "$w: $(head -c 400 $D/bench_$w.json)"
done
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/ref_c2.log 2>&1; tail -1 $D/ref_c2.log > $D/ref_c2.json
echo "ref: $(head -c 300 $D/ref_c2.json)"
timeout -s KILL 600 python tools/bwd_timing.py --Ls 1,2,3,4,5,6,8,10 > $D/bwd_timing.jsonl 2>&1; tail -3 $D/bwd_timing.jsonl
