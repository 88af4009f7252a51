# round 2: parity suite + precision table + segment-cost A/B on the c2 sweep
export PYTHONUNBUFFERED=1
D=gpurun_out/${TAG:-r02b}; mkdir -p $D
timeout -s KILL 1200 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider -k "${TESTK:-}" > $D/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" $D/pytest_gpu.log | tail -40
cp gpurun_out/precision_table.json $D/ 2>/dev/null
for seg in 20 1000; do
  TPO_GRID_SEG_SLICES=$seg timeout -s KILL 400 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-parity > $D/bench_seg$seg.log 2>&1
  python - $D/bench_seg$seg.log <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(open(sys.argv[1]).read()[-2000:]); sys.exit()
d = json.loads(l[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['per_kind_L'].items()}, d['roofline']['frac'])
PY
done
