# A/B of the grid kernel's accumulation segments / role split on the c2 sweep (+ grid/Fourier parity)
export PYTHONUNBUFFERED=1
D=gpurun_out/${TAG:-r02c}; mkdir -p $D
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider -k "grid or fourier or weighted" > $D/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" $D/pytest_gpu.log | tail -20
cp gpurun_out/precision_table.json $D/ 2>/dev/null
run() {  # name env...
  name=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-parity > $D/bench_$name.log 2>&1
  python - $D/bench_$name.log $name <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-1500:]); sys.exit()
d = json.loads(l[-1])
print(sys.argv[2], round(d['value']/1e6,1), d['ms_per_step'], [round(v['ms'],4) for v in d['per_kind_L'].values()], d['roofline']['frac'])
PY
}
run split_seg20_red TPO_GRID_SPLIT_ROLES=1 TPO_GRID_SEG_SLICES=20 TPO_GRID_SEG_RED=1
run split_noseg TPO_GRID_SPLIT_ROLES=1 TPO_GRID_SEG_SLICES=1000
run nosplit_noseg TPO_GRID_SPLIT_ROLES=0 TPO_GRID_SEG_SLICES=1000
run split_seg20_rmw TPO_GRID_SPLIT_ROLES=1 TPO_GRID_SEG_SLICES=20 TPO_GRID_SEG_RED=0
run split_seg30_red TPO_GRID_SPLIT_ROLES=1 TPO_GRID_SEG_SLICES=30 TPO_GRID_SEG_RED=1
run nosplit_seg20_red TPO_GRID_SPLIT_ROLES=0 TPO_GRID_SEG_SLICES=20 TPO_GRID_SEG_RED=1
