# stage API parity + the A/B of round-1 vs current library on the c2 sweep
export PYTHONUNBUFFERED=1
D=gpurun_out/r02f; mkdir -p $D
timeout -s KILL 900 python -m pytest tests/test_gpu_stages.py -q -rf --timeout 600 -p no:cacheprovider > $D/pytest_stages.log 2>&1
echo "pytest rc=$?"; grep -E "^FAILED|^E  |passed|failed" $D/pytest_stages.log | head -30
cp gpurun_out/equivariance_large.json $D/ 2>/dev/null
for lib in r01 cur r01 cur; do
  if [ $lib = r01 ]; then export TPO_LIB_PATH=$PWD/tools/ab/libtpo_r01.so; else unset TPO_LIB_PATH; fi
  timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-parity > $D/bench_$lib.log 2>&1
  python - $D/bench_$lib.log $lib <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-1500:]); sys.exit()
d = json.loads(l[-1])
print(sys.argv[2], round(d['value']/1e6,1), d['ms_per_step'], [round(v['ms'],4) for v in d['per_kind_L'].values()], d['roofline']['frac'])
PY
done
