# same-box A/B of several library builds on the c2 sweep: LIBS="r01 A B C" (tools/ab/libtpo_<name>.so)
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for lib in ${LIBS:-r01 A}; do
  export TPO_LIB_PATH=$PWD/tools/ab/libtpo_$lib.so
  timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-parity > /tmp/b_$lib.log 2>&1
  python -c "
import json,sys; d=json.loads([x for x in open('/tmp/b_$lib.log') if x.startswith('{')][-1]); print('$lib', round(d['value']/1e6,1), [round(v['ms'],4) for v in d['per_kind_L'].values()])"
done
done
