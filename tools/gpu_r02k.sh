# MTP SIMT kernel A/B (round-1 vs current) at L = 7..16, then the full parity suite
export PYTHONUNBUFFERED=1
D=gpurun_out/r02k; mkdir -p $D
for lib in r01 cur; do
  if [ $lib = r01 ]; then export TPO_LIB_PATH=$PWD/tools/ab/libtpo_r01.so; else unset TPO_LIB_PATH; fi
  echo "== $lib"; timeout -s KILL 600 python tools/c5_sweep.py 7,8,10,12,14,16 mtp 2>&1 | tee $D/mtp_$lib.jsonl | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d.get('kind'), d.get('L'), d.get('ms'), d.get('hbm_frac', d.get('roofline_frac')))"
done
unset TPO_LIB_PATH
TAG=r02k bash tools/gpu_r02g.sh
