#!/bin/bash
# CGTP block kernel TMEM plan A/B: accumulators of 192 columns + 4 P stages vs 224 + 2 (prebuilt .so copies)
cd /root/repo
P=paper_2506_13523_b200/libtpo_b200.so
cp $P /tmp/lib_orig.so
for V in ${VS:-192 224 192 224}; do
  cp lib_cgtp$V.so.tmp $P
  echo "== $V"
  timeout 600 python tools/c5_sweep.py 6,9,10,12,14 cgtp 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: r=json.loads(l); print(r['L'], r['ms'])
    except Exception: pass"
done
cp lib_cgtp${TV:-224}.so.tmp $P
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -k "cgtp" -x -q 2>&1 | tail -2
cp /tmp/lib_orig.so $P
