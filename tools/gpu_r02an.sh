#!/bin/bash
# CGTP block kernel: per-block y staging threshold (TPO_CGTP_YSEG_MIN) at L = 9..12
cd /root/repo
for Y in 196 100 196 100; do
  echo "== YSEG_MIN=$Y"
  TPO_CGTP_YSEG_MIN=$Y timeout 600 python tools/c5_sweep.py 8,9,10,11,12 cgtp 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: r=json.loads(l); print(r['L'], r['ms'])
    except Exception: pass"
done
TPO_CGTP_YSEG_MIN=64 timeout 900 python -m pytest tests/test_gpu_parity.py -k "cgtp_tensor_cores" -x -q 2>&1 | tail -1
