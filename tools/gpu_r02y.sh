#!/bin/bash
# row-quad kernel: timing per register-budget variant (grid / Fourier, L = 12..16) + parity
cd /root/repo
D=gpurun_out/${TAG:-r02y}; mkdir -p $D
for V in ${VARIANTS:-0 256 320}; do
  TPO_QUAD_VARIANT=$V timeout 300 python tools/grid_quad_timing.py 12,13,14,15,16 simt gtp_grid 2>/dev/null | sed "s/^{/{\"variant\": $V, /"
  TPO_QUAD_VARIANT=$V timeout 300 python tools/grid_quad_timing.py 12,13,14,15,16 sep gtp_fourier 2>/dev/null | sed "s/^{/{\"variant\": $V, /"
done > $D/quad_v2.jsonl
F=$D/quad_v2.jsonl python - <<'PY'
import json, os
for l in open(os.environ["F"]):
    r = json.loads(l); k = "simt" if "simt" in r else "sep"; print(r["variant"], r["kind"], r["L"], r[k])
PY
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -k "simt or separable" -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -k "separable" -x -q 2>&1 | tail -2
