#!/bin/bash
# row-quad kernel: register-budget variant (grid and Fourier, L = 10..16), then parity
cd /root/repo
mkdir -p gpurun_out
: > gpurun_out/quad_variants2.jsonl
for V in 0 256 320; do
  for K in gtp_grid gtp_fourier; do
    P=simt; [ $K = gtp_fourier ] && P=sep
    TPO_QUAD_VARIANT=$V timeout 300 python tools/grid_quad_timing.py 10,11,12,13,14,15,16 $P $K 2>/dev/null | sed "s/^{/{\"variant\": $V, /" >> gpurun_out/quad_variants2.jsonl
  done
done
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/quad_variants2.jsonl") if l.startswith("{")]
for r in rows:
    k = "simt" if "simt" in r else "sep"
    print(r["variant"], r["kind"], r["L"], r.get(k))
PY
timeout 900 python -m pytest tests/test_gpu_parity.py -k "simt or separable or fourier" -x -q 2>&1 | tail -3
