# per-shape timing of the segmented grid / Fourier shapes (2^19 products) + their precision tests
cat > /tmp/t.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2506_13523_b200 as tpo
for kind, L in (("gtp_fourier", 7), ("gtp_fourier", 8), ("gtp_fourier", 10), ("gtp_fourier", 12), ("gtp_grid", 10), ("gtp_grid", 11), ("gtp_grid", 12)):
    x = torch.randn(1 << 19, (L+1)**2, device='cuda'); y = torch.randn(1 << 19, (L+1)**2, device='cuda')
    for _ in range(3): tpo.run(kind, x, y, L, L, 2*L)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): tpo.run(kind, x, y, L, L, 2*L)
    b.record(); b.synchronize()
    print(kind, L, "ms", round(a.elapsed_time(b) / 5, 3), flush=True)
PY
python /tmp/t.py
timeout -s KILL 900 python -m pytest tests/test_gpu_parity_scale.py -q -x -k "adversarial and (fourier or grid)" -p no:cacheprovider 2>&1 | tail -2
python - <<'PY'
import json
t = json.load(open('gpurun_out/precision_table.json'))
print({k: round(v['worst'] * 1e6, 2) for k, v in sorted(t.items()) if int(k.split('_L')[1]) >= 6})
PY
