# precision without GEMM-2 segments + in-kernel cycle accounting of the grid kernel (L = 6, 10)
export PYTHONUNBUFFERED=1
D=gpurun_out/r02d; mkdir -p $D
TPO_GRID_SEG_SLICES=1000 timeout -s KILL 900 python -m pytest tests/test_gpu_parity_scale.py -q -rf --timeout 600 -p no:cacheprovider > $D/pytest_noseg.log 2>&1
echo "pytest(noseg) rc=$?"; grep -E "^FAILED|passed|failed" $D/pytest_noseg.log | tail -20
cp gpurun_out/precision_table.json $D/precision_noseg.json
cat > /tmp/prof.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2506_13523_b200 as tpo
for L in (6, 10):
    x = torch.randn(65536, (L+1)**2, device='cuda'); y = torch.randn(65536, (L+1)**2, device='cuda')
    for _ in range(3): tpo.gtp_grid(x, y, L, L, 2*L)
    torch.cuda.synchronize()
    print("L", L, flush=True)
PY
for seg in 1000 20; do
  echo "== seg $seg"; TPO_GRID_SEG_SLICES=$seg TPO_GRID_PROF=1 TPO_GRID_VERBOSE=1 python /tmp/prof.py 2>&1 | grep -E "tpo|^L" | tail -8
done
