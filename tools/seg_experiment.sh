cat > /tmp/t.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2506_13523_b200 as tpo
kind, L = sys.argv[1], int(sys.argv[2])
x = torch.randn(1 << 19, (L+1)**2, device='cuda'); y = torch.randn(1 << 19, (L+1)**2, device='cuda')
for _ in range(3): tpo.run(kind, x, y, L, L, 2*L)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): tpo.run(kind, x, y, L, L, 2*L)
b.record(); b.synchronize()
print(kind, L, "ms", round(a.elapsed_time(b) / 5, 3), flush=True)
PY
for cfg in "SEG=1000" "SEG=20" "SEG=28" "SEG=20 DBG=8" "SEG=28 DBG=8"; do
  eval "export $cfg"; echo "== $cfg"
  for kl in "gtp_fourier 8" "gtp_fourier 10" "gtp_grid 11"; do
    TPO_GRID_SEG_SLICES=$SEG TPO_GRID_MAX_CHAIN=1 TPO_GRID_DBG=${DBG:-0} python /tmp/t.py $kl
  done
  unset DBG
done
