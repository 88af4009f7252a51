"""Grid GTP backward at bench-like batches: the tcgen05 degree-group VJP (auto) against the swapped-
operand forward on the separable kernel (grid_path "simt"), normwise per row; two independent paths."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch, paper_2506_13523_b200 as tpo
ctx = tpo.context()
for L, B in ((7, 5000), (8, 3000), (9, 2000), (7, 130), (3, 77)):
    d = (L + 1) ** 2; dout = (2 * L + 1) ** 2
    g = torch.Generator(device='cuda').manual_seed(L)
    x = torch.randn(B, d, device='cuda', generator=g); y = torch.randn(B, d, device='cuda', generator=g)
    go = torch.randn(B, dout, device='cuda', generator=g)
    ctx.set_grid_path('auto'); gx, gy = tpo.backward('gtp_grid', x, y, go, L, L, 2 * L)
    ctx.set_grid_path('simt'); sx, sy = tpo.backward('gtp_grid', x, y, go, L, L, 2 * L)
    ctx.set_grid_path('auto')
    def nw(a, b):
        return ((a - b).abs().amax(1) / b.abs().amax(1).clamp_min(1e-30)).max().item()
    print(L, B, nw(gx, sx), nw(gy, sy), torch.isfinite(gx).all().item())
