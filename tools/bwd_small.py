"""One small CGTP backward (debugging: run under compute-sanitizer)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2506_13523_b200 as tpo

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B = int(sys.argv[2]) if len(sys.argv) > 2 else 24
D = (L + 1) ** 2
x = torch.randn(B, D, device='cuda'); y = torch.randn(B, D, device='cuda'); g = torch.randn(B, D * D, device='cuda')
gx, gy = tpo.backward('cgtp', x, y, g, L, L, 2 * L)
torch.cuda.synchronize()
print("ok", gx.abs().sum().item())
