"""One CGTP backward (L = 6, batch 65,536, both gradients) for ncu captures."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2506_13523_b200 as tpo

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
B = 65536
D = (L + 1) ** 2
x = torch.randn(B, D, device='cuda'); y = torch.randn(B, D, device='cuda'); g = torch.randn(B, D * D, device='cuda')
for _ in range(3):
    tpo.backward('cgtp', x, y, g, L, L, 2 * L)
torch.cuda.synchronize()
