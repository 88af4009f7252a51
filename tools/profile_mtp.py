"""One MTP forward (L from argv, 65,536 rows) for ncu captures."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2506_13523_b200 as tpo

L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
B = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
D = (L + 1) ** 2
x = torch.randn(B, D, device='cuda'); y = torch.randn(B, D, device='cuda')
for _ in range(3):
    o = tpo.mtp(x, y, L, L, 2 * L)
torch.cuda.synchronize()
