"""SIMT MTP (carrier dt > 13) device time per launch, warmed up, L2 flushed between reps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
fl = torch.empty(64 << 20, device=dev)
cases = []
for L, B in ((7, 65536), (8, 65536), (10, 65536), (16, 16384)):
    d = (L + 1) ** 2
    x = torch.randn(B, d, device=dev); y = torch.randn(B, d, device=dev)
    cases.append((L, B, x, y, tpo.mtp(x, y, L, L, 2 * L)))
for _ in range(3):  # warm clocks and caches
    for L, B, x, y, o in cases:
        tpo.mtp(x, y, L, L, 2 * L, out=o)
torch.cuda.synchronize()
for L, B, x, y, o in cases:
    tot = 0.0
    for _ in range(10):
        fl.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); tpo.mtp(x, y, L, L, 2 * L, out=o); b.record(); b.synchronize()
        tot += a.elapsed_time(b)
    print(f"L={L} {tot / 10:.4f} ms")
