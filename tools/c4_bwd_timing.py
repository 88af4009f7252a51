"""Backward of the channel-wise CGTP (config C4 shape: L=3, 128 channels, y shared per edge):
grad_x only (grad_y would be a channel reduction), 16,384 edges, L2 flushed."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
E, C, L = 16384, 128, 3
x = torch.randn((E, C, 16), device=dev); y = torch.randn((E, 16), device=dev)
g = torch.randn((E, C, 256), device=dev)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


fwd = timeit(lambda: tpo.cgtp(x, y, L, L))
bwd = timeit(lambda: tpo.backward("cgtp", x, y, g, L, L, 6, need_y=False))
byts = E * (C * 256 * 4 + 16 * 4 + C * 16 * 4)  # read grad_out, y; write grad_x
print(json.dumps({"edges": E, "channels": C, "fwd_ms": round(fwd, 4), "bwd_grad_x_ms": round(bwd, 4),
                  "bwd_gbs": round(byts / bwd / 1e6, 1), "bwd_hbm_frac": round(byts / (6550.7e9) / (bwd / 1e3), 4)}))
