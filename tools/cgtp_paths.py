"""CGTP forward device time per L on the current dispatch (TPO_CGTP_TC env picks the path)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
Ls = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8,10,12,13,14,15,16").split(",")]
for L in Ls:
    B = 148 * 128 * 2  # two full waves of 128-row tiles
    d = (L + 1) ** 2
    x = torch.randn(B, d, device=dev); y = torch.randn(B, d, device=dev)
    o = tpo.run("cgtp", x, y, L, L, 2 * L)
    for _ in range(2):
        tpo.run("cgtp", x, y, L, L, 2 * L, out=o)
    tot = 0.0
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); tpo.run("cgtp", x, y, L, L, 2 * L, out=o); b.record(); b.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / 5
    gbs = B * (2 * d + (L + 1) ** 4) * 4 / ms / 1e6
    print(json.dumps({"L": L, "B": B, "ms": round(ms, 4), "ms_per_2^19": round(ms * (1 << 19) / B, 2), "gbs": round(gbs, 1)}), flush=True)
    del x, y, o
