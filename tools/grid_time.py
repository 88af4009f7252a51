"""Device time of single grid/Fourier GTP launches at chosen L (L2 flushed between reps).
usage: python tools/grid_time.py [kind] L1 L2 ..."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

kind = sys.argv[1] if not sys.argv[1].isdigit() else "gtp_grid"
Ls = [int(a) for a in sys.argv[1:] if a.isdigit()]
dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
B = 65536
for L in Ls:
    d, do = (L + 1) ** 2, (2 * L + 1) ** 2
    x = torch.randn((B, d), device=dev); y = torch.randn((B, d), device=dev); o = torch.empty((B, do), device=dev)
    for _ in range(3):
        tpo.run(kind, x, y, L, L, 2 * L, out=o)
    tot = 0.0
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); tpo.run(kind, x, y, L, L, 2 * L, out=o); b.record(); b.synchronize()
        tot += a.elapsed_time(b)
    print(json.dumps({"kind": kind, "L": L, "ms": round(tot / 10, 4), "path": tpo.context(0).last_grid_path}), flush=True)
