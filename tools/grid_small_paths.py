"""Grid / Fourier GTP at small L on each path (tcgen05 vs SIMT), 65,536 products, L2 flushed."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
ctx = tpo.context()
B = 65536
for kind in ("gtp_grid", "gtp_fourier"):
    for L in (1, 2, 3, 4, 5, 6, 7):
        d = (L + 1) ** 2
        x = torch.randn(B, d, device=dev); y = torch.randn(B, d, device=dev)
        res = {}
        for path in ("auto", "tc", "simt"):
            ctx.set_grid_path(path)
            o = tpo.run(kind, x, y, L, L, 2 * L)
            for _ in range(3):
                tpo.run(kind, x, y, L, L, 2 * L, out=o)
            tot = 0.0
            for _ in range(20):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); tpo.run(kind, x, y, L, L, 2 * L, out=o); b.record(); b.synchronize()
                tot += a.elapsed_time(b)
            res[path] = round(tot / 20, 4)
        ctx.set_grid_path("auto")
        print(json.dumps({"kind": kind, "L": L, **res}), flush=True)
