"""Grid / Fourier GTP at large L: SIMT separable kernel (row-quad, or the one-product-per-block kernel with
TPO_GRID_SIMT_OLD=1) against the tcgen05 path, 2^19 products (one c5 shard), L2 flushed, ms."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
ctx = tpo.context()
B = 1 << 19
Ls = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8, 10, 11, 12, 13, 14, 15, 16]
paths = sys.argv[2].split(",") if len(sys.argv) > 2 else ["simt", "auto"]
kind = sys.argv[3] if len(sys.argv) > 3 else "gtp_grid"
for L in Ls:
    d = (L + 1) ** 2
    x = torch.randn(B, d, device=dev); y = torch.randn(B, d, device=dev)
    res = {"kind": kind, "L": L}
    for path in paths:
        ctx.set_grid_path(path)
        o = tpo.run(kind, x, y, L, L, 2 * L)
        tpo.run(kind, x, y, L, L, 2 * L, out=o)
        used = ctx.last_grid_path
        reps = 3 if L >= 12 else 10
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); tpo.run(kind, x, y, L, L, 2 * L, out=o); b.record(); b.synchronize()
            tot += a.elapsed_time(b)
        res[path] = round(tot / reps, 3)
        res[path + "_used"] = used
    ctx.set_grid_path("auto")
    print(json.dumps(res), flush=True)
