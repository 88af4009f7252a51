"""Grid GTP tcgen05 plan knobs (env TPO_GRID_*) at the c2 batch: ms per 65,536 products, L2 flushed."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
B = 65536
env = {k: v for k, v in os.environ.items() if k.startswith("TPO_GRID_")}
res = {"env": env}
for L in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8,9,10").split(",")]:
    d = (L + 1) ** 2
    x = torch.randn(B, d, device=dev); y = torch.randn(B, d, device=dev)
    try:
        o = tpo.run("gtp_grid", x, y, L, L, 2 * L)
        for _ in range(3):
            tpo.run("gtp_grid", x, y, L, L, 2 * L, out=o)
        tot = 0.0
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); tpo.run("gtp_grid", x, y, L, L, 2 * L, out=o); b.record(); b.synchronize()
            tot += a.elapsed_time(b)
        res[f"L{L}"] = round(tot / 20, 4)
    except Exception as e:  # a forced plan that does not fit
        res[f"L{L}"] = str(e)[:60]
print(json.dumps(res), flush=True)
