"""Device time per kind at the BASELINE configs (L2 flushed between reps)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
g = torch.Generator(device=dev)
g.manual_seed(1)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    tot = 0.0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        flush.zero_()
        a.record(); fn(); b.record(); b.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


cases = [(k, L, 65536, 0) for k in ("gtp_grid", "gtp_fourier", "mtp", "cgtp") for L in (1, 2, 3, 4, 6, 8, 10)]
cases += [("cgtp", 3, 16384, 128), ("mtp", 16, 16384, 0), ("gtp_fourier", 16, 4096, 0), ("gtp_grid", 16, 16384, 0)]
for kind, L, B, C in cases:
    d = (L + 1) ** 2
    x = torch.randn((B, C, d) if C else (B, d), generator=g, device=dev)
    y = torch.randn((B, d), generator=g, device=dev)
    L3 = 0 if kind == "cgtp" else 2 * L
    try:
        o = tpo.run(kind, x, y, L, L, L3)
        ms = timeit(lambda: tpo.run(kind, x, y, L, L, L3, out=o))
        byts = 4 * (x.numel() + y.numel() + o.numel())
        print(json.dumps({"kind": kind, "L": L, "B": B, "C": C, "ms": round(ms, 4), "tp_per_s": round(B * max(C, 1) / ms * 1e3),
                          "gbs": round(byts / ms / 1e6, 1), "path": tpo.context(0).last_grid_path}), flush=True)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"kind": kind, "L": L, "error": str(e)[:200]}), flush=True)
    del x, y
    torch.cuda.empty_cache()
