"""Backward (tpo_backward_f32) vs forward device time per kind and L, batch 65,536.

    python tools/bwd_timing.py [--kinds gtp_grid,mtp,cgtp,gtp_fourier] [--Ls 1,2,...]
One JSON line per (kind, L): fwd_ms, bwd_ms (grad_x + grad_y), L2 flushed before each rep.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="gtp_grid,gtp_fourier,mtp,cgtp")
    ap.add_argument("--Ls", default="1,2,3,4,5,6,8,10")
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--path", default="auto", help="grid path for both passes: auto | tc | simt")
    a = ap.parse_args()
    import torch

    import paper_2506_13523_b200 as tpo

    dev = torch.device("cuda:0")
    tpo.context(0).set_grid_path(a.path)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    B = a.batch

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / reps

    for kind in a.kinds.split(","):
        for L in map(int, a.Ls.split(",")):
            if kind == "cgtp" and L > 8:
                continue
            d = (L + 1) ** 2
            dout = (L + 1) ** 4 if kind == "cgtp" else (2 * L + 1) ** 2
            x = torch.randn((B, d), device=dev); y = torch.randn((B, d), device=dev)
            g = torch.randn((B, dout), device=dev)
            fwd = timeit(lambda: tpo.run(kind, x, y, L, L, 2 * L))
            bwd = timeit(lambda: tpo.backward(kind, x, y, g, L, L, 2 * L))
            print(json.dumps({"kind": kind, "L": L, "path": a.path, "fwd_ms": round(fwd, 4), "bwd_ms": round(bwd, 4),
                              "ratio": round(bwd / fwd, 2)}), flush=True)
            del x, y, g


if __name__ == "__main__":
    main()
