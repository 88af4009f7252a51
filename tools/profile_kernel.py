"""Launch one TPO kernel a few times on resident inputs (for ncu captures).

    ncu --set full -k regex:gtp_grid_tc -s 2 -c 1 -o prof python tools/profile_kernel.py --kind gtp_grid --L 10
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="gtp_grid")
    ap.add_argument("--L", type=int, default=10)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--channels", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--path", default="auto")
    a = ap.parse_args()
    import torch

    import paper_2506_13523_b200 as tpo

    dev = torch.device("cuda:0")
    L, B = a.L, a.batch
    d = (L + 1) ** 2
    if a.channels:
        x = torch.randn((B, a.channels, d), device=dev)
    else:
        x = torch.randn((B, d), device=dev)
    y = torch.randn((B, d), device=dev)
    tpo.context(0).set_grid_path(a.path)
    for _ in range(a.reps):
        out = tpo.run(a.kind, x, y, L, L, 2 * L)
    torch.cuda.synchronize()
    print(a.kind, L, B, tuple(out.shape), tpo.context(0).last_grid_path)


if __name__ == "__main__":
    main()
