"""Small runs of every kernel path for compute-sanitizer (memcheck): ragged batches,
shared y, weights, host batch API."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(5)
for kind, L, B in (("gtp_grid", 3, 300), ("gtp_grid", 7, 130), ("gtp_fourier", 4, 200), ("mtp", 6, 300),
                   ("mtp", 2, 129), ("cgtp", 6, 140), ("cgtp", 3, 77)):
    d = (L + 1) ** 2
    x = torch.randn((B, d), generator=g, device=dev)
    y = torch.randn((B, d), generator=g, device=dev)
    tpo.run(kind, x, y, L, L, 0 if kind == "cgtp" else 2 * L)
x = torch.randn((3, 128, 16), generator=g, device=dev)
y = torch.randn((3, 16), generator=g, device=dev)
tpo.cgtp(x, y, 3, 3)  # C4 edge kernel
x = torch.randn((150, 36), generator=g, device=dev)
y = torch.randn((150, 36), generator=g, device=dev)
tpo.weighted_gtp(x, y, np.ones(6), np.ones(6), np.ones(11), 5, 5, 10)
hx = torch.randn(500, 16).pin_memory(); hy = torch.randn(500, 16).pin_memory()
ho = torch.empty(500, 49).pin_memory(); hm = torch.empty(500, 49).pin_memory()
tpo.run_host_batch([("gtp_grid", hx, hy, ho, 3, 3, 6), ("mtp", hx, hy, hm, 3, 3, 6)])
# K > 128 grid / Fourier instantiation (L = 11, 12), CGTP blocks at L = 13
for kind, L, B in (("gtp_grid", 11, 130), ("gtp_fourier", 12, 70), ("cgtp", 13, 9)):
    d = (L + 1) ** 2
    x = torch.randn((B, d), generator=g, device=dev)
    y = torch.randn((B, d), generator=g, device=dev)
    tpo.run(kind, x, y, L, L, 0 if kind == "cgtp" else 2 * L)
# backward of every kind: degree groups + gather + accumulate (grid L=7, MTP L=6), CGTP kernel,
# shared-y grad_x
for kind, L, B in (("gtp_grid", 7, 130), ("gtp_grid", 3, 77), ("mtp", 6, 150), ("mtp", 2, 40),
                   ("cgtp", 6, 70), ("cgtp", 2, 33)):
    d = (L + 1) ** 2
    dout = (L + 1) ** 4 if kind == "cgtp" else (2 * L + 1) ** 2
    x = torch.randn((B, d), generator=g, device=dev)
    y = torch.randn((B, d), generator=g, device=dev)
    go = torch.randn((B, dout), generator=g, device=dev)
    tpo.backward(kind, x, y, go, L, L, 2 * L)
x = torch.randn((3, 64, 16), generator=g, device=dev)
y = torch.randn((3, 16), generator=g, device=dev)
go = torch.randn((3, 64, 256), generator=g, device=dev)
tpo.backward("cgtp", x, y, go, 3, 3, 6, need_y=False)
# round 2: CGTP backward on tcgen05 (L = 4 / 6 / 7 N parts; ragged tails < 4 rows take SIMT), MTP
# SIMT past dt = 13 (double-buffered staging, interleaved terms), the L = 1 small GTP kernel
for L, B in ((4, 131), (6, 66), (7, 40), (8, 36)):
    d = (L + 1) ** 2
    x = torch.randn((B, d), generator=g, device=dev)
    y = torch.randn((B, d), generator=g, device=dev)
    go = torch.randn((B, d * d), generator=g, device=dev)
    tpo.backward("cgtp", x, y, go, L, L)
for L, B in ((7, 70), (9, 33)):
    d = (L + 1) ** 2
    x = torch.randn((B, d), generator=g, device=dev)
    y = torch.randn((B, d), generator=g, device=dev)
    tpo.mtp(x, y, L, L, 2 * L)
for kind in ("gtp_grid", "gtp_fourier"):
    x = torch.randn((3, 70, 4), generator=g, device=dev)
    y = torch.randn((3, 4), generator=g, device=dev)
    tpo.run(kind, x, y, 1, 1, 2)
torch.cuda.synchronize()
print("sanitize run done")
# round 2: the row-quad separable kernel (grid nodes and the Fourier torus), ragged quads, odd band,
# shared y, and both register-budget variants (L = 12: 320 threads... L = 13: 256)
ctx = tpo.context()
for path, kind, L1, L2, L3, B in (("simt", "gtp_grid", 13, 13, 26, 7), ("simt", "gtp_grid", 3, 2, 4, 5),
                                  ("sep", "gtp_fourier", 12, 12, 24, 6), ("sep", "gtp_fourier", 5, 2, 9, 3),
                                  ("sep", "gtp_fourier", 16, 16, 32, 2)):
    ctx.set_grid_path(path)
    x = torch.randn((B, (L1 + 1) ** 2), generator=g, device=dev)
    y = torch.randn((B, (L2 + 1) ** 2), generator=g, device=dev)
    tpo.run(kind, x, y, L1, L2, L3)
ctx.set_grid_path("auto")
x = torch.randn((3, 5, 196), generator=g, device=dev)
y = torch.randn((3, 196), generator=g, device=dev)
tpo.run("gtp_fourier", x, y, 13, 13, 26)
torch.cuda.synchronize()
print("sanitize_small: separable ok")
