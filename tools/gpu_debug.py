"""Run parity cases one per subprocess with a hard timeout (a hung kernel
cannot take the rest of the run down) and print one line per case."""
import json
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CASE = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/oracle')
import oracle, paper_2506_13523_b200 as tpo
kind, L, B, path = {kind!r}, {L}, {B}, {path!r}
ctx = tpo.context(0); ctx.set_grid_path(path)
rng = np.random.default_rng(L + 17)
d = (L + 1) ** 2
x = rng.standard_normal((B, d)).astype(np.float32); y = rng.standard_normal((B, d)).astype(np.float32)
xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
o = tpo.run(kind, xt, yt, L, L, 2 * L); torch.cuda.synchronize()
out = o.cpu().numpy().astype(np.float64)
ref = oracle.batch_mimo(kind, L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
err = np.abs(out - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)
bad = int((err > 1e-5).sum())
# timing
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
xb = torch.randn((65536, d), device='cuda'); yb = torch.randn((65536, d), device='cuda')
for _ in range(3): tpo.run(kind, xb, yb, L, L, 2 * L)
ev[0].record();
for _ in range(5): tpo.run(kind, xb, yb, L, L, 2 * L)
ev[1].record(); torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / 5
print(json.dumps(dict(kind=kind, L=L, B=B, path=ctx.last_grid_path, max_err=float(err.max()), n_bad=bad,
      argmax=int(err.argmax()), ms_65536=round(ms, 4), tp_per_s=round(65536 / ms * 1e3))))
"""


def run(kind, L, B=1000, path="auto", timeout=120):
    code = CASE.format(root=str(ROOT), kind=kind, L=L, B=B, path=path)
    t0 = time.time()
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=timeout)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 and r.stdout.strip() else \
            json.dumps(dict(kind=kind, L=L, path=path, rc=r.returncode, err=r.stderr.strip()[-600:]))
    except subprocess.TimeoutExpired:
        line = json.dumps(dict(kind=kind, L=L, path=path, timeout=timeout))
    print(line, f"({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "grid"):
        for L in range(0, 11):
            run("gtp_grid", L, path="tc", timeout=45)
    if which in ("all", "simt"):
        for L in (1, 3, 6, 11, 16):
            run("gtp_grid", L, B=200, path="simt")
    if which in ("all", "other"):
        for kind, Ls in (("cgtp", (0, 1, 2, 3, 4, 6, 8)), ("gtp_fourier", (0, 1, 2, 4, 6, 8, 10)),
                         ("mtp", (0, 1, 2, 3, 6, 10, 16))):
            for L in Ls:
                run(kind, L, B=300)
