"""e2e (host buffers through tpo_run_host_f32) for the grid sweep vs chunk size."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_13523_b200 as tpo
B = 65536
ctx = tpo.context(0); lib = tpo.lib()
hx = {L: torch.randn(B, (L + 1) ** 2).pin_memory() for L in range(1, 11)}
hy = {L: torch.randn(B, (L + 1) ** 2).pin_memory() for L in range(1, 11)}
ho = {L: torch.empty(B, (2 * L + 1) ** 2).pin_memory() for L in range(1, 11)}
def step():
    for L in range(1, 11):
        tpo.check(lib.tpo_run_host_f32(ctx.handle, tpo.KINDS["gtp_grid"], L, L, 2 * L, -1, hx[L].data_ptr(),
                                       hy[L].data_ptr(), ho[L].data_ptr(), B, 1, 0))
for _ in range(2): step()
t0 = time.perf_counter()
for _ in range(5): step()
dt = (time.perf_counter() - t0) / 5
print(os.environ.get("TPO_HOST_CHUNK_KB", "default"), round(dt * 1e3, 3), "ms", round(10 * B / dt / 1e6, 1), "M TP/s")
