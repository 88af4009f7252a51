"""e2e of the c2 step through tpo_run_host_batch_f32 (one call, all ten requests), device-timed."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

B = 65536
hx = {L: torch.randn(B, (L + 1) ** 2).pin_memory() for L in range(1, 11)}
hy = {L: torch.randn(B, (L + 1) ** 2).pin_memory() for L in range(1, 11)}
ho = {L: torch.empty(B, (2 * L + 1) ** 2).pin_memory() for L in range(1, 11)}
reqs = [("gtp_grid", hx[L], hy[L], ho[L], L, L, 2 * L) for L in range(10, 0, -1)]
order = os.environ.get("E2E_ORDER", "desc")
if order == "asc":
    reqs = reqs[::-1]
for _ in range(2):
    tpo.run_host_batch(reqs)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tpo.run_host_batch(reqs)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
ms = sorted(ts)[2]
nbytes = sum(t.numel() * 4 for L in range(1, 11) for t in (hx[L], hy[L], ho[L]))
print(f"chunk={os.environ.get('TPO_HOST_CHUNK_KB', 'default')} order={order} {ms:.3f} ms "
      f"{10 * B / ms / 1e3:.1f} M TP/s  {nbytes / ms / 1e6:.1f} GB/s", flush=True)
