"""Per-L time of tpo_run_host_f32 (pinned host buffers) vs its D2H-bound floor."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_13523_b200 as tpo
B = 65536
ctx = tpo.context(0); lib = tpo.lib()
tot = 0.0
for L in range(1, 11):
    hx = torch.randn(B, (L + 1) ** 2).pin_memory(); hy = torch.randn(B, (L + 1) ** 2).pin_memory()
    ho = torch.empty(B, (2 * L + 1) ** 2).pin_memory()
    call = lambda: tpo.check(lib.tpo_run_host_f32(ctx.handle, tpo.KINDS["gtp_grid"], L, L, 2 * L, -1, hx.data_ptr(),
                                                  hy.data_ptr(), ho.data_ptr(), B, 1, 0))
    for _ in range(2): call()
    t0 = time.perf_counter()
    for _ in range(10): call()
    dt = (time.perf_counter() - t0) / 10
    tot += dt
    bin_, bout = hx.numel() * 8, ho.numel() * 4
    print(f"L={L:2d} {dt*1e3:7.3f} ms  in {bin_/1e6:6.1f} MB out {bout/1e6:6.1f} MB  floor(out@57) {bout/57e6:6.3f} ms"
          f"  serial {(bin_/55.5e6 + bout/57e6):6.3f} ms")
print(f"sum {tot*1e3:.3f} ms")
