import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch, paper_2506_13523_b200 as tpo
dev = torch.device("cuda:0"); B, L = 65536, 6
x = torch.randn(B, 49, device=dev); y = torch.randn(B, 49, device=dev)
a, b, c = np.ones(7), np.ones(7), np.ones(13)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize(); return e0.elapsed_time(e1) / reps
print("gtp_grid", round(t(lambda: tpo.gtp_grid(x, y, L, L, 2 * L)), 4), "ms")
print("weighted (fused)", round(t(lambda: tpo.weighted_gtp(x, y, a, b, c, L, L, 2 * L)), 4), "ms")
tpo.context().set_grid_path("simt")
print("weighted (simt + passes)", round(t(lambda: tpo.weighted_gtp(x, y, a, b, c, L, L, 2 * L)), 4), "ms")
