import sys, json
sys.path.insert(0, "/root/repo")
import torch, paper_2506_13523_b200 as tpo
dev = torch.device("cuda:0"); flush = torch.empty(64 << 20, device=dev); B = 65536
for path in ("tc", "simt"):
    tpo.context(0).set_grid_path(path)
    for L in (1, 2, 3, 4):
        d, do = (L + 1) ** 2, (2 * L + 1) ** 2
        x = torch.randn((B, d), device=dev); y = torch.randn((B, d), device=dev); o = torch.empty((B, do), device=dev)
        for _ in range(3): tpo.run("gtp_grid", x, y, L, L, 2 * L, out=o)
        tot = 0.0
        for _ in range(10):
            flush.zero_(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); tpo.run("gtp_grid", x, y, L, L, 2 * L, out=o); b.record(); b.synchronize(); tot += a.elapsed_time(b)
        print(path, L, round(tot / 10, 4), tpo.context(0).last_grid_path)
