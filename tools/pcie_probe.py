"""Pinned host <-> device copy bandwidth: H2D alone, D2H alone, both at once (separate streams)."""
import torch

dev = torch.device("cuda:0")
n = 256 << 20  # bytes
h_in = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n // 4, device=dev)
d_b = torch.empty(n // 4, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    return (h2d + d2h) * n * reps / ms / 1e6


run(True, True, 1)
print(f"H2D {run(True, False):.1f} GB/s  D2H {run(False, True):.1f} GB/s  both {run(True, True):.1f} GB/s (sum)")
