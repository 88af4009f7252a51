"""Grid sweep (L = 1..10, 65,536 TPs each) as one CUDA graph: serial launches vs the ten
independent launches on parallel graph branches (the next problem's CTAs fill the SMs
the previous one frees).  Device time per sweep, L2 flushed before each replay."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2506_13523_b200 as tpo

dev = torch.device("cuda:0")
B, LS = 65536, list(range(1, 11))
xs = {L: torch.randn((B, (L + 1) ** 2), device=dev) for L in LS}
ys = {L: torch.randn((B, (L + 1) ** 2), device=dev) for L in LS}
outs = {L: torch.empty((B, (2 * L + 1) ** 2), device=dev) for L in LS}
flush = torch.empty(64 << 20, device=dev)
for L in LS:
    tpo.gtp_grid(xs[L], ys[L], L, L, 2 * L, out=outs[L])
torch.cuda.synchronize()

serial = torch.cuda.CUDAGraph()
with torch.cuda.graph(serial):
    for L in LS:
        tpo.gtp_grid(xs[L], ys[L], L, L, 2 * L, out=outs[L])

order = sorted(LS, reverse=True) if "--asc" not in sys.argv else LS
side = [torch.cuda.Stream() for _ in LS]
conc = torch.cuda.CUDAGraph()
with torch.cuda.graph(conc):
    main = torch.cuda.current_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    joins = []
    for s, L in zip(side, order):
        s.wait_event(fork)
        with torch.cuda.stream(s):
            tpo.gtp_grid(xs[L], ys[L], L, L, 2 * L, out=outs[L])
        e = torch.cuda.Event()
        e.record(s)
        joins.append(e)
    for e in joins:
        main.wait_event(e)


def t(graph, reps=20):
    for _ in range(3):
        graph.replay()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); graph.replay(); b.record(); b.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


ref = {L: outs[L].clone() for L in LS}
for L in LS:
    outs[L].zero_()
ms_c = t(conc)
ok = all(torch.equal(outs[L], ref[L]) for L in LS)
ms_s = t(serial)
print(f"serial {ms_s:.4f} ms ({10 * B / ms_s / 1e3:.1f} M TP/s)  concurrent {ms_c:.4f} ms ({10 * B / ms_c / 1e3:.1f} M TP/s)"
      f"  identical outputs: {ok}")
