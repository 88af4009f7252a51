"""BASELINE configs[4] (C5) per GPU: all four products, L = 1..16, one GPU's shard
of 2^22 over 8 GPUs = 2^19 products (8 shards are independent: no collective).

Device time per launch (CUDA events, L2 flushed); CGTP outputs at large L
((L+1)^4 floats per product, 175 GB at L = 16) are produced in chunks of
<= 4 GB of output, timed per chunk and scaled to the shard (the chunks are
independent launches over disjoint rows).  Roofline per SURVEY.md 8(d): HBM
bytes 4 (2 Din + Dout) per product against MEASURED_PEAKS.json hbm_gbs; for the
tensor-core grid / Fourier launches also the dense-operator flops against the
bf16 peak / 3 (3xFP16).  One JSON line per (kind, L).
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import paper_2506_13523_b200 as tpo

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    hbm = peaks["hbm_gbs"] * 1e9
    tc = peaks["bf16_tflops"] / 3 * 1e12
    dev = torch.device("cuda:0")
    flush = torch.empty(64 << 20, device=dev)
    SHARD = 1 << 19
    Ls = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(range(1, 17))
    kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["gtp_grid", "gtp_fourier", "mtp", "cgtp"]
    ctx = tpo.context()

    def timeit(fn, reps=5):
        fn(); fn()
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); b.synchronize()
            tot += a.elapsed_time(b)
        return tot / reps

    for kind in kinds:
        for L in Ls:
            din = (L + 1) ** 2
            dout = (L + 1) ** 4 if kind == "cgtp" else (2 * L + 1) ** 2
            L3 = 0 if kind == "cgtp" else 2 * L
            B = min(SHARD, max(4096, int(4e9 // (4 * dout)) // 128 * 128))
            slow = kind == "mtp" and L >= 7
            if slow:  # SIMT paths: a 16384-row sample keeps the sweep within minutes
                B = min(B, 16384)
            g = torch.Generator(device=dev); g.manual_seed(L)
            x = torch.randn((B, din), generator=g, device=dev)
            y = torch.randn((B, din), generator=g, device=dev)
            o = torch.empty((B, dout), device=dev)
            ms = timeit(lambda: tpo.run(kind, x, y, L, L, L3, out=o)) * SHARD / B
            t = ms / 1e3
            byts = 4 * (2 * din + dout) * SHARD
            rec = {"kind": kind, "L": L, "shard": SHARD, "sample_rows": B, "ms": round(ms, 4),
                   "tp_per_s": round(SHARD / t), "gbs": round(byts / t / 1e9, 1), "hbm_frac": round(byts / hbm / t, 4)}
            if kind in ("gtp_grid", "gtp_fourier"):
                rec["path"] = ctx.last_grid_path
                if rec["path"] == "tcgen05":
                    G = (2 * L + 1) * (4 * L + 1) if kind == "gtp_grid" else (4 * L + 2) ** 2 // 2
                    fl = 2 * G * (2 * din + dout) * SHARD
                    rec["tflops_dense"] = round(fl / t / 1e12, 1)
                    rec["tensor_frac"] = round(fl / tc / t, 4)
            print(json.dumps(rec), flush=True)
            del x, y, o
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
