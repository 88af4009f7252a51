#!/usr/bin/env python
"""Benchmark of the TPO hot path (BASELINE.json metric: tensor products/sec vs
L_max, % of roofline).

Workloads (``--workload``; every one is a BASELINE.json config):

* ``c2`` (default; configs[1], the metric's headline): S2-grid Gaunt TP, L_max
  sweep 1..10, 65,536 x 1 channel per GPU, L3 = 2L.  One step = the ten launches
  of the fused tcgen05 kernel (one per L) over inputs resident in HBM, captured
  once into a CUDA graph and replayed.  Weak scaling: every rank owns its own
  65,536-sample shard.
* ``c3`` (configs[2]): Fourier GTP, MTP and grid GTP at L=6, 65,536 per GPU.
* ``c4`` (configs[3]): channel-wise CGTP, L=3, 128 channels, y shared per edge,
  2^20 edges in total, strong-scaled over the ranks (each owns 2^20/N edges and
  writes its 128 x 256 outputs per edge to HBM).
* ``c5`` (configs[4]): all four products, L = 1..16, 2^19 products per GPU
  (2^22 over 8 GPUs), weak scaling.

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
synchronize, CUDA events on the launching stream, L2 flushed (256 MiB write)
before every step outside the events, max over ranks.  After the timed region:
outputs (c2/c3) or a parity subsample (c4/c5) are gathered to rank 0 over NCCL
and a strided subsample of every rank's shard is checked against the fp64 CPU
oracle (the checker; ``max_rel_err`` in the line).

``--impl reference`` times the reference CPU algorithm on the same workload and
config: the fp64 oracle port of proj/src/{sphere,gtp,cgtp,mtp}.cpp (the
reference itself cannot be built here: Eigen 3 is missing) on all host cores,
on a bounded sample of every step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tensor products/sec vs L_max for CGTP/grid-GTP/Fourier-GTP/MTP; % of roofline"
UNIT = "TP/s"
SEED = 20240901
C2_LS = list(range(1, 11))
C2_BATCH = 65536
C4_EDGES, C4_CHANNELS, C4_L = 1 << 20, 128, 3
C5_BATCH = 1 << 19
C5_LS = list(range(1, 17))
KINDS4 = ("gtp_grid", "gtp_fourier", "mtp", "cgtp")


# ---------------------------------------------------------------- per-TP work
def din(L):
    return (L + 1) ** 2


def dout(kind, L):
    return (L + 1) ** 4 if kind == "cgtp" else (2 * L + 1) ** 2


def bytes_per_tp(kind, L):
    return 4 * (2 * din(L) + dout(kind, L))


def c4_bytes_per_edge():
    """read x (128 channels x 16) and the shared y (16) once, write 128 x 256."""
    return C4_CHANNELS * 16 * 4 + 16 * 4 + C4_CHANNELS * 256 * 4


def dense_flops_per_tp(kind, L):
    """Dense-GEMM flops of the fused tcgen05 kernels: grid 2 G (2 Din + Dout) with
    G = (2L+1)(4L+1) product-grid points; Fourier the same on the N^2/2 folded torus
    points (N = 4L+2)."""
    G = (2 * L + 1) * (4 * L + 1) if kind == "gtp_grid" else (4 * L + 2) ** 2 // 2
    return 2 * G * (2 * din(L) + dout(kind, L))


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


FP32_TFLOPS = 2 * 148 * 128 * 1.965e9 / 1e12  # FFMA peak at max clock (not in MEASURED_PEAKS.json)


GTP_SEP_MIN_L = 11  # capi.cpp kGridSepMinL / kFourierSepMinL: the row-quad separable SIMT kernel


def gtp_path(kind, L):
    return "sep" if kind in ("gtp_grid", "gtp_fourier") and L >= GTP_SEP_MIN_L else "tc"


def sep_flops_per_tp(kind, L):
    """FFMA flops of the row-quad separable kernel (gtp_grid_simt.cu) per product, both grid
    symmetries folded: Legendre synthesis / analysis (din1 + din2 + dout) x node pairs, phi
    synthesis and analysis nodes x half-period points x (nm1 + nm2 + nm3)."""
    band = 2 * L
    nt = band + 1 if kind == "gtp_grid" else 2 * L + 2
    njp, nkp = (nt + 1) // 2, band + 1
    fma = (2 * din(L) + dout(kind, L)) * njp + nt * nkp * (2 * (2 * L + 1) + 2 * band + 1)
    return 2 * fma


def roofline_time(kind, L, n, peaks, path="tc"):
    """T_roof per SURVEY.md 8(d): max(bytes / HBM, flops / pipe peak) for n products."""
    t_hbm = bytes_per_tp(kind, L) * n / (peaks["hbm_gbs"] * 1e9)
    if kind in ("gtp_grid", "gtp_fourier") and path == "tc":
        return max(t_hbm, dense_flops_per_tp(kind, L) * n / (peaks["bf16_tflops"] / 3 * 1e12)), "tensor"
    if kind in ("gtp_grid", "gtp_fourier") and path == "sep":
        return max(t_hbm, sep_flops_per_tp(kind, L) * n / (FP32_TFLOPS * 1e12)), "fp32"
    return t_hbm, "hbm"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML polled every
    ~0.2 ms from a thread; nvidia-smi -lms 20 fallback).  Only samples taken while a
    region is open (``with clk.region():``) are summarised."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, set]] = []
        self.max_mhz = None
        self.source = None
        self._open = False
        self._stop = threading.Event()
        self._t = None
        self.proc = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            bits = [(n, getattr(pynvml, a)) for n, a in self.REASONS]

            def poll():
                while not self._stop.is_set():
                    if self._open:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, {n for n, b in bits if r & b}))
                    time.sleep(0.0002)

            self.source = "nvml (0.2 ms poll)"
            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi -lms 20"
            self._t = threading.Thread(target=self._read_smi, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read_smi(self):
        names = [n for n, _ in self.REASONS[:4]]
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if not self._open or len(parts) < 7:
                continue
            try:
                sm = float(parts[0])
                self.max_mhz = float(parts[1])
            except ValueError:
                continue
            self.samples.append((sm, {n for n, v in zip(names, parts[3:7]) if v.lower() == "active"}))

    class _Region:
        def __init__(self, outer):
            self.o = outer

        def __enter__(self):
            self.o._open = True

        def __exit__(self, *exc):
            self.o._open = False

    def region(self):
        return ClockSampler._Region(self)

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self._t:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        sm = [s for s, _ in self.samples]
        reasons = set().union(*[r for _, r in self.samples]) if self.samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


def dist_setup():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------- workload descriptions (shared by both arms)
def workload_config(args, world: int) -> dict:
    """The `config` object of the JSON line: identical for `--impl ours` and `--impl reference`."""
    w = args.workload
    if w == "c2":
        return {"workload": "S2-grid GTP L_max sweep 1-10, batch 65536 x 1 channel per GPU, L3=2L (BASELINE.json configs[1])",
                "batch_per_gpu": args.batch or C2_BATCH, "L": C2_LS, "channels": 1,
                "l2": "flushed between steps (256 MiB write, untimed)",
                "parallelism": f"dp{world} (independent shards, no data-path collective)"}
    if w == "c3":
        return {"workload": "Fourier GTP, MTP and S2-grid GTP at L_max=6, batch 65536 per GPU, L3=2L (BASELINE.json configs[2])",
                "batch_per_gpu": args.batch or C2_BATCH, "L": [6], "kinds": ["gtp_fourier", "mtp", "gtp_grid"],
                "l2": "flushed between steps (256 MiB write, untimed)",
                "parallelism": f"dp{world} (independent shards, no data-path collective)"}
    if w == "c4":
        return {"workload": "channel-wise CGTP L_max=3, 128 channels, y shared per edge, 2^20 edges in total "
                            "(BASELINE.json configs[3])",
                "edges_total": args.edges or C4_EDGES, "channels": C4_CHANNELS, "L": [C4_L],
                "tp_unit": "one (edge, channel) product", "l2": "inputs + outputs (146 GB) >> L2",
                "parallelism": f"dp{world} strong scaling (edges_total / {world} edges per GPU, no data-path collective)"}
    if w == "c5":
        return {"workload": "all four TPOs (CGTP, grid GTP, Fourier GTP, MTP) L_max sweep 1-16, 2^19 products per GPU "
                            "(2^22 over 8 GPUs; BASELINE.json configs[4])",
                "batch_per_gpu": args.batch or C5_BATCH, "L": C5_LS, "kinds": list(KINDS4),
                "l2": "flushed between steps (256 MiB write, untimed)",
                "parallelism": f"dp{world} (independent shards, no data-path collective)"}
    raise ValueError(w)


def step_units(args, world: int) -> list[tuple[str, int, int]]:
    """(kind, L, products per GPU) of one step on one rank (c4: this rank's edge shard x channels)."""
    w = args.workload
    if w == "c2":
        return [("gtp_grid", L, args.batch or C2_BATCH) for L in C2_LS]
    if w == "c3":
        return [(k, 6, args.batch or C2_BATCH) for k in ("gtp_fourier", "mtp", "gtp_grid")]
    if w == "c4":
        from paper_2506_13523_b200.dist import shard_range

        E = args.edges or C4_EDGES
        s0, s1 = shard_range(E, world, int(os.environ.get("RANK", "0")))
        return [("cgtp_edge", C4_L, (s1 - s0) * C4_CHANNELS)]
    return [(k, L, args.batch or C5_BATCH) for k in KINDS4 for L in C5_LS]


# ---------------------------------------------------------------- CPU reference (oracle port; checker + baseline)
def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # noqa: E402  (allowed: the CPU baseline / parity-checker legs)

    return oracle


def cpu_reference(args, seconds_per_unit: float, nthreads: int):
    """Reference CPU algorithm (fp64 oracle port) on host cores, per (kind, L) of the
    workload on a bounded sample; returns (TP/s over one step of the workload, samples)."""
    import numpy as np

    orc = _oracle()
    rng = np.random.default_rng(SEED)
    units = step_units(args, 1)
    seconds_per_unit *= 10.0 / max(10, len(units))  # c5: 64 (kind, L) units share the c2 budget
    total_t, total_n, samples = 0.0, 0, {}
    for kind, L, n_step in units:
        okind = "cgtp" if kind == "cgtp_edge" else kind
        C = C4_CHANNELS if kind == "cgtp_edge" else 1
        n = max(nthreads, 4)
        while True:
            B = max(1, n // C)
            x = rng.standard_normal((B, C, din(L)))
            y = rng.standard_normal((B, din(L)) if C > 1 else (B, 1, din(L)))
            t0 = time.perf_counter()
            orc.batch_mimo(okind, L, x, y, channels=C, y_shared=C > 1, nthreads=nthreads)
            dt = time.perf_counter() - t0
            if dt >= seconds_per_unit or B * C >= n_step:
                break
            n = min(n_step, int(B * C * max(2.0, 1.2 * seconds_per_unit / max(dt, 1e-6))))
        per_tp = dt / (B * C)
        samples[f"{kind}_L{L}"] = B * C
        total_t += per_tp * n_step
        total_n += n_step
    return total_n / total_t, samples


# ---------------------------------------------------------------- GPU arm
class Timer:
    def __init__(self, stream):
        import torch

        self.stream = stream
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        self.a.record(self.stream)
        return self

    def __exit__(self, *exc):
        self.b.record(self.stream)
        self.b.synchronize()
        self.ms = self.a.elapsed_time(self.b)


def normwise(out, ref):
    import numpy as np

    out = out.reshape(-1, out.shape[-1]).astype(np.float64)
    ref = ref.reshape(-1, ref.shape[-1])
    return float((np.abs(out - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)).max())


def subsample_idx(n, k):
    import numpy as np

    return np.unique(np.concatenate([np.linspace(0, n - 1, min(k, n)).astype(np.int64), [n - 1]])) if n else np.zeros(0, np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--batch", type=int, default=0, help="products per GPU (c2/c3/c5); 0 = the config's")
    ap.add_argument("--edges", type=int, default=0, help="c4: edges in total; 0 = 2^20")
    ap.add_argument("--cpu-seconds", type=float, default=1.0, help="CPU baseline seconds per (kind, L)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the per-kind side measurements (c2)")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-run oracle subsample check")
    ap.add_argument("--serial-sweep", action="store_true",
                    help="c2: capture the 10 launches in stream order instead of as parallel graph branches")
    ap.add_argument("--no-graph", action="store_true",
                    help="eager launches instead of CUDA-graph replay (ncu launch lists)")
    ap.add_argument("--plan-only", action="store_true",
                    help="print the per-rank plan (shards, bytes, config) and exit; needs no GPU (gloo under torchrun)")
    args = ap.parse_args()
    world, rank, local = dist_setup()

    if args.plan_only:
        return plan_only(args, world, rank)
    if args.impl == "reference":
        return run_reference(args, world, rank)
    run_ours(args, world, rank, local)


def plan_only(args, world, rank):
    """Host-side plan of the N>1 run (covered by tests/test_multiproc.py with gloo on CPU)."""
    import torch
    import torch.distributed as dist

    from paper_2506_13523_b200.dist import gather_checksums

    if world > 1:
        dist.init_process_group("gloo")
    units = step_units(args, world)
    mine = [sum(n for _, _, n in units), sum(c4_bytes_per_edge() * (n // C4_CHANNELS) if k == "cgtp_edge"
                                               else bytes_per_tp(k, L) * n for k, L, n in units)]
    every = gather_checksums(mine)
    if rank == 0:
        print(json.dumps({"plan": True, "n_gpus": world, "config": workload_config(args, world),
                          "per_rank_products": [int(e[0]) for e in every],
                          "per_rank_bytes": [int(e[1]) for e in every]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import paper_2506_13523_b200 as tpo
    from paper_2506_13523_b200.dist import gather_checksums, max_over_ranks, shard_range

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    ctx = tpo.context(local)
    stream = torch.cuda.current_stream(dev)
    peaks = load_peaks()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    g = torch.Generator(device=dev)
    w = args.workload

    # ---------------- problem set of this rank: list of launches (kind, L, x, y, out, rows)
    probs = []
    if w in ("c2", "c3", "c5"):
        B = args.batch or (C5_BATCH if w == "c5" else C2_BATCH)
        cg_ring = None
        for kind, L, _ in step_units(args, world):
            g.manual_seed(SEED + 1000 * rank + 17 * L + KINDS4.index(kind))
            x = torch.randn((B, din(L)), generator=g, device=dev)
            y = torch.randn((B, din(L)), generator=g, device=dev)
            if kind == "cgtp" and B * dout(kind, L) * 4 > (4 << 30):
                # CGTP outputs past 4 GiB (c5, L >= 8: 175 GB at L = 16) stream through one reused
                # 16 GiB buffer in row chunks; every chunk is computed and written to HBM
                if cg_ring is None:
                    cg_ring = torch.empty((16 << 30) // 4, dtype=torch.float32, device=dev)
                rows = max(1, cg_ring.numel() // dout(kind, L))
                for r0 in range(0, B, rows):
                    r1 = min(B, r0 + rows)
                    probs.append((kind, L, x[r0:r1], y[r0:r1], cg_ring[: (r1 - r0) * dout(kind, L)].view(r1 - r0, -1),
                                  r1 - r0, (r0, r1)))
            else:
                probs.append((kind, L, x, y, torch.empty((B, dout(kind, L)), device=dev), B, (0, B)))
    else:  # c4
        E = args.edges or C4_EDGES
        s0, s1 = shard_range(E, world, rank)
        Er = s1 - s0
        g.manual_seed(SEED + 1000 * rank)
        x = torch.randn((Er, C4_CHANNELS, din(C4_L)), generator=g, device=dev)
        y = torch.randn((Er, din(C4_L)), generator=g, device=dev)
        free = torch.cuda.mem_get_info(dev)[0]
        need = Er * C4_CHANNELS * dout("cgtp", C4_L) * 4
        if need <= free - (2 << 30):
            o = torch.empty((Er, C4_CHANNELS, dout("cgtp", C4_L)), device=dev)
            probs.append(("cgtp", C4_L, x, y, o, Er * C4_CHANNELS, (0, Er)))
        else:  # chunk through a reused buffer (not needed on a 180 GB B200)
            ring_edges = max(1, (free - (4 << 30)) // (C4_CHANNELS * dout("cgtp", C4_L) * 4))
            o = torch.empty((ring_edges, C4_CHANNELS, dout("cgtp", C4_L)), device=dev)
            for e0 in range(0, Er, ring_edges):
                e1 = min(Er, e0 + ring_edges)
                probs.append(("cgtp", C4_L, x[e0:e1], y[e0:e1], o[: e1 - e0], (e1 - e0) * C4_CHANNELS, (e0, e1)))

    def launch(p):
        kind, L, x, y, o = p[:5]
        tpo.run(kind, x, y, L, L, 0 if kind == "cgtp" else 2 * L, out=o)

    def step():
        for p in probs:
            launch(p)

    # eager warm-up builds the device tables
    step()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    graph = None
    if w == "c2" and not args.no_graph:
        # the ten L problems are independent, so they are captured as parallel graph branches,
        # largest L first: the next problem's persistent CTAs fill the SMs freed by a launch's
        # last wave (bit-identical outputs; --serial-sweep captures the stream order)
        graph = torch.cuda.CUDAGraph()
        side = [torch.cuda.Stream(dev) for _ in probs]
        with torch.cuda.graph(graph):
            if args.serial_sweep:
                step()
            else:
                cap = torch.cuda.current_stream(dev)
                fork = torch.cuda.Event()
                fork.record(cap)
                joins = []
                for s_, p in zip(side, sorted(probs, key=lambda q: -q[1])):
                    s_.wait_event(fork)
                    with torch.cuda.stream(s_):
                        launch(p)
                    e = torch.cuda.Event()
                    e.record(s_)
                    joins.append(e)
                for e in joins:
                    cap.wait_event(e)
        launches_per_step = ctx.launches - launches0
        run_step = graph.replay
    else:
        step()
        launches_per_step = ctx.launches - launches0
        run_step = step
    torch.cuda.synchronize()

    per_ms = {}
    total_ms = 0.0
    with ClockSampler(local) as clk:
        for _ in range(max(args.warmup, 3)):
            run_step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        with clk.region():
            for _ in range(args.steps):
                flush.zero_()  # evict L2 (untimed)
                with Timer(stream) as t:
                    run_step()
                total_ms += t.ms
            torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        # per-(kind, L) breakdown outside the headline timing, same flush discipline
        with clk.region():
            reps = max(2, min(5, args.steps // 4))
            keys = []
            for p in probs:
                k = (p[0], p[1])
                if k not in keys:
                    keys.append(k)
            for k in keys:
                ps = [p for p in probs if (p[0], p[1]) == k]
                fn = lambda: [launch(p) for p in ps]  # noqa: E731
                if graph is not None:  # replayed like the step, so host launch gaps stay out of the events
                    gk = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gk):
                        fn()
                    fn = gk.replay
                acc = 0.0
                for _ in range(reps):
                    flush.zero_()
                    with Timer(stream) as t:
                        fn()
                    acc += t.ms
                per_ms[k] = acc / reps
    launches = launches_per_step * args.steps
    total_ms = max_over_ranks(total_ms, dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ms_per_step = total_ms / args.steps
    n_rank = sum(p[5] for p in probs)
    n_all = int(sum(e[0] for e in gather_checksums([float(n_rank)], dev)))
    value = n_all / (ms_per_step / 1e3)

    # ---------------- per-(kind, L) roofline
    per, dom = {}, None
    for (kind, L), ms in per_ms.items():
        n = sum(p[5] for p in probs if (p[0], p[1]) == (kind, L))
        ek = "cgtp" if kind == "cgtp" else kind
        t_roof, bound = roofline_time(ek, L, n, peaks, gtp_path(kind, L))
        if w == "c4":
            t_roof = n // C4_CHANNELS * c4_bytes_per_edge() / (peaks["hbm_gbs"] * 1e9)
            bound = "hbm"
        per[f"{kind}_L{L}"] = {"ms": round(ms, 5), "tp_per_s": round(n / (ms / 1e3), 1), "bound": bound,
                               "roofline_frac": round(t_roof / (ms / 1e3), 4)}
        if dom is None or ms > per_ms[dom]:
            dom = (kind, L)
    dk, dL = dom
    dn = sum(p[5] for p in probs if (p[0], p[1]) == dom)
    dms = per_ms[dom]
    if dk in ("gtp_grid", "gtp_fourier") and gtp_path(dk, dL) == "tc":
        ach = dense_flops_per_tp(dk, dL) * dn / (dms / 1e3) / 1e12
        roofline = {"bound": "tensor", "kernel": f"gtp_grid_tc_kernel {dk} L={dL} (3xFP16 tcgen05)",
                    "achieved": round(ach, 2), "peak": round(peaks["bf16_tflops"] / 3, 1), "unit": "TFLOP/s",
                    "frac": round(ach / (peaks["bf16_tflops"] / 3), 4),
                    "peak_note": f"{peaks['source']} bf16 dense {peaks['bf16_tflops']} TF/s / 3 (three fp16 MMAs per "
                                 f"3xFP16 product); algorithmic flops = dense 2*G*(2Din+Dout) per TP x {dn} TPs per launch"}
    else:
        by = (dn // C4_CHANNELS * c4_bytes_per_edge() if w == "c4"
              else bytes_per_tp("cgtp" if dk == "cgtp" else dk, dL) * dn)
        ach = by / (dms / 1e3) / 1e9
        kname = {"cgtp": "cgtp_edge_tc_kernel" if w == "c4" else "cgtp (tcgen05 blocks / SIMT)",
                 "mtp": "mtp kernels", "gtp_grid": "gtp_grid SIMT", "gtp_fourier": "gtp_fourier SIMT"}[dk]
        roofline = {"bound": "hbm", "kernel": f"{kname} L={dL}", "achieved": round(ach, 1),
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4),
                    "peak_note": f"{peaks['source']} HBM copy bandwidth; algorithmic bytes = read x, y once + write "
                                 f"the outputs once, per launch of {dn} TPs"}
    roofline["share_of_step"] = round(sum(per_ms[k] for k in [dom]) / ms_per_step, 3)
    roofline["traffic"] = None
    tf_path = ROOT / "profiles" / "ncu_traffic.json"
    if tf_path.exists():  # DRAM bytes of one ncu --set full capture of the same kernel (tools/profile_kernel.py)
        try:
            tr = json.loads(tf_path.read_text()).get(f"{dk}_L{dL}" + ("_c4" if w == "c4" else ""))
            if tr is not None:
                # captures: 65,536 rows (c2 / c3 / grid / Fourier), 16,384 edges x 128 channels (c4),
                # 16,384 rows (MTP SIMT), 2,048 rows (CGTP L = 16): scaled to this launch's rows
                cap_rows = {"c4": 16384 * C4_CHANNELS}.get(w, 65536)
                if dk == "cgtp" and dL == 16:
                    cap_rows = 2048
                elif dk == "mtp" and dL > 6:
                    cap_rows = 16384
                roofline["traffic"] = round(tr * dn / cap_rows, 1)
                roofline["traffic_note"] = (f"ncu dram__bytes_read+write of a {cap_rows}-row capture "
                                            f"(profiles/ncu_traffic.json), scaled to the {dn}-row launch")
        except Exception:
            pass
    step_roof = sum(roofline_time("cgtp" if k == "cgtp" else k, L, sum(p[5] for p in probs if (p[0], p[1]) == (k, L)),
                                  peaks, gtp_path(k, L))[0]
                    for (k, L) in per_ms) if w != "c4" else None
    if step_roof is not None:
        roofline["step_frac"] = round(step_roof / (ms_per_step / 1e3), 4)

    # ---------------- results to rank 0 and oracle parity of a subsample of every shard
    parity = None
    gather_ms = None
    if not args.no_parity:
        t0 = time.perf_counter()
        parity, gather_ms = gather_and_check(args, world, rank, probs, dev, dist, launch)
        parity["seconds"] = round(time.perf_counter() - t0, 2)

    # ---------------- e2e through the C ABI with pinned host buffers
    e2e = end_to_end(args, world, rank, probs, tpo, ctx, dev, max_over_ranks)

    extras = None
    if w == "c2" and not args.no_extras and rank == 0:
        extras = side_measurements(tpo, dev, stream, flush, peaks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nth = os.cpu_count() or 1
        v_all, samples = cpu_reference(args, args.cpu_seconds, nth)
        v_one, samples1 = cpu_reference(args, args.cpu_seconds / 2, 1)
        cpu = {"value": round(v_all, 1), "unit": UNIT, "cores": nth, "kind": "port",
               "sample": f"fp64 oracle port (proj/src/{{sphere,gtp,cgtp,mtp}}.cpp) on {nth} host threads, per-(kind, L) "
                         f"samples {samples}, scaled to the step's products",
               "single_thread": {"value": round(v_one, 1), "unit": UNIT, "cores": 1,
                                 "sample": f"same port, 1 thread (the reference protocol, proj/include/tpo/bench.hpp:47-50), "
                                           f"samples {samples1}"}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong" if w == "c4" else "weak", "vs_baseline": None,
            "dtype": "f32 (3xFP16 tcgen05, fp32 accumulate; SIMT fp32 where noted)",
            "data": f"synthetic N(0,1) irreps generated on device, seed {SEED}+1000*rank",
            "config": workload_config(args, world),
            "per_kind_L": per, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "max_rel_err": parity["max_rel_err"] if parity else None, "parity": parity,
            "gather_ms": gather_ms, "clocks": clk.summary(), "wall_s_timed": round(wall, 3),
            "timing": ("CUDA graph of the 10-launch sweep replayed per step" if graph is not None else
                       "eager launches per step") + "; CUDA events on the launch stream; L2 flushed (256 MiB write) "
                                                   "before every step, outside the events; max over ranks",
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def gather_and_check(args, world, rank, probs, dev, dist, launch):
    """After the timed region: every rank's parity subsample (inputs + outputs of strided rows,
    the last rows included) goes to rank 0 over NCCL (c2/c3: the whole output shards are
    all-gathered first, as the result gather), and rank 0 checks it against the fp64 oracle."""
    import numpy as np
    import torch

    t_gather = None
    per_unit = {}
    k_rows = 1024 if args.workload in ("c2", "c3") else 128
    for p in probs:
        kind, L, x, y, o, n, span = p
        if (kind, L) in per_unit:
            continue  # one subsample per (kind, L): the first chunk
        if args.workload in ("c2", "c3") and world > 1:
            # result gather: every rank's full output shard (GTP/MTP outputs fit: 8 x 0.45 GB)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            full = torch.empty((world,) + tuple(o.shape), dtype=o.dtype, device=dev)
            dist.all_gather_into_tensor(full, o.contiguous())
            torch.cuda.synchronize()
            t_gather = (t_gather or 0.0) + (time.perf_counter() - t0) * 1e3
        # outputs past 4 GiB share one ring buffer across chunks (and the timed steps overwrote it):
        # recompute the sampled launch (deterministic) before reading its rows
        launch(p)
        torch.cuda.synchronize()
        rows = x.shape[0]
        idx = torch.from_numpy(subsample_idx(rows, k_rows)).to(dev)
        xs, ys, os_ = x[idx].contiguous(), y[idx].contiguous(), o[idx].contiguous()
        if world > 1:
            def gat(t):
                parts = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=dev)
                dist.all_gather_into_tensor(parts, t)
                return parts
            xs, ys, os_ = gat(xs), gat(ys), gat(os_)
            if args.workload in ("c2", "c3"):  # the gathered shards must hold the same rows
                os_full = full[:, idx]
                assert torch.equal(os_full, os_), "gathered output shard differs from the rank's own"
        else:
            xs, ys, os_ = xs[None], ys[None], os_[None]
        per_unit[(kind, L)] = (xs.cpu().numpy(), ys.cpu().numpy(), os_.cpu().numpy())
    res = {"rows_checked_per_rank": k_rows, "per_kind_L": {}}
    if rank == 0:
        orc = _oracle()
        worst = 0.0
        for (kind, L), (xs, ys, os_) in per_unit.items():
            xs = xs.reshape((-1,) + xs.shape[2:]).astype(np.float64)
            ys = ys.reshape((-1,) + ys.shape[2:]).astype(np.float64)
            if args.workload == "c4":
                ref = orc.batch_mimo("cgtp", L, xs, ys, channels=C4_CHANNELS, y_shared=True)
            else:
                ref = orc.batch_mimo(kind, L, xs[:, None], ys[:, None])[:, 0]
            e = normwise(os_.reshape(ref.shape), ref)
            res["per_kind_L"][f"{kind}_L{L}"] = e
            worst = max(worst, e)
        res["max_rel_err"] = worst
        res["tolerance"] = 1e-5
        res["pass"] = worst <= 1e-5
    return res, (round(t_gather, 2) if t_gather is not None else None)


def end_to_end(args, world, rank, probs, tpo, ctx, dev, max_over_ranks):
    """Same metric through the reference-facing C ABI with HOST buffers: tpo_run_host_batch_f32
    copies each request's inputs from pinned host memory, computes, and copies the outputs back
    (copies inside the timed region).  c4/c5 use a bounded sample of every launch (stated)."""
    import torch

    w = args.workload
    cap_rows = {"c2": None, "c3": None, "c4": 4096, "c5": 16384}[w]
    reqs, seen, h2d, d2h, n = [], set(), 0, 0, 0
    for p in probs:
        kind, L, x, y, o, rows_tp, span = p
        if (kind, L) in seen:
            continue
        seen.add((kind, L))
        # bounded sample: at most cap_rows rows and 256 MiB of outputs per request
        row_bytes = o[:1].numel() * 4
        rows = x.shape[0] if cap_rows is None else min(x.shape[0], cap_rows, max(1, (256 << 20) // row_bytes))
        hx = x[:rows].cpu().pin_memory()
        hy = y[:rows].cpu().pin_memory()
        ho = torch.empty((rows,) + tuple(o.shape[1:]), pin_memory=True)
        reqs.append((kind, hx, hy, ho, L, L, 0 if kind == "cgtp" else 2 * L))
        h2d += (hx.numel() + hy.numel()) * 4
        d2h += ho.numel() * 4
        n += rows * (C4_CHANNELS if w == "c4" else 1)

    def run():
        tpo.run_host_batch(reqs, dev.index)

    for _ in range(2):
        run()
    k = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(k):
        run()
    et = max_over_ranks((time.perf_counter() - t0) / k, dev)
    return {"value": round(world * n / et, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(et * 1e3, 3),
            "path": "tpo_run_host_batch_f32 (C ABI, pinned host buffers, all of a step's requests in one call)",
            "sample": None if cap_rows is None else
            f"first min({cap_rows}, 256 MiB of outputs) rows of every (kind, L) launch per rank"}


def side_measurements(tpo, dev, stream, flush, peaks):
    """Throughput and roofline fraction of the other kinds (c3 shapes, a C4 chunk, CGTP blocks,
    backward), device time, one launch each, L2 flushed."""
    import torch

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            with Timer(stream) as t:
                fn()
            tot += t.ms
        return tot / reps

    hbm = peaks["hbm_gbs"] * 1e9
    res = {}
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    L, B = 6, 65536
    x = torch.randn((B, din(L)), generator=g, device=dev)
    y = torch.randn((B, din(L)), generator=g, device=dev)
    o = torch.empty((B, dout("mtp", L)), device=dev)
    for kind in ("gtp_grid", "gtp_fourier", "mtp"):
        ms = timeit(lambda: tpo.run(kind, x, y, L, L, 2 * L, out=o))
        t = ms / 1e3
        byts = bytes_per_tp(kind, L) * B
        if kind == "mtp":
            fl = 2 * 6378 * B  # 2 x reference sparse muls
            roof = max(byts / hbm, fl / (FP32_TFLOPS * 1e12))
            bound = "max(HBM, FP32 at the reference sparse op count, nominal clock)"
        else:
            fl = dense_flops_per_tp(kind, L) * B
            roof = max(byts / hbm, fl / (peaks["bf16_tflops"] / 3 * 1e12))
            bound = "tensor (dense operators, 3xFP16)"
        res[f"{kind}_L{L}_B{B}"] = {"ms": round(ms, 4), "tp_per_s": round(B / t, 1), "tflops": round(fl / t / 1e12, 2),
                                     "gbs": round(byts / t / 1e9, 1), "roofline_frac": round(roof / t, 4), "bound": bound}
    L, C, B = 3, 128, 1 << 14
    x = torch.randn((B, C, 16), generator=g, device=dev)
    y = torch.randn((B, 16), generator=g, device=dev)
    o = torch.empty((B, C, 256), device=dev)
    ms = timeit(lambda: tpo.cgtp(x, y, L, L, out=o))
    byts = B * (C * 16 * 4 + 16 * 4 + C * 256 * 4)
    res[f"cgtp_L3_C128_B{B}"] = {"ms": round(ms, 4), "channel_tp_per_s": round(B * C / ms * 1e3, 1),
                                  "gbs": round(byts / ms / 1e6, 1), "roofline_frac": round(byts / hbm / (ms / 1e3), 4),
                                  "bound": "HBM (139,328 B per edge)"}
    L, B = 6, 65536
    x = torch.randn((B, din(L)), generator=g, device=dev)
    y = torch.randn((B, din(L)), generator=g, device=dev)
    o = torch.empty((B, dout("cgtp", L)), device=dev)
    ms = timeit(lambda: tpo.cgtp(x, y, L, L, out=o))
    byts = bytes_per_tp("cgtp", L) * B
    res[f"cgtp_L{L}_B{B}"] = {"ms": round(ms, 4), "tp_per_s": round(B / ms * 1e3, 1), "gbs": round(byts / ms / 1e6, 1),
                              "roofline_frac": round(byts / hbm / (ms / 1e3), 4), "bound": "HBM"}
    del o
    bwd = {}
    for kind in KINDS4:
        go = torch.randn((B, dout(kind, L)), generator=g, device=dev)
        ms = timeit(lambda: tpo.backward(kind, x, y, go, L, L, 2 * L))
        byts = 4 * (4 * din(L) + dout(kind, L)) * B
        bwd[f"{kind}_L{L}_B{B}"] = {"ms": round(ms, 4), "tp_per_s": round(B / ms * 1e3, 1),
                                    "gbs": round(byts / ms / 1e6, 1), "hbm_frac": round(byts / hbm / (ms / 1e3), 4)}
        del go
    res["backward"] = bwd
    return res


def run_reference(args, world, rank):
    """Reference arm: the reference CPU algorithm (fp64 oracle port) on this box's host cores,
    same workload / config / metric; rank 0 only under torchrun."""
    if world > 1 and rank != 0:
        return
    nth = os.cpu_count() or 1
    cpu_reference(args, 0.01, nth)  # table caches (untimed)
    for _ in range(max(args.warmup, 0)):
        cpu_reference(args, 0.02, nth)
    vals = []
    t0 = time.perf_counter()
    samples = None
    for _ in range(args.steps):
        v, samples = cpu_reference(args, args.cpu_seconds / 4, nth)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    n_step = sum(n for _, _, n in step_units(args, world))
    sample = (f"fp64 oracle port of the reference CPU path (proj/src/{{sphere,gtp,cgtp,mtp}}.cpp) on {nth} threads, "
              f"per-(kind, L) samples {samples}, scaled to the step's products")
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(n_step * world / value * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if args.workload == "c4" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic N(0,1), seed {SEED}", "config": workload_config(args, world), "impl": "reference",
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": nth, "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 2),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
