#!/usr/bin/env python
"""Benchmark of the TPO hot path (BASELINE.json metric: tensor products/sec vs
L_max, % of roofline).

Workload (BASELINE.json configs[1]): S2-grid Gaunt TP, L_max sweep 1..10,
batch 65,536 x 1 channel per GPU, L3 = 2L.  One step = one pass of the sweep
(ten launches of the fused tcgen05 kernel, one per L) over inputs resident in
HBM, captured once into a CUDA graph and replayed (no host launch gaps in the
device time).  L2 (126 MB) is flushed between steps by writing a 256 MiB
buffer; the flush is outside the CUDA-event-timed region.  Multi-GPU (torchrun): every
rank processes its own 65,536-sample shard (weak scaling, no collective on
the data path); per-rank device times are max-reduced and a per-shard
checksum is all-gathered after the timed region.

`--impl reference` times the reference CPU algorithm instead: the fp64 oracle
port of proj/src/{sphere,gtp}.cpp (the reference itself cannot be built here,
Eigen 3 is missing) on all host cores, on a bounded sample of the same sweep.
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
LS = list(range(1, 11))
BATCH = 65536


def grid_flops_per_tp(L: int) -> int:
    """Dense-GEMM algorithmic flops of one grid GTP:
    2 G (2 Din + Dout), G = (2L+1)(4L+1) product-grid points."""
    G = (2 * L + 1) * (4 * L + 1)
    return 2 * G * (2 * (L + 1) ** 2 + (2 * L + 1) ** 2)


def grid_bytes_per_tp(L: int) -> int:
    return 4 * (2 * (L + 1) ** 2 + (2 * L + 1) ** 2)


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region.

    NVML is polled from a thread every ~0.2 ms (nvidia-smi's 20 ms cadence and
    process start-up miss a few-ms region entirely); only samples taken while a
    region is open (``with clk.region():``) are summarised.  Falls back to
    ``nvidia-smi -lms 20`` when NVML is unavailable."""

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
        self.samples: list[tuple[float, set]] = []  # (sm MHz, reasons) inside open regions
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
        try:  # fallback: nvidia-smi loop
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
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference(Ls, seconds_per_L: float, nthreads: int, steps: int = 1):
    """Reference CPU algorithm (fp64 oracle port of the grid GTP) on host cores.
    Returns (TP/s over the sweep, sample description)."""
    import numpy as np

    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # noqa: E402  (allowed here: the CPU baseline leg)

    rng = np.random.default_rng(SEED)
    per_tp = {}
    samples = {}
    for L in Ls:
        d = (L + 1) ** 2
        n = max(nthreads, 64)
        while True:
            x = rng.standard_normal((n, 1, d))
            y = rng.standard_normal((n, 1, d))
            t0 = time.perf_counter()
            for _ in range(steps):
                oracle.batch_mimo("gtp_grid", L, x, y, nthreads=nthreads)
            dt = (time.perf_counter() - t0) / steps
            if dt >= seconds_per_L or n >= BATCH:
                break
            n = min(BATCH, int(n * max(2.0, 1.2 * seconds_per_L / max(dt, 1e-6))))
        per_tp[L] = dt / n
        samples[L] = n
    # whole sweep with BATCH TPs per L, as on the GPU
    sweep_time = sum(BATCH * per_tp[L] for L in Ls)
    value = len(Ls) * BATCH / sweep_time
    return value, samples, per_tp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--cpu-seconds", type=float, default=1.0, help="CPU baseline seconds per L")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the per-kind side measurements")
    ap.add_argument("--serial-sweep", action="store_true",
                    help="capture the 10 launches in stream order instead of as parallel graph branches")
    ap.add_argument("--no-graph", action="store_true",
                    help="eager launches instead of CUDA-graph replay (for ncu launch lists; ncu cannot replay "
                         "kernels inside stream capture)")
    args = ap.parse_args()
    world, rank, local = dist_setup()

    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import numpy as np
    import torch

    import paper_2506_13523_b200 as tpo

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    ctx = tpo.context(local)
    stream = torch.cuda.current_stream(dev)
    B = args.batch
    g = torch.Generator(device=dev)
    g.manual_seed(SEED + 1000 * rank)
    xs = {L: torch.randn((B, (L + 1) ** 2), generator=g, device=dev) for L in LS}
    ys = {L: torch.randn((B, (L + 1) ** 2), generator=g, device=dev) for L in LS}
    outs = {L: torch.empty((B, (2 * L + 1) ** 2), device=dev) for L in LS}
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    def sweep(Ls):
        for L in Ls:
            tpo.gtp_grid(xs[L], ys[L], L, L, 2 * L, out=outs[L])

    # eager warm-up builds the device tables, then the sweep (and each L on its
    # own, for the per-L breakdown) is captured into CUDA graphs
    sweep(LS)
    torch.cuda.synchronize()
    launches0 = ctx.launches
    if args.no_graph:
        class _Eager:  # same interface as a captured graph
            def __init__(self, Ls):
                self.Ls = Ls

            def replay(self):
                sweep(self.Ls)

        graph = _Eager(LS)
        sweep(LS)
        launches_per_step = ctx.launches - launches0
        graphs_L = {L: _Eager([L]) for L in LS}
    else:
        # The ten L problems are independent (own inputs and outputs), so by default they
        # are captured as parallel graph branches, largest L first: each kernel's CTAs
        # (persistent, static tile ranges; 512 tiles on 148 SMs leave ~13% of the SMs idle
        # during a launch's last wave) are followed on the freed SMs by the next problem's
        # CTAs.  Outputs are bit-identical to the serial order (tools/sweep_concurrent.py).
        graph = torch.cuda.CUDAGraph()
        side = [torch.cuda.Stream(dev) for _ in LS]
        with torch.cuda.graph(graph):
            if args.serial_sweep:
                sweep(LS)
            else:
                cap = torch.cuda.current_stream(dev)
                fork = torch.cuda.Event()
                fork.record(cap)
                joins = []
                for s_, L in zip(side, sorted(LS, reverse=True)):
                    s_.wait_event(fork)
                    with torch.cuda.stream(s_):
                        sweep([L])
                    e = torch.cuda.Event()
                    e.record(s_)
                    joins.append(e)
                for e in joins:
                    cap.wait_event(e)
        launches_per_step = ctx.launches - launches0
        graphs_L = {}
        for L in LS:
            graphs_L[L] = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graphs_L[L]):
                sweep([L])
    torch.cuda.synchronize()

    per_L = {L: 0.0 for L in LS}
    total_ms = 0.0
    with ClockSampler(local) as clk:
        for _ in range(max(args.warmup, 3)):
            graph.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with clk.region():
            for _ in range(args.steps):
                flush.zero_()  # evict L2 (untimed)
                ev0.record(stream)
                graph.replay()
                ev1.record(stream)
                ev1.synchronize()
                total_ms += ev0.elapsed_time(ev1)
            torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        # per-L breakdown (outside the headline timing; same flush discipline)
        with clk.region():
            for L in LS:
                for _ in range(max(3, args.steps // 5)):
                    flush.zero_()
                    ev0.record(stream)
                    graphs_L[L].replay()
                    ev1.record(stream)
                    ev1.synchronize()
                    per_L[L] += ev0.elapsed_time(ev1) / max(3, args.steps // 5) * args.steps
    launches = launches_per_step * args.steps
    from paper_2506_13523_b200.dist import gather_checksums, max_over_ranks

    total_ms = max_over_ranks(total_ms, dev)  # device time, max over ranks
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms_per_step = total_ms / args.steps
    value = world * len(LS) * B / (ms_per_step / 1e3)

    # result gather after the timed region: per-shard checksums over NCCL
    checks = gather_checksums(torch.stack([outs[L].double().sum() for L in LS]), dev)

    peaks = load_peaks()
    tc_peak = peaks["bf16_tflops"] / 3.0  # 3xFP16 split on the fp16/bf16 tensor pipe
    per = {}
    for L in LS:
        ms = per_L[L] / args.steps
        fl = grid_flops_per_tp(L) * B
        by = grid_bytes_per_tp(L) * B
        tf = fl / (ms / 1e3) / 1e12
        gbs = by / (ms / 1e3) / 1e9
        t_roof = max(by / (peaks["hbm_gbs"] * 1e9), fl / (tc_peak * 1e12))
        per[str(L)] = {"ms": round(ms, 5), "tp_per_s": round(B / (ms / 1e3), 1), "tflops": round(tf, 2),
                       "gbs": round(gbs, 1), "roofline_frac": round(t_roof / (ms / 1e3), 4)}
    # dominant kernel = largest share of the step
    domL = max(LS, key=lambda L: per_L[L])
    dom_ms = per_L[domL] / args.steps
    traffic = None
    tf_path = ROOT / "profiles" / "ncu_traffic.json"
    if tf_path.exists():
        try:
            traffic = json.loads(tf_path.read_text()).get(f"gtp_grid_L{domL}")
        except Exception:
            traffic = None
    roofline = {
        "bound": "tensor",
        "kernel": f"gtp_grid_tc_kernel L={domL} (3xFP16 tcgen05)",
        "achieved": round(grid_flops_per_tp(domL) * B / (dom_ms / 1e3) / 1e12, 2),
        "peak": round(tc_peak, 1),
        "unit": "TFLOP/s",
        "frac": round(grid_flops_per_tp(domL) * B / (dom_ms / 1e3) / 1e12 / tc_peak, 4),
        "traffic": traffic,
        "peak_note": f"{peaks['source']} bf16 tensor peak {peaks['bf16_tflops']} TF/s / 3 (3xFP16 split); "
                     f"algorithmic flops = dense 2*G*(2Din+Dout) per TP x {B} TPs per launch",
        "share_of_step": round(dom_ms / ms_per_step, 3),
    }

    # e2e through the C ABI with host buffers (pinned), H2D + kernel + D2H per step
    e2e = None
    if rank == 0 or world > 1:
        import ctypes as C

        hx = {L: xs[L].cpu().pin_memory() for L in LS}
        hy = {L: ys[L].cpu().pin_memory() for L in LS}
        ho = {L: torch.empty(outs[L].shape, pin_memory=True) for L in LS}
        lib = tpo.lib()

        def e2e_step_per_call():  # one synchronous tpo_run_host_f32 per L
            for L in LS:
                tpo.check(lib.tpo_run_host_f32(ctx.handle, tpo.KINDS["gtp_grid"], L, L, 2 * L, -1,
                                               hx[L].data_ptr(), hy[L].data_ptr(), ho[L].data_ptr(), B, 1, 0))

        reqs = [("gtp_grid", hx[L], hy[L], ho[L], L, L, 2 * L) for L in LS]

        def e2e_step_batch():  # the sweep's 10 requests in one tpo_run_host_batch_f32 call
            tpo.run_host_batch(reqs, local)

        n_e2e = max(2, min(args.steps, 5))

        def timed(fn):
            for _ in range(2):
                fn()
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                fn()
            return max_over_ranks((time.perf_counter() - t0) / n_e2e, dev)

        et_call = timed(e2e_step_per_call)
        et = timed(e2e_step_batch)
        e2e = {"value": round(world * len(LS) * B / et, 1), "unit": UNIT,
               "h2d_bytes_per_step": int(sum(2 * B * (L + 1) ** 2 * 4 for L in LS)),
               "d2h_bytes_per_step": int(sum(B * (2 * L + 1) ** 2 * 4 for L in LS)),
               "ms_per_step": round(et * 1e3, 3),
               "path": "tpo_run_host_batch_f32 (C ABI, pinned host buffers, the 10 requests in one call)",
               "per_call": {"value": round(world * len(LS) * B / et_call, 1), "ms_per_step": round(et_call * 1e3, 3),
                            "path": "one tpo_run_host_f32 per L"}}

    extras = None
    if not args.no_extras and rank == 0:
        extras = side_measurements(tpo, dev, stream, flush, load_peaks())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nth = os.cpu_count() or 1
        v, samples, _ = cpu_reference(LS, args.cpu_seconds, nth)
        cpu = {"value": round(v, 1), "unit": UNIT, "cores": nth, "kind": "port",
               "sample": f"fp64 oracle port of gtp_grid_select, L=1..10, per-L samples {samples}, "
                         f"scaled to {B} TPs per L"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (3xFP16 tcgen05, fp32 accumulate)",
            "data": f"synthetic N(0,1) irreps on device, seed {SEED}+1000*rank",
            "config": {"workload": "S2-grid GTP L_max sweep 1-10, batch 65536 x 1 channel per GPU, L3=2L "
                                   "(BASELINE.json configs[1])",
                       "batch_per_gpu": B, "L": LS, "l2": "flushed between steps (256 MiB write, untimed)",
                       "parallelism": f"dp{world} (independent shards, no data-path collective)"},
            "per_L": per, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "wall_s_timed": round(wall, 3), "checksums": checks,
            "timing": "CUDA graph of the 10-launch sweep replayed per step; CUDA events on the replay stream; "
                      "L2 flushed (256 MiB write) before every step, outside the events",
            "sweep_launch": ("10 launches in stream order" if args.serial_sweep or args.no_graph else
                             "10 independent launches as parallel CUDA-graph branches (L descending); "
                             "--serial-sweep for stream order"),
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def side_measurements(tpo, dev, stream, flush, peaks):
    """Throughput and roofline fraction of the other kinds at their BASELINE configs (device time,
    one launch, L2 flushed).  Bounds: dense GEMM flops on the 3xFP16 tensor peak
    for the tcgen05 kinds, HBM bytes for CGTP, max(HBM, FP32 SIMT) for the SIMT MTP."""
    import torch

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream); fn(); b.record(stream); b.synchronize()
            tot += a.elapsed_time(b)
        return tot / reps

    tc_peak = peaks["bf16_tflops"] / 3.0 * 1e12
    hbm = peaks["hbm_gbs"] * 1e9
    fp32 = 2 * 148 * 128 * 1.965e9  # FFMA peak (nominal clock; not in MEASURED_PEAKS.json)
    res = {}
    g = torch.Generator(device=dev); g.manual_seed(7)
    L, B = 6, 65536
    din, dout = (L + 1) ** 2, (2 * L + 1) ** 2
    byts = 4 * (2 * din + dout) * B
    x = torch.randn((B, din), generator=g, device=dev)
    y = torch.randn((B, din), generator=g, device=dev)
    o = torch.empty((B, dout), device=dev)
    for kind in ("gtp_grid", "gtp_fourier", "mtp"):
        ms = timeit(lambda: tpo.run(kind, x, y, L, L, 2 * L, out=o))
        t = ms / 1e3
        if kind == "gtp_grid":
            G = (2 * L + 1) * (4 * L + 1)
            fl = 2 * G * (2 * din + dout) * B
            roof = max(byts / hbm, fl / tc_peak)
            bound = "tensor (dense S2-grid operators, 3xFP16)"
        elif kind == "gtp_fourier":
            N = 4 * L + 2  # torus points per axis; antipodal pairs folded: N^2 / 2 points
            fl = 2 * (N * N // 2) * (2 * din + dout) * B
            roof = max(byts / hbm, fl / tc_peak)
            bound = "tensor (dense torus operators on the N^2/2 antipodal-pair points, 3xFP16)"
        else:
            fl = 2 * 6378 * B  # 2 x reference sparse muls
            roof = max(byts / hbm, fl / fp32)
            bound = "max(HBM, FP32 at the reference sparse op count, nominal clock)"
        res[f"{kind}_L{L}_B{B}"] = {"ms": round(ms, 4), "tp_per_s": round(B / t, 1), "tflops": round(fl / t / 1e12, 2),
                                     "gbs": round(byts / t / 1e9, 1), "roofline_frac": round(roof / t, 4), "bound": bound}
    # channel-wise CGTP, config C4 shape (L=3, 128 channels, y shared per edge) on a 2^14-edge chunk
    L, C, B = 3, 128, 1 << 14
    x = torch.randn((B, C, 16), generator=g, device=dev)
    y = torch.randn((B, 16), generator=g, device=dev)
    o = torch.empty((B, C, 256), device=dev)
    ms = timeit(lambda: tpo.cgtp(x, y, L, L, out=o))
    byts = B * (C * 16 * 4 + 16 * 4 + C * 256 * 4)
    res[f"cgtp_L3_C128_B{B}"] = {"ms": round(ms, 4), "edges_per_s": round(B / ms * 1e3, 1),
                                  "channel_tp_per_s": round(B * C / ms * 1e3, 1),
                                  "gbs": round(byts / ms / 1e6, 1), "roofline_frac": round(byts / hbm / (ms / 1e3), 4),
                                  "bound": "HBM (139,328 B per edge)"}
    # general CGTP at L=6 (per-(l1, l2) block GEMMs on tcgen05): output-write bound
    L, B = 6, 65536
    din, dout = (L + 1) ** 2, (L + 1) ** 4
    x = torch.randn((B, din), generator=g, device=dev)
    y = torch.randn((B, din), generator=g, device=dev)
    o = torch.empty((B, dout), device=dev)
    ms = timeit(lambda: tpo.cgtp(x, y, L, L, out=o))
    byts = 4 * (2 * din + dout) * B
    res[f"cgtp_L{L}_B{B}"] = {"ms": round(ms, 4), "tp_per_s": round(B / ms * 1e3, 1), "gbs": round(byts / ms / 1e6, 1),
                              "roofline_frac": round(byts / hbm / (ms / 1e3), 4), "bound": "HBM"}
    del o
    # backward (tpo_backward_f32: grad_x and grad_y) of each kind at L=6, batch 65536
    bwd = {}
    for kind in ("gtp_grid", "gtp_fourier", "mtp", "cgtp"):
        dout = (L + 1) ** 4 if kind == "cgtp" else (2 * L + 1) ** 2
        go = torch.randn((B, dout), generator=g, device=dev)
        ms = timeit(lambda: tpo.backward(kind, x, y, go, L, L, 2 * L))
        byts = 4 * (4 * din + dout) * B  # read x, y, grad_out; write grad_x, grad_y
        bwd[f"{kind}_L{L}_B{B}"] = {"ms": round(ms, 4), "tp_per_s": round(B / ms * 1e3, 1),
                                    "gbs": round(byts / ms / 1e6, 1),
                                    "hbm_frac": round(byts / hbm / (ms / 1e3), 4)}
        del go
    res["backward"] = bwd
    return res


def run_reference(args, world, rank):
    if world > 1 and rank != 0:
        return
    nth = os.cpu_count() or 1
    # warm the table caches (untimed), then K steps of a bounded sample
    cpu_reference(LS, 0.01, nth)
    vals = []
    t0 = time.perf_counter()
    for _ in range(max(args.warmup, 0)):
        cpu_reference(LS, 0.05, nth)
    for _ in range(args.steps):
        v, samples, _ = cpu_reference(LS, args.cpu_seconds / 4, nth)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    sample = (f"fp64 oracle port of gtp_grid_select (reference CPU algorithm, proj/src/sphere.cpp + gtp.cpp), "
              f"L=1..10, per-L samples {samples}, scaled to {BATCH} TPs per L")
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(len(LS) * BATCH / value * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": f"synthetic N(0,1), seed {SEED}",
        "config": {"workload": "S2-grid GTP L_max sweep 1-10, batch 65536 x 1 channel (BASELINE.json configs[1])",
                   "batch_per_gpu": BATCH, "L": LS},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": nth, "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 2),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
