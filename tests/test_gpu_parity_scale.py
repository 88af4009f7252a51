"""GPU parity at the bench scale and under adversarial dynamic range.

1. Bench-scale oracle parity.  The persistent tcgen05
   kernels give each CTA a contiguous range of (tile, output group) units; a
   batch of 148*128*4+77 rows makes every CTA run several units, so the
   multi-unit hand-offs (next-tile raw prefetch, the in-place XY_FREE hand-off,
   Z_EMPTY and ring phases across units, the 2-group split at L=10) and the
   ragged last tile are all exercised.  A strided subsample of >= 4096 rows
   (plus the whole tail tile) is checked against the fp64 oracle
   (oracle.batch_mimo = proj/src/gtp.cpp:228-327, mtp.cpp:99-117,
   cgtp.cpp:145-177) at the 1e-5 normwise contract.

2. Adversarial precision.  The 3xFP16 split scales whole
   rows by powers of two, so dynamic range INSIDE a row is the hard case: the
   fp16 lo parts of small coefficients go subnormal.  Every kind at L=1..14 is
   checked on rows whose degrees decay as 10^(-l/2), grow towards the top
   degree, have one dominant degree, exact zeros, per-coefficient magnitudes
   spread over six decades, and whole rows scaled by 1e+-18..20 (outputs kept
   inside the fp32 normal range, which is the contract's representable set).
   The worst error per (kind, L) is written to gpurun_out/precision_table.json.
"""
import json
from pathlib import Path

import numpy as np
import pytest

TOL = 1e-5
pytestmark = pytest.mark.gpu

BIG = 148 * 128 * 4 + 77  # 4+ units per CTA on 148 SMs, ragged tail of 77 rows


@pytest.fixture(scope="module")
def tpo():
    import torch

    assert torch.cuda.is_available()
    import paper_2506_13523_b200 as m

    return m


def _normwise_rows(out, ref):
    out = out.reshape(-1, out.shape[-1]).astype(np.float64)
    ref = ref.reshape(-1, ref.shape[-1])
    scale = np.maximum(np.abs(ref).max(axis=1), 1e-300)
    return np.abs(out - ref).max(axis=1) / scale


def _subsample(B, n=4096):
    idx = np.unique(np.concatenate([np.linspace(0, B - 1, n).astype(np.int64), np.arange(max(0, B - 128), B)]))
    return idx


def _run_big(tpo, orc, kind, L, B, seed, path=None):
    import torch

    ctx = tpo.context()
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    d = (L + 1) ** 2
    x = torch.randn((B, d), generator=g, device="cuda")
    y = torch.randn((B, d), generator=g, device="cuda")
    L3 = 0 if kind == "cgtp" else 2 * L
    if path:
        ctx.set_grid_path(path)
    try:
        out = tpo.run(kind, x, y, L, L, L3)
        used = ctx.last_grid_path
    finally:
        if path:
            ctx.set_grid_path("auto")
    idx = torch.from_numpy(_subsample(B)).cuda()
    xs = x[idx].cpu().numpy().astype(np.float64)
    ys = y[idx].cpu().numpy().astype(np.float64)
    os_ = out[idx].cpu().numpy()
    assert torch.isfinite(out).all().item()
    ref = orc.batch_mimo(kind, L, xs[:, None], ys[:, None])[:, 0]
    err = float(_normwise_rows(os_, ref).max())
    return err, used


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier"])
@pytest.mark.parametrize("L", list(range(1, 13)))
def test_gtp_tcgen05_bench_scale(tpo, orc, kind, L):
    err, used = _run_big(tpo, orc, kind, L, BIG, 9000 + L + (100 if kind == "gtp_fourier" else 0), path="tc")
    assert used == "tcgen05"
    assert err <= TOL, (kind, L, err)


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier"])
@pytest.mark.parametrize("L", [13, 14])
def test_gtp_degree_groups_bench_scale(tpo, orc, kind, L):
    err, used = _run_big(tpo, orc, kind, L, BIG // 2, 9200 + L + (100 if kind == "gtp_fourier" else 0), path="tc")
    assert used == "tcgen05"
    assert err <= TOL, (kind, L, err)


def test_gtp_bench_config_exact(tpo, orc):
    # the bench's own configuration: 65,536 rows per L (512 tiles, 3-4 units per CTA; 2 output
    # groups at L = 10), checked on the subsample for every L of the sweep
    worst = {}
    for L in range(1, 11):
        err, used = _run_big(tpo, orc, "gtp_grid", L, 65536, 20240901 + L)
        assert used == ("small" if L == 1 else "tcgen05")
        worst[L] = err
    assert max(worst.values()) <= TOL, worst


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier"])
@pytest.mark.parametrize("L", [1])
def test_gtp_small_degree_simt(tpo, orc, kind, L):
    # L1 = L2 = 1, L3 = 2 runs on the small-degree SIMT kernel (gtp_small.cu) in "auto" mode:
    # several tiles per block, ragged tail
    err, used = _run_big(tpo, orc, kind, L, BIG, 9600 + L + (100 if kind == "gtp_fourier" else 0))
    assert used == "small"
    assert err <= TOL, (kind, L, err)


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier"])
def test_gtp_small_shared_y_matches_tcgen05(tpo, kind):
    # shared y (one per batch entry across channels) and L3 < 2L shapes: the small kernel against
    # the tcgen05 kernel (both oracle-checked above) on the same inputs
    import torch

    ctx = tpo.context()
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    L, B, C = 1, 333, 7
    x = torch.randn((B, C, (L + 1) ** 2), generator=g, device="cuda")
    y = torch.randn((B, (L + 1) ** 2), generator=g, device="cuda")
    a = tpo.run(kind, x, y, L, L, 2 * L)
    assert ctx.last_grid_path == "small"
    ctx.set_grid_path("tc")
    try:
        b = tpo.run(kind, x, y, L, L, 2 * L)
        assert ctx.last_grid_path == "tcgen05"
    finally:
        ctx.set_grid_path("auto")
    err = float(_normwise_rows(a.cpu().numpy(), b.double().cpu().numpy()).max())
    assert err <= 2 * TOL, err
    tpo.run(kind, x, y, L, L, 3)  # L3 != 2L: not a small-kernel shape
    assert ctx.last_grid_path == "tcgen05"


@pytest.mark.parametrize("L", [15, 16])
def test_fourier_degree_groups_high_L(tpo, orc, L):
    # L = 15, 16 Fourier GTP on tcgen05 degree groups (forced; automatic selection takes the
    # separable torus kernel from L = 13)
    err, used = _run_big(tpo, orc, "gtp_fourier", L, 148 * 128 // 4 + 77, 9300 + L, path="tc")
    assert used == "tcgen05"
    assert err <= TOL, (L, err)


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier"])
@pytest.mark.parametrize("L", [11, 12, 13, 14, 15, 16])
def test_gtp_separable_bench_scale(tpo, orc, kind, L):
    # the automatic path from L = 11: the row-quad separable kernels (grid nodes / reference torus)
    err, used = _run_big(tpo, orc, kind, L, 148 * 128 + 77, 9400 + L + (100 if kind == "gtp_fourier" else 0))
    assert used == ("simt" if kind == "gtp_grid" else "separable")
    assert err <= TOL, (kind, L, err)


def test_cgtp_blocks_L15(tpo, orc):
    # CGTP block GEMMs at L = 15 (several tiles per CTA, ragged tail)
    err, _ = _run_big(tpo, orc, "cgtp", 15, 128 * 3 + 5, 9415)
    assert err <= TOL, err


def test_cgtp_block_y_segments_forced_small_L(tmp_path):
    # the per-block y staging of the CGTP block kernel (default from L2 = 13) forced down to L = 4..6
    # (TPO_CGTP_YSEG_MIN is read once per process: a child process), against the oracle
    import subprocess
    import sys
    import textwrap

    code = textwrap.dedent("""
        import sys, numpy as np, torch
        sys.path.insert(0, %r); sys.path.insert(0, %r)
        import paper_2506_13523_b200 as tpo, oracle as orc
        orc.build()
        worst = 0.0
        for L, B in ((4, 300), (5, 131), (6, 77)):
            g = torch.Generator(device="cuda"); g.manual_seed(70 + L)
            d = (L + 1) ** 2
            x = torch.randn((B, d), generator=g, device="cuda"); y = torch.randn((B, d), generator=g, device="cuda")
            out = tpo.run("cgtp", x, y, L, L, 0).cpu().numpy().astype(np.float64)
            ref = orc.batch_mimo("cgtp", L, x.cpu().numpy().astype(np.float64)[:, None],
                                 y.cpu().numpy().astype(np.float64)[:, None])[:, 0]
            err = (np.abs(out - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)).max()
            worst = max(worst, float(err))
        print("WORST", worst)
    """ % (str(Path(__file__).resolve().parents[1]), str(Path(__file__).resolve().parents[1] / "oracle")))
    env = dict(__import__("os").environ, TPO_CGTP_YSEG_MIN="16")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    worst = float(r.stdout.strip().split("WORST")[-1])
    assert worst <= TOL, worst


@pytest.mark.parametrize("L", [1, 3, 6, 7, 10])
def test_mtp_bench_scale(tpo, orc, L):
    err, _ = _run_big(tpo, orc, "mtp", L, BIG, 9400 + L)
    assert err <= TOL, (L, err)


@pytest.mark.parametrize("L", [3, 6])
def test_cgtp_bench_scale(tpo, orc, L):
    err, _ = _run_big(tpo, orc, "cgtp", L, BIG if L <= 3 else BIG // 4, 9500 + L)
    assert err <= TOL, (L, err)


# ---------------------------------------------------------------- adversarial dynamic range
def _degree_of_cols(L):
    return np.concatenate([np.full(2 * l + 1, l) for l in range(L + 1)])


def adversarial_rows(L, rng, per=6):
    """Pairs (x, y) [n, (L+1)^2] fp32 with dynamic range inside each row."""
    d = (L + 1) ** 2
    deg = _degree_of_cols(L)
    xs, ys, names = [], [], []

    def add(name, fx, fy):
        for _ in range(per):
            x = rng.standard_normal(d) * fx()
            y = rng.standard_normal(d) * fy()
            xs.append(x); ys.append(y); names.append(name)

    one = lambda: np.ones(d)  # noqa: E731
    decay = lambda: 10.0 ** (-deg / 2.0)  # noqa: E731
    grow = lambda: 10.0 ** (-(L - deg) / 2.0)  # noqa: E731

    def dominant():
        s = np.full(d, 1e-3)
        s[deg == rng.integers(0, L + 1)] = 1.0
        return s

    def zeros():
        s = (rng.random(d) < 0.5).astype(np.float64)
        s[deg == rng.integers(0, L + 1)] = 0.0
        return s

    spread = lambda: 10.0 ** rng.uniform(-6, 0, d)  # noqa: E731
    add("decay", decay, decay)
    add("grow", grow, grow)
    add("decay_x_grow_y", decay, grow)
    add("dominant_degree", dominant, dominant)
    add("exact_zeros", zeros, zeros)
    add("six_decades", spread, spread)
    add("rows_1e20_1e-20", lambda: 1e20 * one(), lambda: 1e-20 * one())
    add("rows_1e-18_1e18", lambda: 1e-18 * one(), lambda: 1e18 * one())
    add("rows_1e15_1e15", lambda: 1e15 * one(), lambda: 1e15 * one())
    add("rows_1e-15_1e-3", lambda: 1e-15 * one(), lambda: 1e-3 * one())
    # whole-zero rows: output must be exactly zero
    xs.append(np.zeros(d)); ys.append(rng.standard_normal(d)); names.append("zero_row")
    return np.stack(xs).astype(np.float32), np.stack(ys).astype(np.float32), names


_TABLE = {}


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier", "mtp", "cgtp"])
@pytest.mark.parametrize("L", list(range(1, 17)))
def test_adversarial_precision(tpo, orc, kind, L):
    import torch

    rng = np.random.default_rng(31337 + 17 * L)
    x, y, names = adversarial_rows(L, rng, per=4 if L >= 12 else 6)
    L3 = 0 if kind == "cgtp" else 2 * L
    out = tpo.run(kind, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), L, L, L3).cpu().numpy()
    ref = orc.batch_mimo(kind, L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
    assert np.isfinite(out).all()
    zero_rows = [i for i, n in enumerate(names) if n == "zero_row"]
    assert np.all(out[zero_rows] == 0.0)
    err = _normwise_rows(out, ref)
    per_case = {}
    for n, e in zip(names, err):
        per_case[n] = max(per_case.get(n, 0.0), float(e))
    _TABLE[f"{kind}_L{L}"] = {"worst": float(err.max()), "path": tpo.context().last_grid_path
                              if kind.startswith("gtp") else None, "cases": per_case}
    out_dir = Path(__file__).resolve().parents[1] / "gpurun_out"
    if out_dir.exists():
        (out_dir / "precision_table.json").write_text(json.dumps(_TABLE, indent=1, sort_keys=True))
    assert float(err.max()) <= TOL, (kind, L, {k: v for k, v in per_case.items() if v > TOL})


@pytest.mark.parametrize("kind,L", [("gtp_grid", 8), ("gtp_grid", 10), ("gtp_fourier", 10)])
def test_strict_precision_mode(tpo, orc, kind, L):
    # tpo_set_precision(ctx, 1): segmented accumulation for every chain past 20 K-steps
    import torch

    ctx = tpo.context()
    prev = ctx.set_precision("strict")
    try:
        rng = np.random.default_rng(4242 + L)
        x, y, names = adversarial_rows(L, rng, per=6)
        out = tpo.run(kind, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), L, L, 2 * L).cpu().numpy()
        ref = orc.batch_mimo(kind, L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
        assert float(_normwise_rows(out, ref).max()) <= 5e-6
    finally:
        ctx.set_precision(prev)
