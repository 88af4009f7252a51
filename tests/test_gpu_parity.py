"""GPU parity: every kernel through the C ABI vs the fp64 CPU oracle.

Contract (north star / SURVEY.md 8(d)): per tensor product, normwise
max|gpu - ref| / max|ref| <= 1e-5 with the oracle evaluated in fp64 on the
same fp32-rounded inputs.
"""
import math

import numpy as np
import pytest

TOL = 1e-5  # normwise relative error per TP, fp32 contract

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tpo():
    import torch

    assert torch.cuda.is_available()
    import paper_2506_13523_b200 as m

    return m


def _inputs(B, L1, L2, seed, C=None, shared=False):
    rng = np.random.default_rng(seed)
    if C is None:
        x = rng.standard_normal((B, (L1 + 1) ** 2)).astype(np.float32)
        y = rng.standard_normal((B, (L2 + 1) ** 2)).astype(np.float32)
    else:
        x = rng.standard_normal((B, C, (L1 + 1) ** 2)).astype(np.float32)
        y = rng.standard_normal((B, (L2 + 1) ** 2) if shared else (B, C, (L2 + 1) ** 2)).astype(np.float32)
    return x, y


def _gpu(tpo, kind, x, y, L1, L2, L3, lt=-1):
    import torch

    xt = torch.from_numpy(x).cuda()
    yt = torch.from_numpy(y).cuda()
    out = tpo.run(kind, xt, yt, L1, L2, L3, lt)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def _ref_single(orc, kind, x, y, L1, L2, L3, lt=-1):
    t1, t2 = orc.tower(L1), orc.tower(L2)
    x = x.astype(np.float64); y = y.astype(np.float64)
    if kind == "cgtp":
        return orc.cgtp_mimo(t1, x, t2, y)
    if kind == "gtp_grid":
        return orc.gtp_grid(t1, x, t2, y, L3)
    if kind == "gtp_fourier":
        return orc.gtp_fourier(t1, x, t2, y, L3)
    return orc.mtp(t1, x, t2, y, L3, lt_override=lt)


def _normwise(out, ref):
    out = out.reshape(-1, out.shape[-1]); ref = ref.reshape(-1, ref.shape[-1])
    scale = np.maximum(np.abs(ref).max(axis=1), 1e-300)
    return float((np.abs(out - ref).max(axis=1) / scale).max())


def _check_batch(tpo, orc, kind, L, B, seed, L3=None):
    L3 = 2 * L if L3 is None else L3
    x, y = _inputs(B, L, L, seed)
    out = _gpu(tpo, kind, x, y, L, L, L3)
    ref = orc.batch_mimo(kind, L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
    err = _normwise(out, ref)
    assert err <= TOL, (kind, L, err)
    return err


# ---------------------------------------------------------------- per kind, L sweep
@pytest.mark.parametrize("L", list(range(0, 13)))
def test_gtp_grid_tcgen05(tpo, orc, L):
    ctx = tpo.context()
    ctx.set_grid_path("tc")
    try:
        _check_batch(tpo, orc, "gtp_grid", L, 1000, 100 + L)
        assert ctx.last_grid_path == "tcgen05"
    finally:
        ctx.set_grid_path("auto")


@pytest.mark.parametrize("L", [1, 3, 6, 11, 13, 16])
def test_gtp_grid_simt(tpo, orc, L):
    ctx = tpo.context()
    ctx.set_grid_path("simt")
    try:
        _check_batch(tpo, orc, "gtp_grid", L, 64 if L > 10 else 300, 200 + L)
        assert ctx.last_grid_path == "simt"
    finally:
        ctx.set_grid_path("auto")


@pytest.mark.parametrize("L1,L2,L3,B,C,shared", [
    (0, 0, 0, 7, None, False),     # band 0: one node, one azimuth
    (3, 2, 4, 13, None, False),    # odd band: no middle node; truncated output
    (2, 5, 9, 6, None, False),     # L2 > L1, output past the band (zero degrees)
    (5, 0, 5, 5, None, False),     # y a scalar
    (4, 4, 3, 3, 3, True),         # shared y over channels, rows not a multiple of 4
    (6, 3, 9, 2, 5, False),
])
def test_gtp_grid_simt_shapes(tpo, orc, L1, L2, L3, B, C, shared):
    # the row-quad separable kernel: folded theta / phi symmetries at odd and even bands, ragged
    # row quads, shared y
    ctx = tpo.context()
    ctx.set_grid_path("simt")
    try:
        x, y = _inputs(B, L1, L2, 17 * L1 + 5 * L2 + L3, C, shared)
        out = _gpu(tpo, "gtp_grid", x, y, L1, L2, L3)
        assert ctx.last_grid_path == "simt"
    finally:
        ctx.set_grid_path("auto")
    xs = x.reshape(-1, x.shape[-1])
    ys = np.repeat(y, C, axis=0) if shared else y.reshape(-1, y.shape[-1])
    ref = np.stack([_ref_single(orc, "gtp_grid", xs[i], ys[i], L1, L2, L3) for i in range(xs.shape[0])])
    assert _normwise(out.reshape(ref.shape), ref) <= TOL


@pytest.mark.parametrize("L", [0, 1, 2, 3, 5, 8, 11, 13, 16])
def test_gtp_fourier_separable(tpo, orc, L):
    # the reference torus evaluated separably on the row-quad kernel (forced at every L)
    ctx = tpo.context()
    ctx.set_grid_path("sep")
    try:
        _check_batch(tpo, orc, "gtp_fourier", L, 64 if L > 10 else 203, 250 + L)
        assert ctx.last_grid_path == "separable"
    finally:
        ctx.set_grid_path("auto")


@pytest.mark.parametrize("L1,L2,L3,B,C,shared", [
    (0, 0, 0, 7, None, False),
    (3, 2, 4, 13, None, False),
    (2, 5, 9, 6, None, False),
    (5, 0, 5, 5, None, False),
    (4, 4, 3, 3, 3, True),
    (6, 3, 11, 2, 5, False),
])
def test_gtp_fourier_separable_shapes(tpo, orc, L1, L2, L3, B, C, shared):
    ctx = tpo.context()
    ctx.set_grid_path("sep")
    try:
        x, y = _inputs(B, L1, L2, 19 * L1 + 5 * L2 + L3, C, shared)
        out = _gpu(tpo, "gtp_fourier", x, y, L1, L2, L3)
        assert ctx.last_grid_path == "separable"
    finally:
        ctx.set_grid_path("auto")
    xs = x.reshape(-1, x.shape[-1])
    ys = np.repeat(y, C, axis=0) if shared else y.reshape(-1, y.shape[-1])
    ref = np.stack([_ref_single(orc, "gtp_fourier", xs[i], ys[i], L1, L2, L3) for i in range(xs.shape[0])])
    assert _normwise(out.reshape(ref.shape), ref) <= TOL


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier"])
@pytest.mark.parametrize("L1,L2,L3", [(13, 5, 15), (4, 12, 16), (11, 11, 9)])
def test_gtp_separable_auto_unequal(tpo, orc, kind, L1, L2, L3):
    # the automatic path past L = 10 with unequal / truncated degrees: odd and even bands, the
    # Fourier torus of max(L1, L2) against the product band L1 + L2
    ctx = tpo.context()
    x, y = _inputs(9, L1, L2, 23 * L1 + L2 + L3)
    out = _gpu(tpo, kind, x, y, L1, L2, L3)
    assert ctx.last_grid_path == ("simt" if kind == "gtp_grid" else "separable")
    ref = np.stack([_ref_single(orc, kind, x[i], y[i], L1, L2, L3) for i in range(x.shape[0])])
    assert _normwise(out, ref) <= TOL


@pytest.mark.parametrize("L", [0, 1, 2, 3, 4, 6, 8])
def test_cgtp(tpo, orc, L):
    _check_batch(tpo, orc, "cgtp", L, 257, 300 + L)


@pytest.mark.parametrize("L,C,B", [(3, 128, 7), (3, 256, 3), (1, 128, 5)])
def test_cgtp_edge_tensor_cores(tpo, orc, L, C, B):
    # shared y, channels a multiple of 128: per-edge dense GEMM x . M_y on tcgen05
    x, y = _inputs(B, L, L, 340 + C + L, C=C, shared=True)
    x[0, 3] *= 1e-3  # rows of different magnitude (per-row power-of-two scaling)
    x[1, 5] *= 1e3
    out = _gpu(tpo, "cgtp", x, y, L, L, 0)
    ref = orc.batch_mimo("cgtp", L, x.astype(np.float64), y.astype(np.float64), channels=C, y_shared=True)
    assert _normwise(out, ref) <= TOL


@pytest.mark.parametrize("C", [32, 96])
def test_cgtp_edge_tiles(tpo, orc, C):
    # shared-y fast path (channels a multiple of the 32-row tile), ragged batch tail
    L, B = 3, 5
    x, y = _inputs(B, L, L, 330 + C, C=C, shared=True)
    out = _gpu(tpo, "cgtp", x, y, L, L, 0)
    ref = orc.batch_mimo("cgtp", L, x.astype(np.float64), y.astype(np.float64), channels=C, y_shared=True)
    assert _normwise(out, ref) <= TOL


@pytest.mark.parametrize("L,B", [(4, 5000), (5, 148 * 128 * 2 + 77), (6, 148 * 128 + 5), (7, 700), (8, 300), (10, 200),
                                 (11, 150), (12, 40), (13, 24), (14, 16)])
def test_cgtp_tensor_cores(tpo, orc, L, B):
    # per-(l1, l2) block GEMMs on tcgen05: several tiles per CTA, ragged tail, rows of
    # very different magnitude (per-row power-of-two scaling)
    x, y = _inputs(B, L, L, 360 + L)
    x[0] *= 1e-3
    y[1] *= 1e3
    out = _gpu(tpo, "cgtp", x, y, L, L, 0)
    ref = orc.batch_mimo("cgtp", L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
    assert _normwise(out, ref) <= TOL


def test_cgtp_tc_unequal_and_shared(tpo, orc):
    # block path with L1 != L2, and with y shared per edge at a channel count the
    # edge kernel does not take
    x, y = _inputs(90, 5, 3, 380)
    out = _gpu(tpo, "cgtp", x, y, 5, 3, 0)
    ref = np.stack([_ref_single(orc, "cgtp", x[b], y[b], 5, 3, 0) for b in range(90)])
    assert _normwise(out, ref) <= TOL
    x, y = _inputs(7, 5, 5, 381, C=24, shared=True)
    out = _gpu(tpo, "cgtp", x, y, 5, 5, 0)
    ref = orc.batch_mimo("cgtp", 5, x.astype(np.float64), y.astype(np.float64), channels=24, y_shared=True)
    assert _normwise(out, ref) <= TOL


def test_cgtp_simt_path():
    # SIMT kernel (the default below L = 5; forced here in a fresh process at larger L)
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import oracle, paper_2506_13523_b200 as tpo
worst = 0.0
for L, B in ((5, 200), (6, 100)):
    rng = np.random.default_rng(970 + L)
    d = (L + 1) ** 2
    x = rng.standard_normal((B, d)).astype(np.float32); y = rng.standard_normal((B, d)).astype(np.float32)
    out = tpo.run("cgtp", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), L, L, 0).cpu().numpy()
    ref = oracle.batch_mimo("cgtp", L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
    err = (np.abs(out - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)).max()
    worst = max(worst, float(err))
print(worst)
""" % (str(root), str(root / "oracle"))
    env = dict(os.environ, TPO_CGTP_TC="0")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL


@pytest.mark.parametrize("L", [12, 16])
def test_cgtp_large(tpo, orc, L):
    _check_batch(tpo, orc, "cgtp", L, 8, 310 + L)


@pytest.mark.parametrize("L", list(range(0, 13)))
def test_gtp_fourier_tcgen05(tpo, orc, L):
    # torus-grid dense operators (convolution theorem) on the fused tcgen05 kernel
    ctx = tpo.context()
    ctx.set_grid_path("tc")
    try:
        _check_batch(tpo, orc, "gtp_fourier", L, 1000 if L <= 8 else 300 if L <= 10 else 160, 400 + L)
        assert ctx.last_grid_path == "tcgen05"
    finally:
        ctx.set_grid_path("auto")


@pytest.mark.parametrize("L", [0, 1, 2, 4, 6, 11, 16])
def test_gtp_fourier_simt(tpo, orc, L):
    # direct spectral convolution on the Hermitian half plane (SIMT)
    ctx = tpo.context()
    ctx.set_grid_path("simt")
    try:
        _check_batch(tpo, orc, "gtp_fourier", L, 129 if L <= 8 else 16, 420 + L)
        assert ctx.last_grid_path == "simt"
    finally:
        ctx.set_grid_path("auto")


@pytest.mark.parametrize("L", [0, 1, 2, 3, 6, 10, 16])
def test_mtp(tpo, orc, L):
    _check_batch(tpo, orc, "mtp", L, 129 if L <= 8 else 16, 500 + L)


@pytest.mark.parametrize("L", [0, 1, 2, 3, 4, 5, 6])
def test_mtp_tensor_cores_many_tiles(tpo, orc, L):
    # tcgen05 path (carrier dt <= 13): several 128-row tiles per CTA, ragged tail
    B = 148 * 128 * 2 + 77 if L >= 5 else 5000
    x, y = _inputs(B, L, L, 560 + L)
    out = _gpu(tpo, "mtp", x, y, L, L, 2 * L)
    ref = orc.batch_mimo("mtp", L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
    assert _normwise(out, ref) <= TOL


def test_mtp_simt_path():
    # SIMT kernel (used past the tcgen05 carrier limit) forced in a fresh process
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import oracle, paper_2506_13523_b200 as tpo
worst = 0.0
for L, B in ((1, 300), (3, 300), (6, 300)):
    rng = np.random.default_rng(950 + L)
    d = (L + 1) ** 2
    x = rng.standard_normal((B, d)).astype(np.float32); y = rng.standard_normal((B, d)).astype(np.float32)
    out = tpo.run("mtp", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), L, L, 2 * L).cpu().numpy()
    ref = oracle.batch_mimo("mtp", L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
    err = (np.abs(out - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)).max()
    worst = max(worst, float(err))
print(worst)
""" % (str(root), str(root / "oracle"))
    env = dict(os.environ, TPO_MTP_TC="0")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL


# ---------------------------------------------------------------- shapes / edge cases
def test_ragged_batch_and_empty(tpo, orc):
    for kind in ("gtp_grid", "cgtp", "gtp_fourier", "mtp"):
        for B in (1, 127, 129):
            _check_batch(tpo, orc, kind, 2, B, 600 + B)
        import torch

        x = torch.empty((0, 9), device="cuda"); y = torch.empty((0, 9), device="cuda")
        assert tpo.run(kind, x, y, 2, 2, 4).shape[0] == 0


@pytest.mark.parametrize("kind", ["cgtp", "gtp_grid", "gtp_fourier", "mtp"])
def test_unequal_degrees(tpo, orc, kind):
    L1, L2, L3 = 3, 1, 3
    x, y = _inputs(40, L1, L2, 700)
    out = _gpu(tpo, kind, x, y, L1, L2, L3)
    ref = np.stack([_ref_single(orc, kind, x[b], y[b], L1, L2, L3) for b in range(40)])
    assert _normwise(out, ref) <= TOL


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier", "mtp"])
def test_output_band_past_product(tpo, orc, kind):
    # degrees past the product band are exactly zero (proj/src/gtp.cpp:237-258)
    x, y = _inputs(33, 1, 1, 710)
    out = _gpu(tpo, kind, x, y, 1, 1, 5)
    ref = np.stack([_ref_single(orc, kind, x[b], y[b], 1, 1, 5) for b in range(33)])
    assert _normwise(out, ref) <= TOL
    if kind != "mtp":
        assert np.all(out[:, 9:] == 0.0)


def test_channels_shared_y(tpo, orc):
    # channel-wise CGTP (config C4 shape, small batch): x [B][C][16], y [B][16]
    L, B, C = 3, 24, 128
    x, y = _inputs(B, L, L, 720, C=C, shared=True)
    for kind in ("cgtp", "gtp_grid", "mtp", "gtp_fourier"):
        out = _gpu(tpo, kind, x, y, L, L, 2 * L)
        ref = orc.batch_mimo(kind, L, x.astype(np.float64), y.astype(np.float64), channels=C, y_shared=True)
        assert _normwise(out, ref) <= TOL, kind


def test_channels_unshared(tpo, orc):
    L, B, C = 2, 10, 7
    x, y = _inputs(B, L, L, 730, C=C, shared=False)
    for kind in ("cgtp", "gtp_grid"):
        out = _gpu(tpo, kind, x, y, L, L, 2 * L)
        ref = orc.batch_mimo(kind, L, x.astype(np.float64), y.astype(np.float64), channels=C, y_shared=False)
        assert _normwise(out, ref) <= TOL


def test_mtp_carrier_override(tpo, orc):
    x, y = _inputs(50, 2, 2, 740)
    out = _gpu(tpo, "mtp", x, y, 2, 2, 4, lt=3)
    ref = np.stack([_ref_single(orc, "mtp", x[b], y[b], 2, 2, 4, lt=3) for b in range(50)])
    assert _normwise(out, ref) <= TOL
    with pytest.raises(ValueError):
        _gpu(tpo, "mtp", x, y, 2, 2, 4, lt=1)


# ---------------------------------------------------------------- known answers (reference tests)
def test_kats(tpo):
    import torch

    x = torch.tensor([[3.0]], device="cuda"); y = torch.tensor([[-2.0]], device="cuda")
    # proj/tests/test_gtp.cpp:36-43
    assert tpo.gtp_grid(x, y, 0, 0, 0).item() == pytest.approx(-6 / math.sqrt(4 * math.pi), rel=1e-6)
    assert tpo.gtp_fourier(x, y, 0, 0, 0).item() == pytest.approx(-6 / math.sqrt(4 * math.pi), rel=1e-6)
    # proj/tests/test_mtp.cpp:73-88
    assert tpo.mtp(x, y, 0, 0, 0).item() == pytest.approx(-6.0, rel=1e-6)
    assert tpo.mtp(x, y, 0, 0, 0, l_tilde=1).item() == pytest.approx(6 / math.sqrt(3), rel=1e-6)
    # proj/tests/test_cgtp.cpp:81-104: (0,0,0) path is the plain product
    assert tpo.cgtp(x, y, 0, 0).item() == pytest.approx(-6.0, rel=1e-6)


@pytest.mark.parametrize("L", [3, 6])
def test_equivariance(tpo, orc, L):
    # SO(3) equivariance of the GPU products (proj/src/verify.cpp:76-117 protocol); L = 6
    # exercises the CGTP block kernel, the dt = 13 MTP kernel and the folded Fourier torus
    rng = orc.Rng(20240901 + L)
    t = orc.tower(L)
    for kind in ("cgtp", "gtp_grid", "gtp_fourier", "mtp"):
        worst, scale = 0.0, 0.0
        for _ in range(5):
            x, y = rng.tower(L), rng.tower(L)
            R = rng.rotation()
            rx, ry = orc.rotate(t, x, R), orc.rotate(t, y, R)
            X = np.stack([x, rx]).astype(np.float32); Y = np.stack([y, ry]).astype(np.float32)
            out = _gpu(tpo, kind, X, Y, L, L, 2 * L)
            if kind == "cgtp":
                out_ls = [l3 for l1 in t for l2 in t for l3 in range(abs(l1 - l2), l1 + l2 + 1)]
            else:
                out_ls = orc.tower(2 * L)
            rhs = orc.rotate(out_ls, out[0], R)
            worst = max(worst, np.abs(out[1] - rhs).max())
            scale = max(scale, np.abs(out[0]).max())
        assert worst / scale < 1e-5, (kind, worst / scale)


def test_bad_arguments(tpo):
    import torch

    x = torch.zeros((4, 9), device="cuda"); y = torch.zeros((4, 9), device="cuda")
    with pytest.raises(ValueError):
        tpo.gtp_grid(x, y, 2, 2, -1)
    with pytest.raises(ValueError):
        tpo.gtp_grid(x, y, 1, 2, 2)  # x has 9 components, L1=1 means 4
    with pytest.raises(ValueError):
        tpo.cgtp(x.cpu(), y.cpu(), 2, 2)
    with pytest.raises(ValueError):
        tpo.weighted_gtp(x, y, np.ones(2), np.ones(3), np.ones(5), 2, 2, 4)


def test_weighted_gtp(tpo, orc):
    x, y = _inputs(20, 2, 2, 760)
    rng = np.random.default_rng(1)
    a, b, c = rng.standard_normal(3), rng.standard_normal(3), rng.standard_normal(5)
    import torch

    out = tpo.weighted_gtp(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), a, b, c, 2, 2, 4).cpu().numpy()
    ref = np.stack([orc.weighted_gtp(orc.tower(2), x[i].astype(np.float64), orc.tower(2),
                                     y[i].astype(np.float64), a, b, c, 4) for i in range(20)])
    assert _normwise(out, ref) <= TOL


def test_native_library_loaded(tpo, orc):
    ctx = tpo.context()
    before = ctx.launches
    _check_batch(tpo, orc, "gtp_grid", 1, 10, 1)
    assert ctx.launches > before
    with open("/proc/self/maps") as f:
        assert "libtpo_b200.so" in f.read()


def test_gtp_cta_pair_path():
    # opt-in tcgen05 cta_group::2 path (CTA pairs, M = 256): parity in a fresh
    # process because the mode is fixed when the device tables are built
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import oracle, paper_2506_13523_b200 as tpo
tpo.context(0).set_grid_path("tc")
worst = 0.0
for kind in ("gtp_grid", "gtp_fourier"):
    for L, B in ((1, 300), (4, 700), (7, 300), (10, 300)):
        rng = np.random.default_rng(900 + L)
        d = (L + 1) ** 2
        x = rng.standard_normal((B, d)).astype(np.float32); y = rng.standard_normal((B, d)).astype(np.float32)
        out = tpo.run(kind, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), L, L, 2 * L).cpu().numpy()
        ref = oracle.batch_mimo(kind, L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
        err = (np.abs(out - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)).max()
        worst = max(worst, float(err))
print(worst)
""" % (str(root), str(root / "oracle"))
    env = dict(os.environ, TPO_GRID_PAIR="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL


def test_cgtp_block_path_small_degrees():
    # the tcgen05 block kernel at L <= 4 (not the default there), fresh process
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import oracle, paper_2506_13523_b200 as tpo
worst = 0.0
for L, B in ((0, 50), (1, 300), (2, 129), (3, 5000), (4, 700)):
    rng = np.random.default_rng(990 + L)
    d = (L + 1) ** 2
    x = rng.standard_normal((B, d)).astype(np.float32); y = rng.standard_normal((B, d)).astype(np.float32)
    out = tpo.run("cgtp", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), L, L, 0).cpu().numpy()
    ref = oracle.batch_mimo("cgtp", L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
    err = (np.abs(out - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)).max()
    worst = max(worst, float(err))
print(worst)
""" % (str(root), str(root / "oracle"))
    env = dict(os.environ, TPO_CGTP_TC_MINL="0")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL


def test_host_batch_api(tpo, orc):
    # tpo_run_host_batch_f32: heterogeneous requests through one pipeline == one call each
    import torch

    reqs, singles = [], []
    for kind, L, B, C, shared in (("gtp_grid", 3, 3000, None, False), ("mtp", 2, 700, None, False),
                                  ("cgtp", 2, 40, 24, True), ("gtp_fourier", 1, 5000, None, False),
                                  ("cgtp", 6, 300, None, False)):
        x, y = _inputs(B, L, L, 990 + L, C=C, shared=shared)
        xt, yt = torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()
        L3 = 0 if kind == "cgtp" else 2 * L
        dout = tpo.out_dim(kind, L, L, L3)
        o = torch.empty(((B, dout) if C is None else (B, C, dout)), pin_memory=True)
        reqs.append((kind, xt, yt, o, L, L, L3))
        singles.append((kind, xt, yt, L, L3, C is not None and shared))
    outs = tpo.run_host_batch(reqs)
    for (kind, xt, yt, L, L3, ys), o in zip(singles, outs):
        ref = tpo.run(kind, xt.cuda(), yt.cuda(), L, L, L3).cpu()
        assert torch.equal(o, ref), kind
    # empty list and empty batch are fine
    tpo.run_host_batch([])


@pytest.mark.parametrize("L,B,C", [(3, 700, None), (7, 300, None), (10, 150, None), (4, 9, 24)])
def test_weighted_gtp_fused(tpo, orc, L, B, C):
    # per-degree weights fused into the tcgen05 kernel (input conversion + epilogue): one
    # launch, parity with the oracle and with the SIMT path (separate scaling passes)
    import torch

    x, y = _inputs(B, L, L, 770 + L, C=C, shared=C is not None)
    rng = np.random.default_rng(L)
    a, b, c = rng.standard_normal(L + 1), rng.standard_normal(L + 1), rng.standard_normal(2 * L + 1)
    ctx = tpo.context()
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    n0 = ctx.launches
    out = tpo.weighted_gtp(xt, yt, a, b, c, L, L, 2 * L).cpu().numpy()
    assert ctx.launches - n0 == 1 and ctx.last_grid_path == "tcgen05"
    xs = x.reshape(-1, x.shape[-1]).astype(np.float64)
    ys = (np.repeat(y, C, axis=0) if C is not None else y).reshape(-1, y.shape[-1]).astype(np.float64)
    ref = np.stack([orc.weighted_gtp(orc.tower(L), xs[i], orc.tower(L), ys[i], a, b, c, 2 * L)
                    for i in range(xs.shape[0])])
    assert _normwise(out.reshape(ref.shape), ref) <= TOL
    ctx.set_grid_path("simt")
    try:
        out_s = tpo.weighted_gtp(xt, yt, a, b, c, L, L, 2 * L).cpu().numpy()
    finally:
        ctx.set_grid_path("auto")
    assert _normwise(out_s.reshape(ref.shape), ref) <= TOL


@pytest.mark.parametrize("kind,L,B", [("gtp_grid", 13, 200), ("gtp_grid", 14, 60), ("gtp_fourier", 13, 40),
                                      ("gtp_fourier", 14, 16)])
def test_gtp_tcgen05_degree_groups(tpo, orc, kind, L, B):
    # inputs past the kernel's K limit (L = 13, 14): sum of launches over (x, y) degree groups
    ctx = tpo.context()
    ctx.set_grid_path("tc")
    try:
        _check_batch(tpo, orc, kind, L, B, 700 + L)
        assert ctx.last_grid_path == "tcgen05"
    finally:
        ctx.set_grid_path("auto")


def test_equivariance_report(tpo, orc):
    """SO(3) equivariance error, reported (north star): 20 Haar rotations per kind and L,
    max|T(Dx, Dy) - D T(x, y)| / max|T(x, y)| on the GPU outputs (fp32), written to
    gpurun_out/equivariance.json when run on a GPU box.  Also O(3) where the product has a
    definite parity: under inversion (x -> (-1)^l x) GTP outputs pick up (-1)^l3 and CGTP paths
    (-1)^(l1 + l2); the MTP mixes parities across paths (its Sum w * paths includes odd
    l1 + l2 + l3), so only its SO(3) error is reported."""
    import json
    from pathlib import Path

    rep = {}
    for L in (3, 6, 10):
        rng = orc.Rng(777 + L)
        t = orc.tower(L)
        par_in = np.concatenate([np.full(2 * l + 1, (-1.0) ** l) for l in t])
        for kind in ("cgtp", "gtp_grid", "gtp_fourier", "mtp"):
            if kind == "cgtp":
                out_ls = [l3 for l1 in t for l2 in t for l3 in range(abs(l1 - l2), l1 + l2 + 1)]
                par_out = np.concatenate([np.full(2 * l3 + 1, (-1.0) ** (l1 + l2)) for l1 in t for l2 in t
                                          for l3 in range(abs(l1 - l2), l1 + l2 + 1)])
            else:
                out_ls = orc.tower(2 * L)
                par_out = np.concatenate([np.full(2 * l + 1, (-1.0) ** l) for l in out_ls])
            xs, ys, rots = [], [], []
            for _ in range(20):
                x, y = rng.tower(L), rng.tower(L)
                R = rng.rotation()
                xs += [x, orc.rotate(t, x, R), par_in * x]
                ys += [y, orc.rotate(t, y, R), par_in * y]
                rots.append(R)
            out = _gpu(tpo, kind, np.stack(xs).astype(np.float32), np.stack(ys).astype(np.float32), L, L, 2 * L)
            so3, o3 = 0.0, 0.0
            for i, R in enumerate(rots):
                base, rot, inv = out[3 * i], out[3 * i + 1], out[3 * i + 2]
                scale = np.abs(base).max()
                so3 = max(so3, np.abs(rot - orc.rotate(out_ls, base, R)).max() / scale)
                o3 = max(o3, np.abs(inv - par_out * base).max() / scale)
            if kind == "mtp":
                o3 = None
            rep[f"{kind}_L{L}"] = {"so3_rel_err": so3, "inversion_rel_err": o3, "rotations": 20}
            assert so3 < 1e-5 and (o3 is None or o3 < 1e-5), (kind, L, so3, o3)
    out_dir = Path(__file__).resolve().parents[1] / "gpurun_out"
    if out_dir.exists():
        (out_dir / "equivariance.json").write_text(json.dumps(rep, indent=1))
    print(json.dumps(rep))
