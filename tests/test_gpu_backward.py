"""GPU parity of the backward pass (tpo_backward_f32).

The reference has no backward; the oracle here is the definition itself:
every product is bilinear, so the vector-Jacobian product for row b is
grad_x = J_x(y_b)^T g_b with J_x(y_b)[a] = T(e_a, y_b), evaluated by the fp64
oracle on basis vectors (no use of the Gaunt / embed identities the kernels
rely on).  Same normwise 1e-5 contract as the forward.  At full sizes the
check is size-independent: <g, T(dx, y)> = <grad_x, dx> (bilinearity).
"""
import numpy as np
import pytest

TOL = 1e-5

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tpo():
    import torch

    assert torch.cuda.is_available()
    import paper_2506_13523_b200 as m

    return m


def _dout(kind, L):
    return (L + 1) ** 4 if kind == "cgtp" else (2 * L + 1) ** 2


def _ref_vjp(orc, kind, L, x, y, g):
    """fp64 (grad_x, grad_y) per row from oracle Jacobians on basis vectors."""
    B, D = x.shape
    eye = np.eye(D)[:, None]
    gx = np.empty((B, D)); gy = np.empty((B, D))
    for b in range(B):
        Jx = orc.batch_mimo(kind, L, eye, np.repeat(y[b][None, None], D, 0))[:, 0]  # [D][Dout]
        Jy = orc.batch_mimo(kind, L, np.repeat(x[b][None, None], D, 0), eye)[:, 0]
        gx[b] = Jx @ g[b]
        gy[b] = Jy @ g[b]
    return gx, gy


def _normwise(out, ref):
    scale = np.maximum(np.abs(ref).max(axis=1), 1e-300)
    return float((np.abs(out - ref).max(axis=1) / scale).max())


def _run(tpo, kind, L, B, seed, L3=None, lt=-1):
    import torch

    L3 = 2 * L if L3 is None else L3
    rng = np.random.default_rng(seed)
    D = (L + 1) ** 2
    x = rng.standard_normal((B, D)).astype(np.float32)
    y = rng.standard_normal((B, D)).astype(np.float32)
    g = rng.standard_normal((B, _dout(kind, L))).astype(np.float32)
    gx, gy = tpo.backward(kind, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(),
                          torch.from_numpy(g).cuda(), L, L, L3, lt)
    torch.cuda.synchronize()
    return x, y, g, gx.cpu().numpy().astype(np.float64), gy.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("kind,L", [("cgtp", 1), ("cgtp", 2), ("cgtp", 3), ("cgtp", 5), ("cgtp", 6),
                                    ("gtp_grid", 1), ("gtp_grid", 3), ("gtp_grid", 5), ("gtp_grid", 6),
                                    ("gtp_grid", 7), ("gtp_grid", 9), ("gtp_grid", 10), ("gtp_grid", 12),
                                    ("gtp_fourier", 2), ("gtp_fourier", 6), ("gtp_fourier", 8),
                                    ("gtp_fourier", 11),
                                    ("mtp", 1), ("mtp", 3), ("mtp", 6), ("mtp", 8)])
def test_backward_vs_oracle(tpo, orc, kind, L):
    B = 6 if L >= 6 else 24
    x, y, g, gx, gy = _run(tpo, kind, L, B, 900 + L)
    rx, ry = _ref_vjp(orc, kind, L, x.astype(np.float64), y.astype(np.float64), g.astype(np.float64))
    ex, ey = _normwise(gx, rx), _normwise(gy, ry)
    assert ex <= TOL and ey <= TOL, (kind, L, ex, ey)


def test_backward_mtp_l_tilde_override(tpo, orc):
    """Larger carrier (l~ = 4 at L = 2): the VJP uses the forward's carrier."""
    L, lt = 2, 4
    x, y, g, gx, gy = _run(tpo, "mtp", L, 4, 77, lt=lt)
    t, t3 = orc.tower(L), orc.tower(2 * L)
    D = (L + 1) ** 2
    for b in range(4):
        Jx = np.stack([orc.mtp(t, np.eye(D)[a], t, y[b].astype(np.float64), 2 * L, lt_override=lt) for a in range(D)])
        Jy = np.stack([orc.mtp(t, x[b].astype(np.float64), t, np.eye(D)[a], 2 * L, lt_override=lt) for a in range(D)])
        assert _normwise(gx[b][None], (Jx @ g[b])[None]) <= TOL
        assert _normwise(gy[b][None], (Jy @ g[b])[None]) <= TOL
    del t3


@pytest.mark.parametrize("kind,L", [("cgtp", 3), ("cgtp", 5), ("gtp_grid", 4), ("mtp", 4)])
def test_backward_shared_y_channels(tpo, orc, kind, L):
    """Channel-wise form (x [B][C][D], y [B][D] shared): grad_x per (b, c)."""
    import torch

    B, C = 3, 64
    rng = np.random.default_rng(31 + L)
    D = (L + 1) ** 2
    x = rng.standard_normal((B, C, D)).astype(np.float32)
    y = rng.standard_normal((B, D)).astype(np.float32)
    g = rng.standard_normal((B, C, _dout(kind, L))).astype(np.float32)
    gx, gy = tpo.backward(kind, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(g).cuda(),
                          L, L, 2 * L, need_y=False)
    assert gy is None
    gx = gx.cpu().numpy().astype(np.float64)
    eye = np.eye(D)[:, None]
    for b in range(B):
        Jx = orc.batch_mimo(kind, L, eye, np.repeat(y[b].astype(np.float64)[None, None], D, 0))[:, 0]
        ref = g[b].astype(np.float64) @ Jx.T  # [C][D]
        assert _normwise(gx[b], ref) <= TOL, (kind, L, b)
    with pytest.raises(ValueError):
        tpo.backward(kind, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(g).cuda(),
                     L, L, 2 * L)


@pytest.mark.parametrize("kind,L", [("gtp_grid", 10), ("gtp_fourier", 6), ("mtp", 6), ("cgtp", 4),
                                    ("gtp_grid", 16), ("gtp_fourier", 16), ("mtp", 16), ("cgtp", 8)])
def test_backward_bilinearity_full_batch(tpo, kind, L):
    """Size-independent check at the BASELINE batch: <g, T(dx, y)> = <grad_x, dx>
    and <g, T(x, dy)> = <grad_y, dy> per row, through the autograd wrapper."""
    import torch

    B = 65536 if kind != "cgtp" and L <= 10 else 4096
    gen = torch.Generator(device="cuda").manual_seed(5)
    D = (L + 1) ** 2
    x = torch.randn(B, D, device="cuda", generator=gen, requires_grad=True)
    y = torch.randn(B, D, device="cuda", generator=gen, requires_grad=True)
    out = tpo.product(kind, x, y, L, L, 2 * L)
    g = torch.randn(out.shape, device="cuda", generator=gen)
    out.backward(g)
    dx = torch.randn(B, D, device="cuda", generator=gen)
    dy = torch.randn(B, D, device="cuda", generator=gen)
    with torch.no_grad():
        lhs_x = (g.double() * tpo.run(kind, dx, y.detach(), L, L, 2 * L).double()).sum(1)
        rhs_x = (x.grad.double() * dx.double()).sum(1)
        lhs_y = (g.double() * tpo.run(kind, x.detach(), dy, L, L, 2 * L).double()).sum(1)
        rhs_y = (y.grad.double() * dy.double()).sum(1)
    for lhs, rhs in ((lhs_x, rhs_x), (lhs_y, rhs_y)):
        scale = (g.double().abs().sum(1) * 1.0).clamp_min(1.0)
        err = ((lhs - rhs).abs() / scale).max().item()
        assert err < 1e-4, (kind, L, err)


@pytest.mark.parametrize("L", [2, 7])
def test_backward_gtp_simt_path(tpo, orc, L):
    """The SIMT fallback (grid_path 'simt': forward kernel with swapped operands)
    gives the same VJP as the tcgen05 degree-group path."""
    ctx = tpo.context()
    ctx.set_grid_path("simt")
    try:
        x, y, g, gx, gy = _run(tpo, "gtp_grid", L, 4, 600 + L)
    finally:
        ctx.set_grid_path("auto")
    rx, ry = _ref_vjp(orc, "gtp_grid", L, x.astype(np.float64), y.astype(np.float64), g.astype(np.float64))
    assert _normwise(gx, rx) <= TOL and _normwise(gy, ry) <= TOL


def _ref_vjp_general(orc, kind, L1, L2, L3, x, y, g):
    """(grad_x, grad_y) from oracle Jacobians for unequal degrees / truncated outputs."""
    d1, d2 = (L1 + 1) ** 2, (L2 + 1) ** 2
    t1, t2 = orc.tower(L1), orc.tower(L2)

    def T(a, b):
        if kind == "gtp_grid":
            return orc.gtp_grid(t1, a, t2, b, L3)
        if kind == "gtp_fourier":
            return orc.gtp_fourier(t1, a, t2, b, L3)
        return orc.mtp(t1, a, t2, b, L3)

    gx = np.empty((x.shape[0], d1)); gy = np.empty((x.shape[0], d2))
    for r in range(x.shape[0]):
        Jx = np.stack([T(e, y[r]) for e in np.eye(d1)])
        Jy = np.stack([T(x[r], e) for e in np.eye(d2)])
        gx[r] = Jx @ g[r]
        gy[r] = Jy @ g[r]
    return gx, gy


@pytest.mark.parametrize("kind", ["gtp_grid", "gtp_fourier", "mtp"])
@pytest.mark.parametrize("L1,L2,L3", [(3, 1, 3), (5, 2, 4), (2, 2, 6), (1, 3, 2)])
def test_backward_unequal_degrees(tpo, orc, kind, L1, L2, L3):
    # the gather-window paths of the VJPs: truncated outputs (L3 < L1 + L2), asymmetric operator
    # degrees, grad_out degrees above what can reach a gradient (VERDICT r1 advisor item)
    import torch

    rng = np.random.default_rng(31 * L1 + 7 * L2 + L3)
    B = 9
    x = rng.standard_normal((B, (L1 + 1) ** 2)).astype(np.float32)
    y = rng.standard_normal((B, (L2 + 1) ** 2)).astype(np.float32)
    g = rng.standard_normal((B, (L3 + 1) ** 2)).astype(np.float32)
    gx, gy = tpo.backward(kind, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(g).cuda(),
                          L1, L2, L3)
    rx, ry = _ref_vjp_general(orc, kind, L1, L2, L3, x.astype(np.float64), y.astype(np.float64), g.astype(np.float64))
    assert _normwise(gx.cpu().numpy().astype(np.float64), rx) <= TOL
    assert _normwise(gy.cpu().numpy().astype(np.float64), ry) <= TOL


def test_backward_unequal_degrees_simt_path(tpo, orc):
    # the same on the SIMT grid path (forced), which the backward falls back to for shapes the
    # tcgen05 kernel does not take
    import torch

    ctx = tpo.context()
    ctx.set_grid_path("simt")
    try:
        for (L1, L2, L3) in ((3, 1, 3), (2, 4, 5)):
            rng = np.random.default_rng(L1 + L2 + L3)
            x = rng.standard_normal((5, (L1 + 1) ** 2)).astype(np.float32)
            y = rng.standard_normal((5, (L2 + 1) ** 2)).astype(np.float32)
            g = rng.standard_normal((5, (L3 + 1) ** 2)).astype(np.float32)
            gx, gy = tpo.backward("gtp_grid", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(),
                                  torch.from_numpy(g).cuda(), L1, L2, L3)
            rx, ry = _ref_vjp_general(orc, "gtp_grid", L1, L2, L3, x.astype(np.float64), y.astype(np.float64),
                                      g.astype(np.float64))
            assert _normwise(gx.cpu().numpy().astype(np.float64), rx) <= TOL
            assert _normwise(gy.cpu().numpy().astype(np.float64), ry) <= TOL
    finally:
        ctx.set_grid_path("auto")


def _cgtp_ref_vjp(orc, L1, L2, x, y, g):
    """CGTP (grad_x, grad_y) for unequal degrees from oracle Jacobians on basis vectors."""
    t1, t2 = orc.tower(L1), orc.tower(L2)
    d1, d2 = (L1 + 1) ** 2, (L2 + 1) ** 2
    gx = np.empty((x.shape[0], d1)); gy = np.empty((x.shape[0], d2))
    for r in range(x.shape[0]):
        Jx = np.stack([orc.cgtp_mimo(t1, e, t2, y[r]) for e in np.eye(d1)])
        Jy = np.stack([orc.cgtp_mimo(t1, x[r], t2, e) for e in np.eye(d2)])
        gx[r] = Jx @ g[r]
        gy[r] = Jy @ g[r]
    return gx, gy


@pytest.mark.parametrize("L1,L2", [(6, 3), (3, 5), (4, 4), (2, 6), (6, 6), (5, 1), (7, 7), (7, 4), (3, 7), (8, 8),
                                   (8, 5), (4, 8)])
def test_backward_cgtp_unequal_degrees(tpo, orc, L1, L2):
    # the tcgen05 block backward (cgtp_bwd_tc.cu) takes L1, L2 <= 8 (blocks wider than 192 columns
    # in row-aligned N parts from 7, one launch per gradient at 8); (5, 1) and small shapes stay on
    # the SIMT term-list kernel
    import torch

    rng = np.random.default_rng(17 * L1 + L2)
    B = 5
    x = rng.standard_normal((B, (L1 + 1) ** 2)).astype(np.float32)
    y = rng.standard_normal((B, (L2 + 1) ** 2)).astype(np.float32)
    g = rng.standard_normal((B, (L1 + 1) ** 2 * (L2 + 1) ** 2)).astype(np.float32)
    gx, gy = tpo.backward("cgtp", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(g).cuda(),
                          L1, L2)
    rx, ry = _cgtp_ref_vjp(orc, L1, L2, x.astype(np.float64), y.astype(np.float64), g.astype(np.float64))
    assert _normwise(gx.cpu().numpy().astype(np.float64), rx) <= TOL
    assert _normwise(gy.cpu().numpy().astype(np.float64), ry) <= TOL


@pytest.mark.parametrize("L", [3, 4, 5, 6, 7, 8])
def test_backward_cgtp_tc_matches_simt(tpo, monkeypatch, L):
    """Ragged batch (1,000 rows: a partial last tile) with per-row scales over 1e-20 .. 1e20 and
    one-sided requests: the tcgen05 backward against the SIMT term-list kernel (fp32 sums, itself
    oracle-checked above), normwise 1e-5 per row."""
    import torch

    B, D = 1000, (L + 1) ** 2
    gen = torch.Generator(device="cuda").manual_seed(40 + L)
    sc = 10.0 ** torch.linspace(-20, 20, B, device="cuda")[torch.randperm(B, device="cuda", generator=gen)]
    x = torch.randn(B, D, device="cuda", generator=gen) * sc[:, None]
    y = torch.randn(B, D, device="cuda", generator=gen) * sc.flip(0)[:, None]
    g = torch.randn(B, D * D, device="cuda", generator=gen) * (sc ** 0.5)[:, None]
    gx, gy = tpo.backward("cgtp", x, y, g, L, L)
    gx1, _ = tpo.backward("cgtp", x, y, g, L, L, need_y=False)
    _, gy1 = tpo.backward("cgtp", x, y, g, L, L, need_x=False)
    monkeypatch.setenv("TPO_CGTP_BWD_TC", "0")
    rx, ry = tpo.backward("cgtp", x, y, g, L, L)
    torch.cuda.synchronize()
    for out, ref in ((gx, rx), (gy, ry), (gx1, rx), (gy1, ry)):
        a, b = out.double().cpu().numpy(), ref.double().cpu().numpy()
        assert np.isfinite(a).all()
        assert _normwise(a, b) <= TOL, (L, _normwise(a, b))
