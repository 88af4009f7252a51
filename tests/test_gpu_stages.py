"""GPU parity of the stage entry points (tpo_to_sphere_f32, tpo_from_sphere_f32, tpo_pointwise_mul_f32,
tpo_mtp_embed/matmul/extract_f32, tpo_apply_linear_f32, tpo_wigner_d_f64, tpo_rotate_f32) against the
fp64 oracle's restatement of the same reference functions (proj/src/sphere.cpp:105-195,
proj/src/mtp.cpp:20-133, proj/src/irreps.cpp:95-129, proj/src/wigner.cpp:288-325), plus the
reference's own stage compositions: to_sphere -> pointwise_mul -> from_sphere == gtp_grid
(proj/src/gtp.cpp:228-260) and embed -> matmul -> extract == mtp (proj/src/mtp.cpp:99-117), the
round trip from_sphere(to_sphere(x)) == x (proj/src/verify.cpp:256-309), and a large-batch
equivariance report with the rotations computed on the GPU."""
import json
from pathlib import Path

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


def _rel(out, ref):
    out = np.asarray(out, np.float64).reshape(-1, np.asarray(out).shape[-1])
    ref = np.asarray(ref, np.float64).reshape(out.shape)
    return float((np.abs(out - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)).max())


def _x(B, L, seed):
    return np.random.default_rng(seed).standard_normal((B, (L + 1) ** 2)).astype(np.float32)


@pytest.mark.parametrize("L,grid_L", [(0, 0), (1, 2), (3, 3), (4, 8), (10, 20), (16, 32)])
def test_to_sphere(tpo, orc, L, grid_L):
    import torch

    x = _x(37, L, 10 + L)
    F = tpo.to_sphere(torch.from_numpy(x).cuda(), L, grid_L).cpu().numpy()
    ref = np.stack([orc.to_sphere(orc.tower(L), r.astype(np.float64), grid_L) for r in x])
    assert _rel(F.reshape(37, -1), ref.reshape(37, -1)) <= TOL


@pytest.mark.parametrize("grid_L,degrees", [(2, [0, 1, 2]), (6, [3, 0, 5]), (20, list(range(21))), (12, [12])])
def test_from_sphere(tpo, orc, grid_L, degrees):
    import torch

    rng = np.random.default_rng(grid_L)
    F = rng.standard_normal((21, grid_L + 1, 2 * grid_L + 1)).astype(np.float32)
    out = tpo.from_sphere(torch.from_numpy(F).cuda(), grid_L, degrees).cpu().numpy()
    ref = np.stack([orc.from_sphere(f.astype(np.float64), grid_L, degrees) for f in F])
    assert _rel(out, ref) <= TOL


def test_sphere_errors(tpo):
    import torch

    x = torch.zeros((2, 16), device="cuda")
    with pytest.raises(ValueError):  # grid band below the input degree (proj/src/sphere.cpp:106-110)
        tpo.to_sphere(x, 3, 2)
    F = torch.zeros((2, 3, 5), device="cuda")
    with pytest.raises(ValueError):  # requested degree above the grid (proj/src/sphere.cpp:160-162)
        tpo.from_sphere(F, 2, [3])


@pytest.mark.parametrize("L", [1, 4, 8])
def test_round_trip_and_grid_pipeline(tpo, orc, L):
    # from_sphere(to_sphere(x)) == x on make_grid(L) (proj/src/verify.cpp:256-309), and the staged
    # grid GTP equals the fused kernel and the oracle (proj/src/gtp.cpp:228-260)
    import torch

    x = torch.from_numpy(_x(64, L, 50 + L)).cuda()
    y = torch.from_numpy(_x(64, L, 60 + L)).cuda()
    back = tpo.from_sphere(tpo.to_sphere(x, L, L), L, list(range(L + 1)))
    assert _rel(back.cpu().numpy(), x.cpu().numpy()) <= TOL
    band = 2 * L
    F = tpo.pointwise_mul(tpo.to_sphere(x, L, band), tpo.to_sphere(y, L, band))
    staged = tpo.from_sphere(F, band, list(range(2 * L + 1))).cpu().numpy()
    fused = tpo.gtp_grid(x, y, L, L, 2 * L).cpu().numpy()
    ref = orc.batch_mimo("gtp_grid", L, x.cpu().numpy().astype(np.float64)[:, None],
                         y.cpu().numpy().astype(np.float64)[:, None])[:, 0]
    assert _rel(staged, ref) <= TOL
    assert _rel(fused, ref) <= TOL


@pytest.mark.parametrize("L,lt", [(0, 0), (2, 1), (3, 2), (6, 6), (10, 10), (4, 7)])
def test_mtp_stages(tpo, orc, L, lt):
    import torch

    x = _x(29, L, 70 + L)
    y = _x(29, L, 80 + L)
    X = tpo.mtp_embed(torch.from_numpy(x).cuda(), L, lt)
    Y = tpo.mtp_embed(torch.from_numpy(y).cuda(), L, lt)
    refX = np.stack([orc.mtp_embed(orc.tower(L), r.astype(np.float64), lt) for r in x])
    assert _rel(X.cpu().numpy().reshape(29, -1), refX.reshape(29, -1)) <= TOL
    Z = tpo.mtp_matmul(X, Y)
    refZ = np.stack([orc.mtp_matmul(a, b) for a, b in zip(X.cpu().numpy().astype(np.float64),
                                                         Y.cpu().numpy().astype(np.float64))])
    assert _rel(Z.cpu().numpy().reshape(29, -1), refZ.reshape(29, -1)) <= TOL
    L3 = min(2 * L, 2 * lt)
    out = tpo.mtp_extract(Z, lt, list(range(L3 + 1))).cpu().numpy()
    refo = np.stack([orc.mtp_extract(z.astype(np.float64), L3, lt) for z in Z.cpu().numpy()])
    assert _rel(out, refo) <= TOL
    # the staged product equals mtp(x, y, L3) with this carrier (proj/src/mtp.cpp:99-117)
    full = np.stack([orc.mtp(orc.tower(L), a.astype(np.float64), orc.tower(L), b.astype(np.float64), L3,
                             lt_override=lt) for a, b in zip(x, y)])
    assert _rel(out, full) <= TOL
    # a permuted degree selection is the same blocks in the requested order; degrees past 2 lt are zero
    sel = [L3, 0, 2 * lt + 1] if L3 > 0 else [0, 2 * lt + 1]
    o2 = tpo.mtp_extract(Z, lt, sel).cpu().numpy()
    if L3 > 0:
        assert np.array_equal(o2[:, : 2 * L3 + 1], out[:, L3 * L3:])
    assert np.all(o2[:, -(2 * (2 * lt + 1) + 1):] == 0.0)


def test_mtp_stage_errors(tpo):
    import torch

    with pytest.raises(ValueError):  # carrier too small (proj/src/mtp.cpp:50-51)
        tpo.mtp_embed(torch.zeros((1, 16), device="cuda"), 3, 1)


def test_apply_linear(tpo):
    # Schur-consistent linear layer (proj/src/irreps.cpp:95-129) vs a numpy restatement
    import torch

    ins = [(2, 0), (1, 1), (3, 2)]
    outs = [(1, 0), (2, 2), (2, 1), (1, 3)]
    conns = tpo.linear_connections(ins, outs)
    rng = np.random.default_rng(3)
    w = rng.standard_normal(len(conns))
    din = sum(m * (2 * l + 1) for m, l in ins)
    x = rng.standard_normal((50, din)).astype(np.float32)
    out = tpo.apply_linear(torch.from_numpy(x).cuda(), ins, outs, w).cpu().numpy()

    def offs(irr):
        o, r = 0, {}
        for e, (m, l) in enumerate(irr):
            for c in range(m):
                r[(e, c)] = o
                o += 2 * l + 1
        return r, o

    io, _ = offs(ins)
    oo, dout = offs(outs)
    ref = np.zeros((50, dout))
    for wi, (ei, ci, eo, co) in zip(w, conns):
        d = 2 * ins[ei][1] + 1
        ref[:, oo[(eo, co)]:oo[(eo, co)] + d] += wi * x[:, io[(ei, ci)]:io[(ei, ci)] + d].astype(np.float64)
    assert _rel(out, ref) <= TOL
    with pytest.raises(ValueError):  # wrong weight count (proj/src/irreps.cpp:106-110)
        tpo.apply_linear(torch.from_numpy(x).cuda(), ins, outs, w[:-1])


@pytest.mark.parametrize("L", [0, 1, 2, 5, 12, 32])
def test_wigner_d(tpo, orc, L):
    import torch

    rng = orc.Rng(40 + L)
    Rs = np.stack([rng.rotation() for _ in range(9)])
    blocks = tpo.wigner_d(torch.from_numpy(Rs).cuda(), L)
    for l, Dl in enumerate(blocks):
        Dl = Dl.cpu().numpy()
        for i in range(len(Rs)):
            ref = orc.wigner_d(l, Rs[i])
            assert np.abs(Dl[i] - ref).max() < 1e-10, (l, i)


@pytest.mark.parametrize("L,C", [(3, None), (6, 5), (20, None)])
def test_rotate(tpo, orc, L, C):
    import torch

    rng = orc.Rng(90 + L)
    B = 24
    Rs = np.stack([rng.rotation() for _ in range(6)])  # sample b uses R[b * 6 // B]
    x = np.random.default_rng(L).standard_normal((B, C, (L + 1) ** 2) if C else (B, (L + 1) ** 2)).astype(np.float32)
    out = tpo.rotate(torch.from_numpy(x).cuda(), torch.from_numpy(Rs).cuda(), L).cpu().numpy()
    xs = x.reshape(B, -1, (L + 1) ** 2)
    ref = np.stack([[orc.rotate(orc.tower(L), xs[b, c].astype(np.float64), Rs[b * 6 // B]) for c in range(xs.shape[1])]
                    for b in range(B)]).reshape(out.shape)
    assert _rel(out, ref) <= TOL


def test_equivariance_large_batch(tpo):
    """SO(3) equivariance of all four products on 65,536 products per (kind, L), each sample with its
    own Haar rotation, rotations applied on the GPU (tpo_rotate_f32):
    max over rows of |T(Dx, Dy) - D T(x, y)| / max|T(x, y)|.  Written to
    gpurun_out/equivariance_large.json on a GPU box."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(123)
    rep = {}
    B = 65536
    for L in (3, 6, 10):
        q = torch.randn((B, 4), generator=g, device="cuda", dtype=torch.float64)
        q = q / q.norm(dim=1, keepdim=True)
        w_, x_, y_, z_ = q.unbind(1)  # unit quaternion -> rotation matrix
        R = torch.stack([1 - 2 * (y_ * y_ + z_ * z_), 2 * (x_ * y_ - z_ * w_), 2 * (x_ * z_ + y_ * w_),
                         2 * (x_ * y_ + z_ * w_), 1 - 2 * (x_ * x_ + z_ * z_), 2 * (y_ * z_ - x_ * w_),
                         2 * (x_ * z_ - y_ * w_), 2 * (y_ * z_ + x_ * w_), 1 - 2 * (x_ * x_ + y_ * y_)], 1)
        R = R.reshape(B, 3, 3).contiguous()
        x = torch.randn((B, (L + 1) ** 2), generator=g, device="cuda")
        y = torch.randn((B, (L + 1) ** 2), generator=g, device="cuda")
        rx, ry = tpo.rotate(x, R, L), tpo.rotate(y, R, L)
        for kind in ("gtp_grid", "gtp_fourier", "mtp", "cgtp"):
            if kind == "cgtp" and L > 6:
                continue
            base = tpo.run(kind, x, y, L, L, 0 if kind == "cgtp" else 2 * L)
            rot = tpo.run(kind, rx, ry, L, L, 0 if kind == "cgtp" else 2 * L)
            if kind == "cgtp":  # outputs are (l1, l2, l3) path blocks: rotate all blocks of one l3 at once
                rb = torch.empty_like(base)
                offs, o = {}, 0
                for l1 in range(L + 1):
                    for l2 in range(L + 1):
                        for l3 in range(abs(l1 - l2), l1 + l2 + 1):
                            offs.setdefault(l3, []).append(o)
                            o += 2 * l3 + 1
                for l3, os_ in offs.items():
                    blk = torch.zeros((B, len(os_), (l3 + 1) ** 2), device="cuda")
                    for i, o in enumerate(os_):
                        blk[:, i, l3 * l3:] = base[:, o:o + 2 * l3 + 1]
                    r = tpo.rotate(blk, R, l3)
                    for i, o in enumerate(os_):
                        rb[:, o:o + 2 * l3 + 1] = r[:, i, l3 * l3:]
            else:
                rb = tpo.rotate(base, R, 2 * L)
            err = ((rot - rb).abs().amax(dim=1) / base.abs().amax(dim=1).clamp_min(1e-30)).max().item()
            rep[f"{kind}_L{L}"] = {"so3_rel_err": err, "products": B, "rotations": B}
            assert err < 1e-5, (kind, L, err)
    out_dir = Path(__file__).resolve().parents[1] / "gpurun_out"
    if out_dir.exists():
        (out_dir / "equivariance_large.json").write_text(json.dumps(rep, indent=1))


@pytest.mark.parametrize("L,C,shared,per_edge", [(3, 128, True, True), (3, 128, True, False), (2, 24, True, True),
                                                 (5, None, False, True), (2, 7, False, False)])
def test_cgtp_per_path_weights(tpo, orc, L, C, shared, per_edge):
    # f2: path p of edge b scaled by w[b, p]; reference = oracle CGTP with each path block scaled
    import torch

    rng = np.random.default_rng(L + (C or 0))
    B = 9
    d = (L + 1) ** 2
    x = rng.standard_normal((B, C, d) if C else (B, d)).astype(np.float32)
    y = rng.standard_normal((B, d) if (shared or not C) else (B, C, d)).astype(np.float32)
    npth = tpo.cgtp_num_paths(L, L)
    w = rng.standard_normal((B, npth) if per_edge else (npth,)).astype(np.float32)
    out = tpo.cgtp_weighted(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(w).cuda(), L, L)
    out = out.cpu().numpy().reshape(B, C or 1, -1)
    ref = orc.batch_mimo("cgtp", L, x.astype(np.float64).reshape(B, C or 1, d),
                         y.astype(np.float64) if shared else y.astype(np.float64).reshape(B, C or 1, d),
                         channels=C or 1, y_shared=bool(shared and C))
    pcol = np.concatenate([np.full(2 * l3 + 1, p) for p, (l1, l2, l3) in enumerate(
        [(a, b, c) for a in range(L + 1) for b in range(L + 1) for c in range(abs(a - b), a + b + 1)])])
    wb = (w[:, None, pcol] if per_edge else w[None, None, pcol]).astype(np.float64)
    assert _rel(out, ref * wb) <= TOL


@pytest.mark.parametrize("L", [3, 6])
def test_linear_gtp_fused_equals_composition(tpo, L):
    # f1: LinearLayer (towers) -> grid GTP -> LinearLayer, fused into one launch, against the three
    # separate GPU stages (apply_linear, run, apply_linear)
    import torch

    rng = np.random.default_rng(300 + L)
    B = 777
    x = torch.from_numpy(rng.standard_normal((B, (L + 1) ** 2)).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.standard_normal((B, (L + 1) ** 2)).astype(np.float32)).cuda()
    tower_in = [(1, l) for l in range(L + 1)]
    tower_out = [(1, l) for l in range(2 * L + 1)]
    wx, wy, wo = rng.standard_normal(L + 1), rng.standard_normal(L + 1), rng.standard_normal(2 * L + 1)
    ctx = tpo.context()
    n0 = ctx.launches
    fused = tpo.linear_gtp(x, y, L, L, 2 * L, wx, wy, wo)
    assert ctx.launches - n0 == 1
    ref = tpo.apply_linear(tpo.run("gtp_grid", tpo.apply_linear(x, tower_in, tower_in, wx),
                                   tpo.apply_linear(y, tower_in, tower_in, wy), L, L, 2 * L),
                           tower_out, tower_out, wo)
    a, b = fused.double().cpu().numpy(), ref.double().cpu().numpy()
    err = (np.abs(a - b).max(axis=1) / np.maximum(np.abs(b).max(axis=1), 1e-300)).max()
    assert err <= 2e-5, err
    with pytest.raises(ValueError):
        tpo.linear_gtp(x, y, L, L, 2 * L, wx[:-1], wy, wo)
