"""Reference Python-module surface (proj/tests/python/test_smoke.py restated)
through the shim paper_2506_13523_b200.so3tpo.  CPU parts run everywhere;
product calls need the GPU."""
import math

import numpy as np
import pytest


@pytest.fixture(scope="module")
def so3():
    from paper_2506_13523_b200 import so3tpo

    return so3tpo


def test_irreps_helpers(so3):
    # proj/tests/python/test_smoke.py:15-20
    assert so3.irreps_dim("2x1+1x0") == 7
    assert so3.single_copies(2) == "1x0+1x1+1x2"
    assert so3.irreps_dim(so3.single_copies(4)) == 25
    with pytest.raises(ValueError):
        so3.irreps_dim("not-irreps")


def test_cg_table_cross_product(so3):
    # proj/tests/python/test_smoke.py:23-35
    rows = so3.cg_table(1, 1, 1)
    assert len(rows) == 6
    for m1, m2, m3, value in rows:
        assert abs(abs(value) - 1 / math.sqrt(2)) < 1e-14
        assert (m1, m2, m3).count(0) == 1
    assert so3.cg_table(1, 1, 3) == []


@pytest.mark.gpu
def test_cgtp_shapes_and_mismatch(so3):
    rng = np.random.default_rng(1)
    irreps = so3.single_copies(1)
    out_irreps, out = so3.cgtp(irreps, rng.standard_normal(4), irreps, rng.standard_normal(4))
    assert so3.irreps_dim(out_irreps) == out.shape[0] == 16
    with pytest.raises(ValueError):
        so3.cgtp(irreps, np.zeros(3), irreps, np.zeros(4))


@pytest.mark.gpu
def test_products_are_equivariant(so3, orc):
    # proj/tests/python/test_smoke.py:45-64 with the fp32 device tolerance
    rng = np.random.default_rng(2)
    L = 2
    irreps = so3.single_copies(L)
    x, y = rng.standard_normal((L + 1) ** 2), rng.standard_normal((L + 1) ** 2)
    axis, angle = np.array([0.3, -1.0, 0.7]), 1.1
    n = axis / np.linalg.norm(axis)
    K = np.array([[0, -n[2], n[1]], [n[2], 0, -n[0]], [-n[1], n[0], 0]])
    R = np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * K @ K
    t = orc.tower(L)
    rx, ry = orc.rotate(t, x, R), orc.rotate(t, y, R)
    for apply_tp in (
        lambda a, b: so3.cgtp(irreps, a, irreps, b),
        lambda a, b: so3.gtp(irreps, a, irreps, b, 2 * L),
        lambda a, b: so3.gtp(irreps, a, irreps, b, 2 * L, impl="fourier"),
        lambda a, b: so3.mtp(irreps, a, irreps, b, 2 * L),
    ):
        out_irreps, lhs = apply_tp(rx, ry)
        _, out = apply_tp(x, y)
        ls = [int(e.split("x")[1]) for e in out_irreps.split("+")]
        rhs = orc.rotate(ls, out, R)
        assert np.abs(lhs - rhs).max() <= 1e-5 * np.abs(out).max()


@pytest.mark.gpu
def test_gtp_impls_agree_and_scalars(so3):
    rng = np.random.default_rng(3)
    irreps = so3.single_copies(3)
    x, y = rng.standard_normal(16), rng.standard_normal(16)
    _, grid = so3.gtp(irreps, x, irreps, y, 6, impl="grid")
    _, fourier = so3.gtp(irreps, x, irreps, y, 6, impl="fourier")
    assert np.abs(grid - fourier).max() <= 1e-5 * np.abs(grid).max()
    _, z = so3.mtp("1x0", np.array([3.0]), "1x0", np.array([-2.0]), 0)
    assert z[0] == pytest.approx(-6.0, rel=1e-6)
