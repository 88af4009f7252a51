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


def test_shim_tables_and_counts_cpu(orc):
    # host-side pieces of the module need no device: cg_table(gaunt=True), mtp_path_weights, count_ops
    from paper_2506_13523_b200 import so3tpo

    g = so3tpo.cg_table(2, 4, 2, gaunt=True)
    ref = orc.gaunt_real(2, 4, 2)
    assert [e[:3] for e in g] == [e[:3] for e in ref]
    assert max(abs(a[3] - b[3]) for a, b in zip(g, ref)) < 1e-13
    assert abs(so3tpo.mtp_path_weights(1, 1, 2, 1) - orc.mtp_path_weight(1, 1, 2, 1)) < 1e-12
    assert so3tpo.count_ops("cgtp", "sparse", "mimo", 2) == orc.count_ops("cgtp", "sparse", "mimo", 2) == 1560
    with pytest.raises(ValueError):
        so3tpo.count_ops("gtp", "naive", "mimo", 2)
    with pytest.raises(ValueError):
        so3tpo.count_ops("cgtp", "sparse", "bogus", 2)


@pytest.mark.gpu
def test_shim_wigner_rotate(orc):
    # py_core.cpp:118-133 signatures, on the GPU
    import numpy as np

    from paper_2506_13523_b200 import so3tpo

    D = so3tpo.wigner_d(3, [1.0, 2.0, -0.5], 0.7)
    R = so3tpo._axis_angle([1.0, 2.0, -0.5], 0.7)
    assert np.abs(D - orc.wigner_d(3, R)).max() < 1e-10
    x = np.random.default_rng(1).standard_normal(so3tpo.irreps_dim("2x1+1x3"))
    out = so3tpo.rotate("2x1+1x3", x, [0.0, 0.0, 1.0], 1.1)
    ref = orc.rotate([1, 1, 3], x, so3tpo._axis_angle([0.0, 0.0, 1.0], 1.1))
    assert np.abs(out - ref).max() < 1e-5 * np.abs(ref).max()
