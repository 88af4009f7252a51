"""Pins the fp64 CPU oracle (oracle/) to the reference's own known-answer
tests and identities, and to independent oracles (sympy, scipy).

Each test cites the reference test it restates (paths under
/root/reference/proj).  These run on CPU (no GPU marker).
"""
import math

import numpy as np
import pytest

SEED = 20240901  # proj/include/tpo/bench.hpp:53


# ------------------------------------------------------------------ RNG / layout
def test_first_random_draw(orc):
    # proj/README.md:108 -- first N(0,1) draw of mt19937_64(20240901)
    assert orc.Rng(SEED).irrep(1)[0] == -1.5095082358763112


def test_rotation_random_is_proper(orc):
    rng = orc.Rng(3)
    for _ in range(5):
        R = rng.rotation()
        assert np.abs(R.T @ R - np.eye(3)).max() < 1e-14
        assert abs(np.linalg.det(R) - 1) < 1e-14


# ------------------------------------------------------------------ tables
def test_racah_vs_sympy(orc):
    # proj/tests/test_wigner.cpp:22-37 (exact-rational Racah oracle to 1e-14, l<=6)
    from sympy.physics.quantum.cg import CG
    from sympy import S

    worst = 0.0
    for l1 in range(0, 4):
        for l2 in range(0, 4):
            for l3 in range(abs(l1 - l2), l1 + l2 + 1):
                for m1 in range(-l1, l1 + 1):
                    for m2 in range(-l2, l2 + 1):
                        m3 = m1 + m2
                        if abs(m3) > l3:
                            continue
                        want = float(CG(S(l1), S(m1), S(l2), S(m2), S(l3), S(m3)).doit())
                        worst = max(worst, abs(orc.cg_coefficient(l1, m1, l2, m2, l3, m3) - want))
    assert worst < 1e-14


def test_real_basis_change_unitary(orc):
    # proj/tests/test_wigner.cpp:59-67
    for l in range(7):
        U = orc.real_basis_change(l)
        assert np.abs(U @ U.conj().T - np.eye(2 * l + 1)).max() < 1e-14


def test_cg_real_111_cross_product_values(orc):
    # proj/tests/test_wigner.cpp:69-80 and proj/README.md:99-103
    t = orc.cg_real(1, 1, 1)
    assert len(t) == 6
    s = 1 / math.sqrt(2)
    for m1, m2, m3, v in t:
        assert abs(abs(v) - s) < 1e-15
        if (m1, m2) == (0, 1):
            assert m3 == -1 and v == pytest.approx(-s, rel=1e-14)
    # CLI row order: "-1,0,1,-0.70710678118654746" then "-1,1,0,0.70710678118654746"
    assert t[0] == (-1, 0, 1, pytest.approx(-0.70710678118654746, abs=1e-16))
    assert t[1] == (-1, 1, 0, pytest.approx(0.70710678118654746, abs=1e-16))
    assert orc.cg_real(1, 1, 3) == []


def test_cg_real_orthonormal(orc):
    # proj/tests/test_wigner.cpp:82-97
    for l1 in range(4):
        for l2 in range(4):
            for l3 in range(abs(l1 - l2), l1 + l2 + 1):
                d3 = 2 * l3 + 1
                gram = np.zeros((d3, d3))
                t = orc.cg_real(l1, l2, l3)
                for a in t:
                    for b in t:
                        if a[0] == b[0] and a[1] == b[1]:
                            gram[a[2] + l3, b[2] + l3] += a[3] * b[3]
                assert np.abs(gram - np.eye(d3)).max() < 1e-13


def test_gaunt_kats_and_sympy(orc):
    # proj/tests/test_wigner.cpp:99-107 plus independent sympy real_gaunt
    from sympy.physics.wigner import real_gaunt

    t = orc.gaunt_real(0, 0, 0)
    assert len(t) == 1 and t[0][3] == pytest.approx(1 / math.sqrt(4 * math.pi), rel=1e-15)
    assert orc.gaunt_real(1, 1, 1) == []
    assert orc.gaunt_real(1, 2, 0) == []
    assert orc.gaunt_real(2, 4, 2) != []
    worst = 0.0
    for (l1, l2, l3) in [(1, 1, 2), (2, 2, 2), (1, 2, 3), (2, 3, 3), (3, 3, 4)]:
        tab = {(a, b, c): v for a, b, c, v in orc.gaunt_real(l1, l2, l3)}
        for m1 in range(-l1, l1 + 1):
            for m2 in range(-l2, l2 + 1):
                for m3 in range(-l3, l3 + 1):
                    want = float(real_gaunt(l1, l2, l3, m1, m2, m3))
                    worst = max(worst, abs(tab.get((m1, m2, m3), 0.0) - want))
    assert worst < 1e-14


def test_wigner_d_group_law_and_geometry(orc):
    # proj/tests/test_wigner.cpp:154-219 ; proj/tests/python/test_smoke.py:83-91
    rng = orc.Rng(11)
    g1, g2 = rng.rotation(), rng.rotation()
    for l in range(5):
        d1, d2, d12 = orc.wigner_d(l, g1), orc.wigner_d(l, g2), orc.wigner_d(l, g1 @ g2)
        assert np.abs(d1 @ d2 - d12).max() < 1e-10
        assert np.abs(d1 @ d1.T - np.eye(2 * l + 1)).max() < 1e-11
    # x-hat rotated 90 deg about z is y-hat; l=1 components ordered (y, z, x)
    Rz = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    out = orc.rotate([1], [0.0, 0.0, 1.0], Rz)
    assert np.abs(out - [1.0, 0.0, 0.0]).max() < 1e-14


# ------------------------------------------------------------------ sphere
def test_gauss_legendre_vs_scipy(orc):
    # proj/tests/test_sphere.cpp:12-22 (Golub-Welsch oracle)
    from scipy.special import roots_legendre

    for n in [1, 2, 5, 12, 33]:
        a, b = orc.gauss_legendre(n)
        x, w = roots_legendre(n)
        assert np.abs(a - x).max() < 1e-14 and np.abs(b - w).max() < 1e-14


def test_lambda_vs_scipy(orc):
    # proj/tests/test_sphere.cpp:35-51 ; Lambda = sqrt(2-d_m0) * Pbar without CS phase
    from scipy.special import lpmv, factorial

    xs = np.linspace(-0.95, 0.95, 7)
    lam = orc.legendre_lambda(8, xs)
    for l in range(9):
        for m in range(l + 1):
            norm = math.sqrt((2 * l + 1) / (4 * math.pi) * factorial(l - m) / factorial(l + m))
            want = (-1) ** m * lpmv(m, l, xs) * norm * (1.0 if m == 0 else math.sqrt(2))
            assert np.abs(lam[l * (l + 1) // 2 + m] - want).max() < 1e-12


def test_sphere_roundtrip_and_l0_product(orc):
    # proj/tests/test_sphere.cpp:88-99,114-128 ; verify.cpp:256-309
    rng = orc.Rng(SEED)
    for band in range(0, 7):
        x = rng.tower(band)
        back = orc.from_sphere(orc.to_sphere(orc.tower(band), x, band), band, orc.tower(band))
        assert np.abs(back - x).max() < 1e-11
    x, y = rng.tower(3), rng.tower(3)
    z = orc.gtp_grid(orc.tower(3), x, orc.tower(3), y, 6)
    assert z[0] == pytest.approx(np.dot(x, y) / math.sqrt(4 * math.pi), rel=1e-12)


# ------------------------------------------------------------------ CGTP
def test_valid_paths_enumeration(orc):
    # proj/tests/test_cgtp.cpp:13-27
    assert orc.valid_paths(1, 1, 2) == [(0, 0, 0), (0, 1, 1), (1, 0, 1), (1, 1, 0), (1, 1, 1), (1, 1, 2)]
    assert len(orc.valid_paths(2, 2, 4)) == 19 and len(orc.valid_paths(3, 3, 6)) == 44


def test_cgtp_path_kernel_is_contraction(orc):
    # proj/tests/test_cgtp.cpp:29-45 and :47-61 (sparse == naive on all paths L<=6)
    rng = np.random.default_rng(31)
    for (l1, l2, l3) in orc.valid_paths(4, 4, 8):
        x, y = rng.standard_normal(2 * l1 + 1), rng.standard_normal(2 * l2 + 1)
        want = np.zeros(2 * l3 + 1)
        for m1, m2, m3, v in orc.cg_real(l1, l2, l3):
            want[m3 + l3] += v * x[m1 + l1] * y[m2 + l2]
        a = orc.cgtp_path(l1, l2, l3, x, y, "naive")
        b = orc.cgtp_path(l1, l2, l3, x, y, "sparse")
        assert np.abs(a - want).max() < 1e-14 and np.abs(a - b).max() < 1e-12


def test_cgtp_invalid_path_and_mismatch(orc):
    # proj/tests/test_cgtp.cpp:63-79
    assert np.all(orc.cgtp_path(1, 1, 3, np.ones(3), np.ones(3), "sparse") == 0)
    with pytest.raises(ValueError):
        orc.cgtp_path(2, 1, 1, np.zeros(3), np.zeros(3), "sparse")
    with pytest.raises(ValueError):
        orc.cgtp_mimo([0, 1], np.zeros(3), [0, 1], np.zeros(4))


def test_cgtp_mimo_L1_closed_forms(orc):
    # proj/tests/test_cgtp.cpp:81-104
    rng = orc.Rng(33)
    x, y = rng.tower(1), rng.tower(1)
    z = orc.cgtp_mimo([0, 1], x, [0, 1], y)
    assert len(z) == 16
    assert z[0] == pytest.approx(x[0] * y[0], rel=1e-14)
    x1, y1 = x[1:4], y[1:4]
    assert z[4 + 3] == pytest.approx(-np.dot(x1, y1) / math.sqrt(3), rel=1e-12)
    v1 = np.array([x1[2], x1[0], x1[1]])
    v2 = np.array([y1[2], y1[0], y1[1]])
    c = np.cross(v1, v2)
    want = np.array([c[1], c[2], c[0]])
    assert np.abs(z[8:11] + want / math.sqrt(2)).max() < 1e-12


def test_cgtp_equivariance_and_bilinearity(orc):
    # proj/tests/test_cgtp.cpp:113-140
    rng = orc.Rng(35)
    L = 3
    t = orc.tower(L)
    paths = [(a, b, c) for a in t for b in t for c in range(abs(a - b), a + b + 1)]
    out_ls = [c for _, _, c in paths]
    worst = 0.0
    for _ in range(5):
        x, y = rng.tower(L), rng.tower(L)
        R = rng.rotation()
        lhs = orc.cgtp_mimo(t, orc.rotate(t, x, R), t, orc.rotate(t, y, R))
        rhs = orc.rotate(out_ls, orc.cgtp_mimo(t, x, t, y), R)
        worst = max(worst, np.abs(lhs - rhs).max())
    assert worst < 1e-10
    x1, x2, y = rng.tower(2), rng.tower(2), rng.tower(2)
    t2 = orc.tower(2)
    lhs = orc.cgtp_mimo(t2, 2 * x1 - 0.5 * x2, t2, y)
    rhs = 2 * orc.cgtp_mimo(t2, x1, t2, y) - 0.5 * orc.cgtp_mimo(t2, x2, t2, y)
    assert np.abs(lhs - rhs).max() < 1e-12


# ------------------------------------------------------------------ GTP
def _gaunt_contract(orc, x, y, L1, L2, L3):
    z = np.zeros((L3 + 1) ** 2)
    for l1 in range(L1 + 1):
        for l2 in range(L2 + 1):
            for l3 in range(abs(l1 - l2), min(l1 + l2, L3) + 1):
                for m1, m2, m3, v in orc.gaunt_real(l1, l2, l3):
                    z[l3 * l3 + m3 + l3] += v * x[l1 * l1 + m1 + l1] * y[l2 * l2 + m2 + l2]
    return z


def test_gtp_scalar_kat(orc):
    # proj/tests/test_gtp.cpp:36-43
    z = orc.gtp_grid([0], [3.0], [0], [-2.0], 0)
    assert z[0] == pytest.approx(-6 / math.sqrt(4 * math.pi), rel=1e-14)


def test_gtp_grid_equals_gaunt_contraction(orc):
    # proj/tests/test_gtp.cpp:45-57 (1e-10)
    rng = orc.Rng(41)
    for L in range(5):
        for _ in range(5):
            x, y = rng.tower(L), rng.tower(L)
            g = orc.gtp_grid(orc.tower(L), x, orc.tower(L), y, 2 * L)
            assert np.abs(g - _gaunt_contract(orc, x, y, L, L, 2 * L)).max() < 1e-10


def test_gtp_symmetric_and_zero_past_band(orc):
    # proj/tests/test_gtp.cpp:59-72
    rng = orc.Rng(42)
    x, y = rng.tower(3), rng.tower(3)
    t = orc.tower(3)
    assert np.abs(orc.gtp_grid(t, x, t, y, 6) - orc.gtp_grid(t, y, t, x, 6)).max() < 1e-13
    x, y = rng.tower(1), rng.tower(1)
    z = orc.gtp_grid([0, 1], x, [0, 1], y, 5)
    assert np.all(z[9:] == 0.0)


def test_gtp_fourier_equals_grid(orc):
    # proj/tests/test_gtp.cpp:74-86 (1e-8)
    rng = orc.Rng(44)
    for L in range(5):
        for _ in range(5):
            x, y = rng.tower(L), rng.tower(L)
            t = orc.tower(L)
            assert np.abs(orc.gtp_fourier(t, x, t, y, 2 * L) - orc.gtp_grid(t, x, t, y, 2 * L)).max() < 1e-8


def test_fourier_tables_roundtrip_and_sparsity(orc):
    # proj/tests/test_gtp.cpp:88-121
    L = 4
    enc, dec = orc.fourier_tables(L, "encode"), orc.fourier_tables(L, "decode")
    for (l, m), ents in enc.items():
        for u, v, _ in ents:
            assert abs(v) == abs(m) and abs(u) <= l
    rng = orc.Rng(45)
    for _ in range(10):
        x = rng.tower(L)
        spec = {}
        for l in range(L + 1):
            for m in range(-l, l + 1):
                for u, v, w in enc[(l, m)]:
                    spec[(u, v)] = spec.get((u, v), 0) + x[l * l + m + l] * w
        for l in range(L + 1):
            for m in range(-l, l + 1):
                acc = sum(w * spec.get((u, v), 0) for u, v, w in dec[(l, m)])
                assert abs(acc - x[l * l + m + l]) < 1e-10


def test_fourier_table_sizes_match_survey(orc):
    # encode/decode entries at L=6 are 452 / 3,669
    enc, dec = orc.fourier_tables(6, "encode"), orc.fourier_tables(6, "decode")
    assert sum(len(v) for v in enc.values()) == 452
    assert sum(len(v) for v in dec.values()) == 3669


def test_weighted_gtp(orc):
    # proj/tests/test_gtp.cpp:123-153
    rng = orc.Rng(46)
    x, y = rng.tower(2), rng.tower(2)
    t = orc.tower(2)
    a = orc.weighted_gtp(t, x, t, y, np.ones(3), np.ones(3), np.ones(5), 4)
    assert np.abs(a - orc.gtp_grid(t, x, t, y, 4)).max() < 1e-13
    w = np.ones(3); w[1] = 0
    got = orc.weighted_gtp(t, x, t, y, w, np.ones(3), np.ones(5), 4)
    xz = x.copy(); xz[1:4] = 0
    assert np.abs(got - orc.gtp_grid(t, xz, t, y, 4)).max() < 1e-13
    with pytest.raises(ValueError):
        orc.weighted_gtp(t, x, t, y, np.ones(2), np.ones(3), np.ones(5), 4)


def test_gtp_equivariance(orc):
    # proj/tests/test_gtp.cpp:167-185 (1e-9)
    rng = orc.Rng(49)
    t = orc.tower(3)
    out_t = orc.tower(6)
    worst = 0.0
    for _ in range(4):
        x, y = rng.tower(3), rng.tower(3)
        R = rng.rotation()
        rx, ry = orc.rotate(t, x, R), orc.rotate(t, y, R)
        for f in (orc.gtp_grid, orc.gtp_fourier):
            worst = max(worst, np.abs(f(t, rx, t, ry, 6) - orc.rotate(out_t, f(t, x, t, y, 6), R)).max())
    assert worst < 1e-9


# ------------------------------------------------------------------ MTP
def test_mtp_kats(orc):
    # proj/tests/test_mtp.cpp:21-40,73-88
    assert [orc.mtp_l_tilde(*a) for a in [(0, 0, 0), (1, 1, 1), (2, 2, 2), (2, 1, 3), (4, 4, 8)]] == [0, 1, 1, 2, 4]
    for lt in (0, 1, 2):
        X = orc.mtp_embed([0], [3.0], lt)
        d = 2 * lt + 1
        want = 3.0 * (-1) ** lt / math.sqrt(d)
        assert np.abs(X - want * np.eye(d)).max() < 1e-14
    assert orc.mtp([0], [3.0], [0], [-2.0], 0)[0] == pytest.approx(-6.0, rel=1e-14)
    assert orc.mtp([0], [3.0], [0], [-2.0], 0, lt_override=1)[0] == pytest.approx(6 / math.sqrt(3), rel=1e-13)
    with pytest.raises(ValueError):
        orc.mtp(orc.tower(2), np.zeros(9), orc.tower(2), np.zeros(9), 2, lt_override=0)


def test_mtp_naive_sparse_and_paths(orc):
    # proj/tests/test_mtp.cpp:53-64,126-161
    rng = orc.Rng(57)
    for L in range(4):
        t = orc.tower(L)
        lt = orc.mtp_l_tilde(L, L, 2 * L)
        x, y = rng.tower(L), rng.tower(L)
        a = orc.mtp(t, x, t, y, 2 * L, "naive")
        b = orc.mtp(t, x, t, y, 2 * L, "sparse")
        assert np.abs(a - b).max() < 1e-12
        want = np.zeros((2 * L + 1) ** 2)
        for (l1, l2, l3) in orc.valid_paths(L, L, 2 * L):
            w = orc.mtp_path_weight(l1, l2, l3, lt)
            if w == 0.0:
                continue
            seg = orc.cgtp_path(l1, l2, l3, x[l1 * l1:(l1 + 1) ** 2], y[l2 * l2:(l2 + 1) ** 2], "naive")
            want[l3 * l3:(l3 + 1) ** 2] += w * seg
        assert np.abs(b - want).max() < 1e-10
        X = orc.mtp_embed(t, x, orc.mtp_l_tilde(L, L, L))
        assert np.abs(orc.mtp_extract(X, L, orc.mtp_l_tilde(L, L, L)) - x).max() < 1e-13
    assert orc.mtp_path_weight(1, 1, 3, 2) == 0.0 and orc.mtp_path_weight(2, 2, 2, 0) == 0.0
    assert abs(orc.mtp_path_weight(1, 1, 1, 1)) > 1e-3
    assert orc.mtp_path_weight(0, 0, 0, 0) == pytest.approx(1.0, rel=1e-14)


# ------------------------------------------------------------------ op counts
@pytest.mark.parametrize(
    "L,cg_naive,cg_sparse,grid,fourier,mtp_naive,mtp_sparse",
    [
        (1, 200, 208, 261, 508, 180, 65),
        (2, 2450, 1560, 1205, 3328, 1200, 328),
        (3, 14112, 6560, 3297, 11992, 4312, 903),
        (4, 54450, 20008, 6993, 31444, 11340, 2048),
        (6, 414050, 107576, 21021, 130728, 47320, 6378),
    ],
)
def test_count_ops_table(orc, L, cg_naive, cg_sparse, grid, fourier, mtp_naive, mtp_sparse):
    # SURVEY.md Appendix C, restated from proj/src/bench.cpp:101-112 OpCounter rules
    assert orc.count_ops("cgtp", "naive", "mimo", L) == cg_naive
    assert orc.count_ops("cgtp", "sparse", "mimo", L) == cg_sparse
    assert orc.count_ops("gtp", "grid", "mimo", L) == grid
    assert orc.count_ops("gtp", "fourier", "mimo", L) == fourier
    assert orc.count_ops("mtp", "naive", "mimo", L) == mtp_naive
    assert orc.count_ops("mtp", "sparse", "mimo", L) == mtp_sparse


def test_count_ops_closed_forms(orc):
    # proj/tests/python/test_smoke.py:106-111 ; proj/tests/test_mtp.cpp:187-204
    assert orc.count_ops("cgtp", "naive", "siso", 4) == 2 * 9 ** 3
    with pytest.raises(ValueError):
        orc.count_ops("cgtp", "grid", "mimo", 2)
    assert orc.expressivity_count("cgtp", 4) == 85 and orc.expressivity_count("gtp", 4) == 17


def test_batch_matches_single(orc):
    rng = np.random.default_rng(0)
    for kind in ("cgtp", "gtp_grid", "gtp_fourier", "mtp"):
        L = 2
        x = rng.standard_normal((6, 1, 9)); y = rng.standard_normal((6, 1, 9))
        out = orc.batch_mimo(kind, L, x, y, nthreads=3)
        single = {
            "cgtp": lambda a, b: orc.cgtp_mimo(orc.tower(L), a, orc.tower(L), b),
            "gtp_grid": lambda a, b: orc.gtp_grid(orc.tower(L), a, orc.tower(L), b, 2 * L),
            "gtp_fourier": lambda a, b: orc.gtp_fourier(orc.tower(L), a, orc.tower(L), b, 2 * L),
            "mtp": lambda a, b: orc.mtp(orc.tower(L), a, orc.tower(L), b, 2 * L),
        }[kind]
        for b in range(6):
            assert np.abs(out[b, 0] - single(x[b, 0], y[b, 0])).max() < 1e-13
