"""The product's own host table builders (paper_2506_13523_b200/csrc/host/
tables.cpp, exposed through tpo_cg_real / tpo_fourier_table) agree with the
oracle's independent restatement -- CPU only, no device needed."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import pytest


def product_cg(l1, l2, l3):
    import paper_2506_13523_b200 as tpo

    lib = tpo.lib()
    n = lib.tpo_cg_real(l1, l2, l3, None, None, None, None, 0)
    assert n >= 0
    a = np.empty(n, np.int32); b = np.empty(n, np.int32); c = np.empty(n, np.int32); v = np.empty(n)
    p = lambda z: z.ctypes.data_as(C.c_void_p)  # noqa: E731
    assert lib.tpo_cg_real(l1, l2, l3, p(a), p(b), p(c), p(v), n) == n
    return [(int(i), int(j), int(k), float(x)) for i, j, k, x in zip(a, b, c, v)]


def product_fourier(L, which):
    import paper_2506_13523_b200 as tpo

    lib = tpo.lib()
    w = 0 if which == "encode" else 1
    lmax = L if w == 0 else 2 * L
    counts = np.empty((lmax + 1) ** 2, np.int32)
    p = lambda z: z.ctypes.data_as(C.c_void_p)  # noqa: E731
    n = lib.tpo_fourier_table(L, w, p(counts), None, None, None, None, 0)
    u = np.empty(n, np.int32); v = np.empty(n, np.int32); re = np.empty(n); im = np.empty(n)
    assert lib.tpo_fourier_table(L, w, p(counts), p(u), p(v), p(re), p(im), n) == n
    out, k = {}, 0
    for l in range(lmax + 1):
        for m in range(-l, l + 1):
            cnt = int(counts[l * l + m + l])
            out[(l, m)] = {(int(u[k + i]), int(v[k + i])): complex(re[k + i], im[k + i]) for i in range(cnt)}
            k += cnt
    return out


def test_real_cg_matches_oracle(orc):
    worst = 0.0
    for l1 in range(7):
        for l2 in range(7):
            for l3 in range(abs(l1 - l2), l1 + l2 + 1):
                a = product_cg(l1, l2, l3)
                b = orc.cg_real(l1, l2, l3)
                assert [e[:3] for e in a] == [e[:3] for e in b], (l1, l2, l3)
                worst = max(worst, max(abs(x[3] - y[3]) for x, y in zip(a, b)))
    assert worst < 1e-14
    assert product_cg(1, 1, 3) == []


def test_real_cg_large_degree(orc):
    for (l1, l2, l3) in [(16, 16, 32), (16, 16, 7), (12, 9, 10)]:
        a, b = product_cg(l1, l2, l3), orc.cg_real(l1, l2, l3)
        assert len(a) == len(b)
        assert max(abs(x[3] - y[3]) for x, y in zip(a, b)) < 1e-12


@pytest.mark.parametrize("L", [0, 1, 3, 6])
def test_fourier_tables_match_oracle(orc, L):
    for which in ("encode", "decode"):
        a = product_fourier(L, which)
        b = orc.fourier_tables(L, which)
        for key, ents in b.items():
            ref = {(u, v): w for u, v, w in ents}
            got = a[key]
            # entries near the 1e-13 cut may differ in presence; values must agree
            for uv in set(ref) | set(got):
                assert abs(got.get(uv, 0) - ref.get(uv, 0)) < 1e-11, (L, which, key, uv)


# ---------------------------------------------------------------- analysis tables (round 2)
def product_gaunt(l1, l2, l3):
    import paper_2506_13523_b200 as tpo

    lib = tpo.lib()
    n = lib.tpo_gaunt_real(l1, l2, l3, None, None, None, None, 0)
    assert n >= 0
    a = np.empty(n, np.int32); b = np.empty(n, np.int32); c = np.empty(n, np.int32); v = np.empty(n)
    p = lambda z: z.ctypes.data_as(C.c_void_p)  # noqa: E731
    assert lib.tpo_gaunt_real(l1, l2, l3, p(a), p(b), p(c), p(v), n) == n
    return [(int(i), int(j), int(k), float(x)) for i, j, k, x in zip(a, b, c, v)]


@pytest.mark.parametrize("l1,l2,l3", [(0, 0, 0), (1, 1, 1), (1, 1, 2), (2, 4, 2), (3, 2, 3), (4, 4, 6), (5, 3, 4),
                                      (6, 6, 12), (7, 5, 8), (2, 3, 7)])
def test_gaunt_real_matches_oracle(orc, l1, l2, l3):
    # proj/src/wigner.cpp:153-198 (the product builds it by exact quadrature instead)
    mine = product_gaunt(l1, l2, l3)
    ref = orc.gaunt_real(l1, l2, l3)
    assert [e[:3] for e in mine] == [e[:3] for e in ref]
    assert max((abs(a[3] - b[3]) for a, b in zip(mine, ref)), default=0.0) < 1e-13


def test_gaunt_kats():
    # proj/tests/test_wigner.cpp:99-107
    import math

    g = product_gaunt(0, 0, 0)
    assert len(g) == 1 and abs(g[0][3] - 1 / math.sqrt(4 * math.pi)) < 1e-15
    assert product_gaunt(1, 1, 1) == []
    assert len(product_gaunt(2, 4, 2)) > 0


def test_s2_grid_and_legendre_match_oracle(orc):
    import paper_2506_13523_b200 as tpo

    lib = tpo.lib()
    p = lambda z: z.ctypes.data_as(C.c_void_p)  # noqa: E731
    for L in (0, 1, 4, 11, 20):
        nodes = np.empty(L + 1); w = np.empty(L + 1)
        assert lib.tpo_s2_grid(L, p(nodes), p(w)) == 0
        rn, rw = orc.gauss_legendre(L + 1)
        assert np.abs(nodes - rn).max() < 1e-14 and np.abs(w - rw).max() < 1e-14
        lam = np.empty(((L + 1) * (L + 2) // 2, L + 1))
        assert lib.tpo_legendre_lambda(L, p(nodes), L + 1, p(lam)) == 0
        assert np.abs(lam - orc.legendre_lambda(L, nodes)).max() < 1e-12


@pytest.mark.parametrize("l1,l2,l3,lt", [(0, 0, 0, 0), (1, 1, 1, 1), (1, 1, 2, 1), (2, 2, 2, 1), (2, 1, 3, 2),
                                         (3, 3, 4, 3), (4, 2, 2, 3), (1, 1, 1, 3), (2, 2, 5, 2)])
def test_mtp_path_weight_matches_oracle(orc, l1, l2, l3, lt):
    import paper_2506_13523_b200 as tpo

    w = tpo.lib().tpo_mtp_path_weight(l1, l2, l3, lt)
    assert abs(w - orc.mtp_path_weight(l1, l2, l3, lt)) < 1e-12
    if (l1, l2, l3, lt) == (0, 0, 0, 0):
        assert abs(w - 1.0) < 1e-15  # proj/tests/test_mtp.cpp:170


def test_count_muls_matches_oracle(orc):
    # the reference's OpCounter tallies (proj/src/bench.cpp:101-112) for every kind / impl / mode
    import paper_2506_13523_b200 as tpo

    lib = tpo.lib()
    kinds = {"cgtp": (0, ("naive", "sparse")), "gtp": (1, ("grid", "fourier")), "mtp": (2, ("naive", "sparse"))}
    impls = {"naive": 0, "sparse": 1, "grid": 2, "fourier": 3}
    modes = {"siso": 0, "simo": 1, "mimo": 2}
    for kind, (k, ims) in kinds.items():
        for im in ims:
            for mode, md in modes.items():
                for L in (0, 1, 2, 3, 4, 6):
                    assert lib.tpo_count_muls(k, impls[im], md, L) == orc.count_ops(kind, im, mode, L), (kind, im, mode, L)
    assert lib.tpo_count_muls(1, 0, 2, 2) < 0  # naive does not apply to the Gaunt product


@pytest.mark.parametrize("L1,L2,L3", [(0, 0, 0), (1, 1, 2), (3, 2, 4), (2, 4, 7), (4, 4, 8)])
def test_fourier_sep_derivation(orc, L1, L2, L3):
    # the separable torus form of the Fourier GTP the row-quad kernel evaluates
    # (Context::fourier_sep): single phi harmonics per order, rows folded onto [0, pi],
    # pair parity (-1)^(l+m) -- restated in numpy and checked against the oracle
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import fourier_sep_check as fsc

    rng = np.random.default_rng(L1 * 31 + L2 * 7 + L3)
    x = rng.standard_normal((L1 + 1) ** 2)
    y = rng.standard_normal((L2 + 1) ** 2)
    out, t = fsc.separable_fourier(orc, L1, L2, L3, x, y)
    ref = orc.gtp_fourier(orc.tower(L1), x, orc.tower(L2), y, L3)
    assert np.abs(out - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1e-300)
    assert t["resid"] < 1e-12
    assert fsc.pair_parity_error(t["E"]) < 1e-12 and fsc.pair_parity_error(t["D"]) < 1e-12
    # the kernel indexes both tables by |m|
    for T in (t["E"], t["D"]):
        assert max((np.abs(v - T[(l, -m)]).max() for (l, m), v in T.items() if m > 0), default=0.0) < 1e-12
