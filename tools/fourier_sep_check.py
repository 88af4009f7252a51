"""Restates Context::fourier_sep (host/context.cpp) in numpy against the fp64 oracle: the Fourier
GTP's torus convolution (proj/src/gtp.cpp:262-327) evaluated separably -- encode / decode spectra as
single phi harmonics per order, torus rows folded onto theta in [0, pi], the odd azimuth grid of the
grid kernel -- reproduces orc.gtp_fourier, and the row pairs a <-> H - a carry parity (-1)^(l+m).
Importable (tests/test_fourier_sep.py) and runnable: python tools/fourier_sep_check.py [L1 L2 L3]."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def tables(orc, L1, L2, L3):
    L = max(L1, L2)
    band = L1 + L2
    L3e = min(L3, band)
    N = 4 * L + 2
    H = N // 2
    nt = H + 1
    npp = 2 * band + 1
    enc = orc.fourier_tables(L, "encode")
    dec = orc.fourier_tables(L, "decode")
    resid = 0.0

    def harmonic(modes, m, sign, n_a, scale):
        nonlocal resid
        a = np.arange(n_a)
        cc = np.zeros(n_a); ss = np.zeros(n_a)
        for (u, v, w) in modes:
            assert abs(v) == abs(m)
            c = w * np.exp(sign * 2j * np.pi * u * a / N) * scale
            im = -c.imag if sign > 0 else c.imag
            cc += c.real
            if v != 0:
                ss += im if v > 0 else -im
        resid = max(resid, float(np.abs(ss if m >= 0 else cc).max()))
        return cc if m >= 0 else ss

    E = {}
    for l in range(L + 1):
        for m in range(-l, l + 1):
            E[(l, m)] = harmonic(enc[(l, m)], m, +1, nt, 1.0)
    D = {}
    for l in range(L3e + 1):
        for m in range(-l, l + 1):
            q = harmonic(dec[(l, m)], m, -1, N, 1.0 / N ** 2)
            sg = (-1) ** abs(m)
            f = q[:nt].copy()
            f[1:H] += sg * q[N - np.arange(1, H)]
            D[(l, m)] = (N / npp) * f
    return dict(E=E, D=D, nt=nt, H=H, npp=npp, L3e=L3e, resid=resid)


def pair_parity_error(T):
    return max(float(np.abs(v[::-1] - (-1) ** (l + abs(m)) * v).max()) for (l, m), v in T.items())


def separable_fourier(orc, L1, L2, L3, x, y):
    t = tables(orc, L1, L2, L3)
    phi = 2 * np.pi * np.arange(t["npp"]) / t["npp"]

    def trig(m):
        return np.cos(m * phi) if m >= 0 else np.sin(-m * phi)

    def torus(v, Lx):
        f = np.zeros((t["nt"], t["npp"]))
        for l in range(Lx + 1):
            for m in range(-l, l + 1):
                f += v[l * l + l + m] * np.outer(t["E"][(l, m)], trig(m))
        return f

    h = torus(x, L1) * torus(y, L2)
    out = np.zeros((L3 + 1) ** 2)
    for (l, m), d in t["D"].items():
        out[l * l + l + m] = np.sum(h * np.outer(d, trig(m)))
    return out, t


def main():
    import oracle.oracle as orc

    L1, L2, L3 = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (3, 3, 6)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((L1 + 1) ** 2); y = rng.standard_normal((L2 + 1) ** 2)
    out, t = separable_fourier(orc, L1, L2, L3, x, y)
    ref = orc.gtp_fourier(orc.tower(L1), x, orc.tower(L2), y, L3)
    print({"err": float(np.abs(out - ref).max() / np.abs(ref).max()), "resid": t["resid"],
           "parity_E": pair_parity_error(t["E"]), "parity_D": pair_parity_error(t["D"])})


if __name__ == "__main__":
    main()
