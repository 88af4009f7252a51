"""Mirror of the reference Python module ``so3tpo`` (proj/bindings/py_core.cpp,
proj/python/so3tpo/__init__.py) for the tensor-product entry points: one
product per call, irreps strings, numpy fp64 vectors in and out, ValueError
on bad input (proj/README.md:149-152).  Computation runs on the B200 through
the C ABI (tpo_run_host_f32); results are fp32-accurate (normwise 1e-5).

Provided: irreps_dim, single_copies, cg_table (real CG or Gaunt), cgtp, gtp
(impl "grid" | "fourier"), mtp, mtp_path_weights, wigner_d, rotate (GPU),
count_ops (the reference's instrumented multiply counts).  The analysis
suites of the reference module (expressivity_*, interactable, verify*) are
outside the hot path and not provided.
"""
from __future__ import annotations

import ctypes as C
import re

import numpy as np

from ._lib import KINDS, TPO_EINVAL, check, context, lib

_ENTRY = re.compile(r"^(\d+)x(\d+)$")


def _parse(irreps: str):
    """Irreps::parse (proj/src/irreps.cpp:20-49): '2x1+1x0' -> [(2, 1), (1, 0)]."""
    if irreps == "":
        return []
    out = []
    for part in irreps.split("+"):
        m = _ENTRY.match(part)
        if not m:
            raise ValueError(f"irreps: cannot parse '{irreps}'")
        mul, l = int(m.group(1)), int(m.group(2))
        if mul < 1:
            raise ValueError("irreps: multiplicity must be >= 1")
        out.append((mul, l))
    return out


def irreps_dim(irreps: str) -> int:
    return sum(mul * (2 * l + 1) for mul, l in _parse(irreps))


def single_copies(L: int) -> str:
    if L < 0:
        raise ValueError("single_copies: L must be >= 0")
    return "+".join(f"1x{l}" for l in range(L + 1))


def cg_table(l1: int, l2: int, l3: int, gaunt: bool = False):
    """Sparse real coupling table as (m1, m2, m3, value) tuples: real CG or, with gaunt=True, the
    real Gaunt coefficients (py_core.cpp:62-72)."""
    fn = lib().tpo_gaunt_real if gaunt else lib().tpo_cg_real
    n = fn(l1, l2, l3, None, None, None, None, 0)
    if n < 0:
        check(-n)
    a = np.empty(n, np.int32); b = np.empty(n, np.int32); c = np.empty(n, np.int32); v = np.empty(n)
    p = lambda z: z.ctypes.data_as(C.c_void_p)  # noqa: E731
    fn(l1, l2, l3, p(a), p(b), p(c), p(v), n)
    return [(int(i), int(j), int(k), float(x)) for i, j, k, x in zip(a, b, c, v)]


def mtp_path_weights(l1: int, l2: int, l3: int, l_tilde: int) -> float:
    """Per-path CG weight realized by the matrix product (py_core.cpp:110-116)."""
    w = lib().tpo_mtp_path_weight(l1, l2, l3, l_tilde)
    if w != w:
        check(TPO_EINVAL)
    return float(w)


_KIND = {"cgtp": 0, "gtp": 1, "mtp": 2}
_IMPL = {"naive": 0, "sparse": 1, "grid": 2, "fourier": 3}
_MODE = {"siso": 0, "simo": 1, "mimo": 2}


def count_ops(kind: str, impl: str, mode: str, L: int) -> int:
    """Instrumented multiply count for one application (py_core.cpp:157-172)."""
    if kind not in _KIND:
        raise ValueError(f"unknown kind '{kind}'")
    if impl not in _IMPL:
        raise ValueError(f"unknown impl '{impl}'")
    if mode not in _MODE:
        raise ValueError(f"unknown mode '{mode}'")
    r = int(lib().tpo_count_muls(_KIND[kind], _IMPL[impl], _MODE[mode], L))
    if r < 0:
        check(-r)
    return r


def _axis_angle(axis, angle):
    """Rotation::from_axis_angle (proj/src/wigner.cpp:200-206), row-major 3x3."""
    a = np.asarray(axis, dtype=np.float64).reshape(3)
    n = float(np.linalg.norm(a))
    if n == 0.0:
        raise ValueError("rotation: zero axis")
    u = a / n
    c, s = np.cos(angle), np.sin(angle)
    K = np.array([[0, -u[2], u[1]], [u[2], 0, -u[0]], [-u[1], u[0], 0]])
    return c * np.eye(3) + (1 - c) * np.outer(u, u) + s * K


def wigner_d(l: int, axis, angle: float):
    """Real Wigner-D matrix of the rotation by `angle` about `axis` (py_core.cpp:118-124), computed
    on the GPU (tpo_wigner_d_f64)."""
    import torch

    if l < 0:
        raise ValueError("wigner_d: negative degree")
    R = torch.from_numpy(_axis_angle(axis, angle)[None]).cuda()
    from . import wigner_d as _wd

    return _wd(R, l)[l][0].cpu().numpy()


def rotate(irreps: str, x, axis, angle: float):
    """Apply a rotation blockwise through the Wigner-D matrices (py_core.cpp:126-133), on the GPU
    (tpo_rotate_f32)."""
    import torch

    from . import rotate as _rot

    ents, data = _vector(irreps, x)
    if not ents:
        return data.copy()
    L = max(l for _, l in ents)
    rows, offs, off = [], [], 0
    for mul, l in ents:  # one row per copy: a tower of the largest degree holding that block
        for _ in range(mul):
            r = np.zeros((L + 1) ** 2, np.float32)
            r[l * l:(l + 1) ** 2] = data[off:off + 2 * l + 1]
            rows.append(r)
            offs.append((l, off))
            off += 2 * l + 1
    R = torch.from_numpy(_axis_angle(axis, angle)[None]).cuda()
    out = _rot(torch.from_numpy(np.stack(rows)).cuda(), R, L).cpu().numpy().astype(np.float64)
    res = np.empty_like(data)
    for i, (l, o) in enumerate(offs):
        res[o:o + 2 * l + 1] = out[i, l * l:(l + 1) ** 2]
    return res


def _vector(irreps: str, data):
    ents = _parse(irreps)
    data = np.asarray(data, dtype=np.float64).reshape(-1)
    dim = sum(mul * (2 * l + 1) for mul, l in ents)
    if data.shape[0] != dim:
        raise ValueError(f"data length {data.shape[0]} does not match irreps dim {dim}")
    return ents, data


def _tower(ents, data, L):
    """Sum every copy into a 0..L tower (exact for the Gaunt / matrix products)."""
    t = np.zeros((L + 1) ** 2, np.float64)
    off = 0
    for mul, l in ents:
        for _ in range(mul):
            t[l * l:(l + 1) ** 2] += data[off:off + 2 * l + 1]
            off += 2 * l + 1
    return t.astype(np.float32)


def _run_host(kind, L1, L2, L3, lt, X, Y, B):
    out = np.empty((B, int(lib().tpo_out_dim(KINDS[kind], L1, L2, L3))), np.float32)
    X = np.ascontiguousarray(X, np.float32); Y = np.ascontiguousarray(Y, np.float32)
    p = lambda z: z.ctypes.data_as(C.c_void_p)  # noqa: E731
    check(lib().tpo_run_host_f32(context().handle, KINDS[kind], L1, L2, L3, lt, p(X), p(Y), p(out), B, 1, 0))
    return out.astype(np.float64)


def cgtp(x_irreps: str, x, y_irreps: str, y, impl: str = "sparse"):
    """Clebsch-Gordan product over all valid paths; returns (irreps, data)."""
    ex, xd = _vector(x_irreps, x)
    ey, yd = _vector(y_irreps, y)
    if any(m != 1 for m, _ in ex) or any(m != 1 for m, _ in ey):
        raise ValueError("cgtp_mimo: inputs must be single-copy towers")
    L1 = max((l for _, l in ex), default=0)
    L2 = max((l for _, l in ey), default=0)
    d1, d2 = (L1 + 1) ** 2, (L2 + 1) ** 2
    pairs = [(i, j) for i in range(len(ex)) for j in range(len(ey))]
    X = np.zeros((max(len(pairs), 1), d1)); Y = np.zeros((max(len(pairs), 1), d2))
    xoff = np.cumsum([0] + [2 * l + 1 for _, l in ex]); yoff = np.cumsum([0] + [2 * l + 1 for _, l in ey])
    for r, (i, j) in enumerate(pairs):
        li, lj = ex[i][1], ey[j][1]
        X[r, li * li:(li + 1) ** 2] = xd[xoff[i]:xoff[i + 1]]
        Y[r, lj * lj:(lj + 1) ** 2] = yd[yoff[j]:yoff[j + 1]]
    full = _run_host("cgtp", L1, L2, 0, -1, X, Y, len(pairs)) if pairs else np.zeros((0, 0))
    # path offsets inside the 0..L1 x 0..L2 tower output (proj/src/cgtp.cpp:152-163)
    offs, o = {}, 0
    for a in range(L1 + 1):
        for b in range(L2 + 1):
            for c in range(abs(a - b), a + b + 1):
                offs[(a, b, c)] = o
                o += 2 * c + 1
    out_irreps, out = [], []
    for r, (i, j) in enumerate(pairs):
        li, lj = ex[i][1], ey[j][1]
        for l3 in range(abs(li - lj), li + lj + 1):
            out_irreps.append(f"1x{l3}")
            s = offs[(li, lj, l3)]
            out.append(full[r, s:s + 2 * l3 + 1])
    return "+".join(out_irreps), (np.concatenate(out) if out else np.zeros(0))


def gtp(x_irreps: str, x, y_irreps: str, y, L3: int, impl: str = "grid"):
    """Gaunt product with outputs 0..L3 (grid or fourier); returns (irreps, data)."""
    if L3 < 0:
        raise ValueError("gtp: L3 must be >= 0")
    ex, xd = _vector(x_irreps, x)
    ey, yd = _vector(y_irreps, y)
    L1 = max((l for _, l in ex), default=0)
    L2 = max((l for _, l in ey), default=0)
    kind = "gtp_fourier" if impl == "fourier" else "gtp_grid"
    out = _run_host(kind, L1, L2, L3, -1, _tower(ex, xd, L1)[None], _tower(ey, yd, L2)[None], 1)[0]
    return single_copies(L3), out


def mtp(x_irreps: str, x, y_irreps: str, y, L3: int, impl: str = "sparse"):
    """Matrix tensor product with outputs 0..L3; returns (irreps, data)."""
    if L3 < 0:
        raise ValueError("mtp: L3 must be >= 0")
    ex, xd = _vector(x_irreps, x)
    ey, yd = _vector(y_irreps, y)
    L1 = max((l for _, l in ex), default=0)
    L2 = max((l for _, l in ey), default=0)
    out = _run_host("mtp", L1, L2, L3, -1, _tower(ex, xd, L1)[None], _tower(ey, yd, L2)[None], 1)[0]
    return single_copies(L3), out
