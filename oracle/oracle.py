"""ctypes wrapper around the fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package
(paper_2506_13523_b200) never does.  The oracle restates the reference CPU
path (/root/reference/proj/src/*.cpp) in fp64; see oracle/tpo_oracle.h for
its pinning status.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "libtpo_oracle.so"

KINDS = {"cgtp": 0, "gtp": 1, "mtp": 2}
IMPLS = {"naive": 0, "sparse": 1, "grid": 2, "fourier": 3}
MODES = {"siso": 0, "simo": 1, "mimo": 2}


class OracleError(RuntimeError):
    pass


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    if not _LIB_PATH.exists():
        build()
    lib = C.CDLL(str(_LIB_PATH))
    i, d, p = C.c_int, C.c_double, C.c_void_p
    u64 = C.c_uint64
    P = C.POINTER
    sig = {
        "orc_last_error": (C.c_char_p, []),
        "orc_rng_new": (p, [u64]),
        "orc_rng_free": (None, [p]),
        "orc_rng_irrep_random": (None, [p, i, p]),
        "orc_rng_rotation": (None, [p, p]),
        "orc_cg_coefficient": (d, [i, i, i, i, i, i]),
        "orc_real_basis_change": (None, [i, p, p]),
        "orc_cg_real": (i, [i, i, i, p, p, p, p, i]),
        "orc_gaunt_real": (i, [i, i, i, p, p, p, p, i]),
        "orc_wigner_d": (i, [i, p, p]),
        "orc_rotate": (i, [p, i, p, p, p]),
        "orc_gauss_legendre": (i, [i, p, p]),
        "orc_legendre_lambda": (i, [i, p, i, p]),
        "orc_to_sphere": (i, [p, i, p, i, p, P(u64)]),
        "orc_from_sphere_select": (i, [i, p, p, i, p, P(u64)]),
        "orc_num_paths": (i, [i, i, i]),
        "orc_valid_paths": (i, [i, i, i, p, p, p, i]),
        "orc_cgtp_path": (i, [i, i, i, i, p, i, p, i, p, i, P(u64)]),
        "orc_cgtp_mimo": (i, [i, p, i, p, p, i, p, p, P(u64)]),
        "orc_gtp_grid_select": (i, [p, i, p, p, i, p, p, i, p, P(u64)]),
        "orc_gtp_fourier_select": (i, [p, i, p, p, i, p, p, i, p, P(u64)]),
        "orc_weighted_gtp": (i, [p, i, p, p, i, p, p, i, p, i, p, i, i, p, P(u64)]),
        "orc_fourier_tables": (i, [i, i, p, p, p, p, p, i]),
        "orc_mtp_l_tilde": (i, [i, i, i]),
        "orc_mtp_embed": (i, [p, i, p, i, i, p, P(u64)]),
        "orc_mtp_matmul": (i, [i, p, p, p, P(u64)]),
        "orc_mtp_extract_select": (i, [i, p, p, i, i, i, p, P(u64)]),
        "orc_mtp": (i, [p, i, p, p, i, p, i, i, i, p, P(u64)]),
        "orc_mtp_path_weight": (d, [i, i, i, i]),
        "orc_count_ops": (C.c_int64, [i, i, i, i]),
        "orc_expressivity_count": (C.c_long, [i, i]),
        "orc_mimo_out_dim": (i, [i, i]),
        "orc_batch_mimo": (i, [i, i, i, C.c_int64, i, i, p, p, p, i]),
        "orc_batch_mimo_f32": (i, [i, i, i, C.c_int64, i, i, p, p, p, i]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ints(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _check(rc: int) -> int:
    if rc < 0:
        msg = lib().orc_last_error().decode()
        if rc == -1:
            raise ValueError(msg)
        if rc == -2:
            raise IndexError(msg)
        raise OracleError(msg)
    return rc


def tower(L: int) -> list[int]:
    return list(range(L + 1))


def dim(ls) -> int:
    return int(sum(2 * l + 1 for l in ls))


# ---------------------------------------------------------------- RNG
class Rng:
    """std::mt19937_64 with the reference's per-vector normal_distribution."""

    def __init__(self, seed: int = 20240901):
        self._h = lib().orc_rng_new(seed)

    def __del__(self):
        try:
            lib().orc_rng_free(self._h)
        except Exception:
            pass

    def irrep(self, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        lib().orc_rng_irrep_random(self._h, n, _ptr(out))
        return out

    def tower(self, L: int) -> np.ndarray:
        return self.irrep((L + 1) ** 2)

    def rotation(self) -> np.ndarray:
        R = np.empty((3, 3), np.float64)
        lib().orc_rng_rotation(self._h, _ptr(R))
        return R


# ---------------------------------------------------------------- tables
def cg_coefficient(l1, m1, l2, m2, l3, m3) -> float:
    return lib().orc_cg_coefficient(l1, m1, l2, m2, l3, m3)


def real_basis_change(l: int) -> np.ndarray:
    d = 2 * l + 1
    re = np.empty((d, d)); im = np.empty((d, d))
    lib().orc_real_basis_change(l, _ptr(re), _ptr(im))
    return re + 1j * im


def _table(fn, l1, l2, l3):
    n = _check(fn(l1, l2, l3, None, None, None, None, 0))
    m1 = np.empty(n, np.int32); m2 = np.empty(n, np.int32); m3 = np.empty(n, np.int32)
    v = np.empty(n, np.float64)
    _check(fn(l1, l2, l3, _ptr(m1), _ptr(m2), _ptr(m3), _ptr(v), n))
    return [(int(a), int(b), int(c), float(x)) for a, b, c, x in zip(m1, m2, m3, v)]


def cg_real(l1, l2, l3):
    return _table(lib().orc_cg_real, l1, l2, l3)


def gaunt_real(l1, l2, l3):
    return _table(lib().orc_gaunt_real, l1, l2, l3)


def wigner_d(l: int, R: np.ndarray) -> np.ndarray:
    D = np.empty((2 * l + 1, 2 * l + 1))
    _check(lib().orc_wigner_d(l, _ptr(_f64(R)), _ptr(D)))
    return D


def rotate(ls, x, R) -> np.ndarray:
    ls = _ints(ls); x = _f64(x)
    out = np.empty_like(x)
    _check(lib().orc_rotate(_ptr(ls), len(ls), _ptr(x), _ptr(_f64(R)), _ptr(out)))
    return out


def gauss_legendre(n: int):
    a = np.empty(n); b = np.empty(n)
    _check(lib().orc_gauss_legendre(n, _ptr(a), _ptr(b)))
    return a, b


def legendre_lambda(lmax: int, cos_theta) -> np.ndarray:
    c = _f64(cos_theta)
    rows = (lmax + 1) * (lmax + 2) // 2
    out = np.empty((rows, len(c)))
    _check(lib().orc_legendre_lambda(lmax, _ptr(c), len(c), _ptr(out)))
    return out


def to_sphere(ls, x, Lgrid: int) -> np.ndarray:
    ls = _ints(ls)
    F = np.empty((Lgrid + 1, 2 * Lgrid + 1))
    _check(lib().orc_to_sphere(_ptr(ls), len(ls), _ptr(_f64(x)), Lgrid, _ptr(F), None))
    return F


def from_sphere(F, Lgrid: int, degrees) -> np.ndarray:
    deg = _ints(degrees)
    out = np.empty(dim(degrees))
    _check(lib().orc_from_sphere_select(Lgrid, _ptr(_f64(F)), _ptr(deg), len(deg), _ptr(out), None))
    return out


# ---------------------------------------------------------------- products
def valid_paths(L1, L2, L3):
    n = lib().orc_num_paths(L1, L2, L3)
    a = np.empty(n, np.int32); b = np.empty(n, np.int32); c = np.empty(n, np.int32)
    _check(lib().orc_valid_paths(L1, L2, L3, _ptr(a), _ptr(b), _ptr(c), n))
    return list(zip(a.tolist(), b.tolist(), c.tolist()))


def _ops():
    return C.c_uint64(0)


def cgtp_path(l1, l2, l3, x, y, impl="sparse", count=False):
    x = _f64(x); y = _f64(y)
    out = np.empty(2 * l3 + 1)
    ops = _ops()
    _check(lib().orc_cgtp_path(IMPLS[impl], l1, l2, l3, _ptr(x), len(x), _ptr(y), len(y),
                               _ptr(out), len(out), C.byref(ops)))
    return (out, ops.value) if count else out


def cgtp_mimo(xls, x, yls, y, impl="sparse", count=False):
    xls = _ints(xls); yls = _ints(yls); x = _f64(x); y = _f64(y)
    if len(x) != dim(xls) or len(y) != dim(yls):
        raise ValueError("data length does not match irreps dim")
    n = _check(lib().orc_cgtp_mimo(IMPLS[impl], _ptr(xls), len(xls), _ptr(x), _ptr(yls), len(yls),
                                   _ptr(y), None, None))
    out = np.empty(n)
    ops = _ops()
    _check(lib().orc_cgtp_mimo(IMPLS[impl], _ptr(xls), len(xls), _ptr(x), _ptr(yls), len(yls),
                               _ptr(y), _ptr(out), C.byref(ops)))
    return (out, ops.value) if count else out


def _gtp(fn, xls, x, yls, y, degrees, count):
    xls = _ints(xls); yls = _ints(yls); x = _f64(x); y = _f64(y); deg = _ints(degrees)
    out = np.empty(dim(degrees))
    ops = _ops()
    _check(fn(_ptr(xls), len(xls), _ptr(x), _ptr(yls), len(yls), _ptr(y), _ptr(deg), len(deg),
              _ptr(out), C.byref(ops)))
    return (out, ops.value) if count else out


def gtp_grid(xls, x, yls, y, L3, count=False):
    return _gtp(lib().orc_gtp_grid_select, xls, x, yls, y, list(range(L3 + 1)), count)


def gtp_fourier(xls, x, yls, y, L3, count=False):
    return _gtp(lib().orc_gtp_fourier_select, xls, x, yls, y, list(range(L3 + 1)), count)


def gtp_grid_select(xls, x, yls, y, degrees, count=False):
    return _gtp(lib().orc_gtp_grid_select, xls, x, yls, y, degrees, count)


def gtp_fourier_select(xls, x, yls, y, degrees, count=False):
    return _gtp(lib().orc_gtp_fourier_select, xls, x, yls, y, degrees, count)


def weighted_gtp(xls, x, yls, y, a, b, c, L3):
    xls = _ints(xls); yls = _ints(yls); x = _f64(x); y = _f64(y)
    a = _f64(a); b = _f64(b); c = _f64(c)
    out = np.empty((L3 + 1) ** 2)
    _check(lib().orc_weighted_gtp(_ptr(xls), len(xls), _ptr(x), _ptr(yls), len(yls), _ptr(y),
                                  _ptr(a), len(a), _ptr(b), len(b), _ptr(c), len(c), L3, _ptr(out),
                                  None))
    return out


def fourier_tables(L: int, which: str = "encode"):
    """-> dict (l, m) -> list of (u, v, complex w)."""
    w = 0 if which == "encode" else 1
    lmax = L if w == 0 else 2 * L
    counts = np.empty((lmax + 1) ** 2, np.int32)
    n = _check(lib().orc_fourier_tables(L, w, _ptr(counts), None, None, None, None, 0))
    u = np.empty(n, np.int32); v = np.empty(n, np.int32); re = np.empty(n); im = np.empty(n)
    _check(lib().orc_fourier_tables(L, w, _ptr(counts), _ptr(u), _ptr(v), _ptr(re), _ptr(im), n))
    out = {}
    k = 0
    for l in range(lmax + 1):
        for m in range(-l, l + 1):
            c = int(counts[l * l + m + l])
            out[(l, m)] = [(int(u[k + i]), int(v[k + i]), complex(re[k + i], im[k + i])) for i in range(c)]
            k += c
    return out


def mtp_l_tilde(L1, L2, L3) -> int:
    return lib().orc_mtp_l_tilde(L1, L2, L3)


def mtp_embed(ls, x, lt, impl="sparse", count=False):
    ls = _ints(ls)
    X = np.empty((2 * lt + 1, 2 * lt + 1))
    ops = _ops()
    _check(lib().orc_mtp_embed(_ptr(ls), len(ls), _ptr(_f64(x)), lt, IMPLS[impl], _ptr(X), C.byref(ops)))
    return (X, ops.value) if count else X


def mtp_matmul(X, Y, count=False):
    X = _f64(X); Y = _f64(Y)
    Z = np.empty_like(X)
    ops = _ops()
    _check(lib().orc_mtp_matmul(X.shape[0], _ptr(X), _ptr(Y), _ptr(Z), C.byref(ops)))
    return (Z, ops.value) if count else Z


def mtp_extract(Z, L3, lt, impl="sparse"):
    Z = _f64(Z); deg = _ints(list(range(L3 + 1)))
    out = np.empty((L3 + 1) ** 2)
    _check(lib().orc_mtp_extract_select(Z.shape[0], _ptr(Z), _ptr(deg), len(deg), lt, IMPLS[impl],
                                        _ptr(out), None))
    return out


def mtp(xls, x, yls, y, L3, impl="sparse", lt_override=-1, count=False):
    xls = _ints(xls); yls = _ints(yls)
    out = np.empty((L3 + 1) ** 2)
    ops = _ops()
    _check(lib().orc_mtp(_ptr(xls), len(xls), _ptr(_f64(x)), _ptr(yls), len(yls), _ptr(_f64(y)), L3,
                         IMPLS[impl], lt_override, _ptr(out), C.byref(ops)))
    return (out, ops.value) if count else out


def mtp_path_weight(l1, l2, l3, lt) -> float:
    return lib().orc_mtp_path_weight(l1, l2, l3, lt)


def count_ops(kind: str, impl: str, mode: str, L: int) -> int:
    r = lib().orc_count_ops(KINDS[kind], IMPLS[impl], MODES[mode], L)
    _check(int(r) if r < 0 else 0)
    return int(r)


def expressivity_count(kind: str, L: int) -> int:
    return int(lib().orc_expressivity_count(KINDS[kind], L))


def mimo_out_dim(kind: str, L: int) -> int:
    return lib().orc_mimo_out_dim(KINDS[kind], L)


# kind names used by the product API -> (oracle kind, oracle impl)
PRODUCT_KINDS = {
    "cgtp": ("cgtp", "sparse"),
    "gtp_grid": ("gtp", "grid"),
    "gtp_fourier": ("gtp", "fourier"),
    "mtp": ("mtp", "sparse"),
}


def batch_mimo(kind: str, L: int, x, y, *, channels: int = 1, y_shared: bool = False,
               nthreads: int | None = None) -> np.ndarray:
    """Batched MIMO application, fp64 or fp32 arrays [B][C][Din]."""
    okind, oimpl = PRODUCT_KINDS.get(kind, (kind, None))
    if oimpl is None:
        raise ValueError(kind)
    nthreads = nthreads or os.cpu_count() or 1
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    B = x.shape[0]
    dout = mimo_out_dim(okind, L)
    if x.dtype == np.float32:
        out = np.empty((B, channels, dout), np.float32)
        fn = lib().orc_batch_mimo_f32
        y = y.astype(np.float32, copy=False)
    else:
        x = x.astype(np.float64, copy=False); y = y.astype(np.float64, copy=False)
        out = np.empty((B, channels, dout), np.float64)
        fn = lib().orc_batch_mimo
    _check(fn(KINDS[okind], IMPLS[oimpl], L, B, channels, int(y_shared), _ptr(x), _ptr(y), _ptr(out),
              nthreads))
    return out
