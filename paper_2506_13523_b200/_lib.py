"""ctypes binding of libtpo_b200.so (the C ABI in include/tpo_capi.h).

The shared library is built in-tree (``python -c 'import __graft_entry__ as g;
g.build()'`` or ``make -C paper_2506_13523_b200/csrc``).  There is no CPU or
pure-PyTorch fallback: if the library is missing or the device is not an
sm_100 part, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libtpo_b200.so"
if os.environ.get("TPO_LIB_PATH"):  # A/B timing of an alternative in-tree build (tools/ab_timing.sh)
    LIB_PATH = Path(os.environ["TPO_LIB_PATH"]).resolve()

TPO_OK, TPO_EINVAL, TPO_ERANGE, TPO_ERUNTIME, TPO_ECUDA = 0, 1, 2, 3, 4
KIND_CGTP, KIND_GTP_GRID, KIND_GTP_FOURIER, KIND_MTP = 0, 1, 2, 3
KINDS = {"cgtp": KIND_CGTP, "gtp_grid": KIND_GTP_GRID, "gtp_fourier": KIND_GTP_FOURIER, "mtp": KIND_MTP}


class HostRequest(C.Structure):
    """Mirror of tpo_host_request (include/tpo_capi.h)."""

    _fields_ = [("kind", C.c_int), ("L1", C.c_int), ("L2", C.c_int), ("L3", C.c_int), ("l_tilde", C.c_int),
                ("y_shared", C.c_int), ("batch", C.c_int64), ("channels", C.c_int64), ("x", C.c_void_p),
                ("y", C.c_void_p), ("out", C.c_void_p)]


class TpoError(RuntimeError):
    """CUDA / runtime failure inside libtpo_b200 (TPO_ECUDA, TPO_ERUNTIME)."""


_lib = None
_lock = threading.RLock()  # reentrant: context() -> Context() -> lib()


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE / 'csrc'}` "
                "(there is no fallback implementation)"
            )
        L = C.CDLL(str(LIB_PATH))
        i, i64, p, d = C.c_int, C.c_int64, C.c_void_p, C.c_double
        sig = {
            "tpo_last_error": (C.c_char_p, []),
            "tpo_version": (C.c_char_p, []),
            "tpo_ctx_create": (i, [i, C.POINTER(p)]),
            "tpo_ctx_destroy": (i, [p]),
            "tpo_ctx_launches": (i64, [p]),
            "tpo_tower_dim": (i64, [i]),
            "tpo_out_dim": (i64, [i, i, i, i]),
            "tpo_mtp_l_tilde": (i, [i, i, i]),
            "tpo_cgtp_mimo_f32": (i, [p, i, i, p, p, p, i64, i64, i, p]),
            "tpo_gtp_grid_f32": (i, [p, i, i, i, p, p, p, i64, i64, i, p]),
            "tpo_gtp_fourier_f32": (i, [p, i, i, i, p, p, p, i64, i64, i, p]),
            "tpo_mtp_f32": (i, [p, i, i, i, i, p, p, p, i64, i64, i, p]),
            "tpo_weighted_gtp_f32": (i, [p, i, i, i, p, p, p, p, p, p, i64, i64, i, p]),
            "tpo_run_f32": (i, [p, i, i, i, i, i, p, p, p, i64, i64, i, p]),
            "tpo_backward_f32": (i, [p, i, i, i, i, i, p, p, p, p, p, i64, i64, i, p]),
            "tpo_run_host_f32": (i, [p, i, i, i, i, i, p, p, p, i64, i64, i]),
            "tpo_run_host_batch_f32": (i, [p, p, i]),
            "tpo_set_gtp_grid_path": (i, [p, i]),
            "tpo_cg_real": (i, [i, i, i, p, p, p, p, i]),
            "tpo_fourier_table": (i, [i, i, p, p, p, p, p, i]),
            "tpo_last_gtp_grid_path": (i, [p]),
            "tpo_to_sphere_f32": (i, [p, i, i, p, p, i64, p]),
            "tpo_from_sphere_f32": (i, [p, i, p, i, p, p, i64, p]),
            "tpo_pointwise_mul_f32": (i, [p, p, p, p, i64, p]),
            "tpo_mtp_embed_f32": (i, [p, i, i, p, p, i64, p]),
            "tpo_mtp_matmul_f32": (i, [p, i, p, p, p, i64, p]),
            "tpo_mtp_extract_f32": (i, [p, i, p, i, p, p, i64, p]),
            "tpo_apply_linear_f32": (i, [p, p, p, i, p, p, i, p, i, p, p, i64, p]),
            "tpo_wigner_d_f64": (i, [p, i, p, p, i64, p]),
            "tpo_wigner_d_size": (i64, [i]),
            "tpo_rotate_f32": (i, [p, i, p, i64, p, p, i64, i64, p]),
            "tpo_gaunt_real": (i, [i, i, i, p, p, p, p, i]),
            "tpo_s2_grid": (i, [i, p, p]),
            "tpo_legendre_lambda": (i, [i, p, i, p]),
            "tpo_mtp_path_weight": (d, [i, i, i, i]),
            "tpo_count_muls": (i64, [i, i, i, i]),
            "tpo_cgtp_num_paths": (i, [i, i]),
            "tpo_set_precision": (i, [p, i]),
            "tpo_cgtp_weighted_f32": (i, [p, i, i, p, i, p, p, p, i64, i64, i, p]),
        }
        for name, (res, args) in sig.items():
            if os.environ.get("TPO_LIB_PATH") and not hasattr(L, name):
                continue  # A/B timing of an older build (tools/gpu_*.sh): bind what it has
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return _lib


EXPORTED = [
    "tpo_last_error", "tpo_version", "tpo_ctx_create", "tpo_ctx_destroy", "tpo_ctx_launches",
    "tpo_tower_dim", "tpo_out_dim", "tpo_mtp_l_tilde", "tpo_cgtp_mimo_f32", "tpo_gtp_grid_f32",
    "tpo_gtp_fourier_f32", "tpo_mtp_f32", "tpo_weighted_gtp_f32", "tpo_run_f32", "tpo_run_host_f32",
    "tpo_run_host_batch_f32", "tpo_backward_f32",
    "tpo_set_gtp_grid_path", "tpo_last_gtp_grid_path", "tpo_cg_real", "tpo_fourier_table",
    "tpo_to_sphere_f32", "tpo_from_sphere_f32", "tpo_pointwise_mul_f32", "tpo_mtp_embed_f32", "tpo_mtp_matmul_f32",
    "tpo_mtp_extract_f32", "tpo_apply_linear_f32", "tpo_wigner_d_f64", "tpo_wigner_d_size", "tpo_rotate_f32",
    "tpo_gaunt_real", "tpo_s2_grid", "tpo_legendre_lambda", "tpo_mtp_path_weight", "tpo_count_muls",
    "tpo_cgtp_num_paths", "tpo_cgtp_weighted_f32", "tpo_set_precision",
]


def check(rc: int) -> int:
    """Map a TPO_* status to the reference's exception types (pybind maps
    std::invalid_argument -> ValueError, proj/README.md:149-152)."""
    if rc == TPO_OK:
        return rc
    msg = lib().tpo_last_error().decode(errors="replace")
    if rc == TPO_EINVAL:
        raise ValueError(msg)
    if rc == TPO_ERANGE:
        raise IndexError(msg)
    raise TpoError(f"status {rc}: {msg}")


class Context:
    """Owns a tpo_ctx bound to one CUDA device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().tpo_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)

    def close(self):
        if getattr(self, "handle", None):
            lib().tpo_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().tpo_ctx_launches(self.handle))

    def set_grid_path(self, path: str) -> None:
        """Kernel selection for the two Gaunt products (tpo_set_gtp_grid_path): "auto", "tc"
        (tcgen05 fused / degree groups), "simt" (separable grid kernel; direct-convolution Fourier),
        "sep" (the separable row-quad kernel for both, Fourier on the folded reference torus)."""
        code = {"auto": 0, "tc": 1, "tcgen05": 1, "simt": 2, "sep": 3}[path]
        r = lib().tpo_set_gtp_grid_path(self.handle, code)
        if r < 0:
            check(-r)

    def set_precision(self, mode: str) -> str:
        """"default" or "strict" accumulation segmentation of the tcgen05 Gaunt products
        (tpo_set_precision); returns the previous mode."""
        code = {"default": 0, "strict": 1}[mode]
        r = lib().tpo_set_precision(self.handle, code)
        if r < 0:
            check(-r)
        return {0: "default", 1: "strict"}[r]

    @property
    def last_grid_path(self) -> str:
        return {0: "none", 1: "tcgen05", 2: "simt", 3: "small", 4: "separable"}[lib().tpo_last_gtp_grid_path(self.handle)]


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    if device is None:
        device = int(os.environ.get("TPO_DEVICE", "0"))
        try:
            import torch

            if torch.cuda.is_available():
                device = torch.cuda.current_device()
        except Exception:
            pass
    with _lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx
