"""B200-native SO(3) tensor-product operations (CGTP, S2-grid GTP,
Fourier GTP, MTP) behind the reference so3tpo operator API.

Batched device API (torch tensors on an sm_100 device, fp32, contiguous):

    out = cgtp(x, y, L1, L2)                       # tpo::cgtp_mimo
    out = gtp_grid(x, y, L1, L2, L3)               # tpo::gtp_grid
    out = gtp_fourier(x, y, L1, L2, L3)            # tpo::gtp_fourier
    out = mtp(x, y, L1, L2, L3, l_tilde=-1)        # tpo::mtp
    out = weighted_gtp(x, y, a, b, c, L1, L2, L3)  # tpo::weighted_gtp
    gx, gy = backward(kind, x, y, grad_out, L1, L2, L3)  # vector-Jacobian products
    out = product(kind, x, y, L1, L2, L3)          # autograd-aware (torch.autograd.Function)

x is [B, Din1] or [B, C, Din1]; y is [B, Din2] (shared across the C
channels when x has a channel axis) or [B, C, Din2].  Results are
[B, (C,) Dout].  Every call goes through the C ABI of libtpo_b200.so on
torch's current CUDA stream; nothing falls back to the CPU.

The one-product-per-call, irreps-string API of the reference's Python
module lives in :mod:`paper_2506_13523_b200.so3tpo`.
"""
from __future__ import annotations

from ._lib import KINDS, Context, HostRequest, TpoError, check, context, lib

__all__ = [
    "cgtp", "gtp_grid", "gtp_fourier", "mtp", "weighted_gtp", "run", "out_dim", "tower_dim",
    "mtp_l_tilde", "backward", "product", "Context", "TpoError", "context", "lib", "KINDS",
]


def tower_dim(L: int) -> int:
    return (L + 1) * (L + 1)


def out_dim(kind: str, L1: int, L2: int, L3: int = 0) -> int:
    r = int(lib().tpo_out_dim(KINDS[kind], L1, L2, L3))
    if r < 0:
        check(-r)
    return r


def mtp_l_tilde(L1: int, L2: int, L3: int) -> int:
    return int(lib().tpo_mtp_l_tilde(L1, L2, L3))


def _prep(x, y, L1, L2, kind, L3):
    import torch

    if not (isinstance(x, torch.Tensor) and isinstance(y, torch.Tensor)):
        raise TypeError("x and y must be torch tensors")
    if not x.is_cuda or not y.is_cuda:
        raise ValueError("inputs must live on a CUDA device (no CPU path)")
    if x.dtype != torch.float32 or y.dtype != torch.float32:
        raise ValueError("inputs must be float32")
    d1, d2 = tower_dim(L1), tower_dim(L2)
    if x.dim() == 2:
        B, C = x.shape[0], 1
        if x.shape[1] != d1:
            raise ValueError(f"x has {x.shape[1]} components, irreps dim is {d1}")
        if tuple(y.shape) != (B, d2):
            raise ValueError(f"y must be [{B}, {d2}]")
        y_shared = 0
    elif x.dim() == 3:
        B, C = x.shape[0], x.shape[1]
        if x.shape[2] != d1:
            raise ValueError(f"x has {x.shape[2]} components, irreps dim is {d1}")
        if tuple(y.shape) == (B, d2):
            y_shared = 1
        elif tuple(y.shape) == (B, C, d2):
            y_shared = 0
        else:
            raise ValueError(f"y must be [{B}, {d2}] or [{B}, {C}, {d2}]")
    else:
        raise ValueError("x must be [B, Din] or [B, C, Din]")
    if y.device != x.device:
        raise ValueError("x and y must be on the same device")
    x = x.contiguous()
    y = y.contiguous()
    dout = out_dim(kind, L1, L2, L3)
    shape = (B, dout) if x.dim() == 2 else (B, C, dout)
    out = torch.empty(shape, dtype=torch.float32, device=x.device)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    return x, y, out, B, C, y_shared, stream


def run(kind: str, x, y, L1: int, L2: int, L3: int = 0, l_tilde: int = -1, out=None):
    """Generic batched dispatch through tpo_run_f32."""
    x, y, o, B, C, ys, stream = _prep(x, y, L1, L2, kind, L3)
    if out is not None:
        if out.shape != o.shape or out.dtype != o.dtype or not out.is_contiguous():
            raise ValueError("out has the wrong shape/dtype or is not contiguous")
        o = out
    ctx = context(x.device.index)
    check(lib().tpo_run_f32(ctx.handle, KINDS[kind], L1, L2, L3, l_tilde, x.data_ptr(), y.data_ptr(),
                            o.data_ptr(), B, C, ys, stream))
    return o


def run_host_batch(requests, device: int = 0):
    """Several independent products with HOST tensors in one synchronous call
    (tpo_run_host_batch_f32): each request is (kind, x, y, out, L1, L2, L3[, l_tilde])
    with contiguous fp32 CPU tensors (pinned for full copy/compute overlap), x
    [B, Din] or [B, C, Din], y [B, Din2] (shared per b when x has channels) or like x,
    out preallocated.  Results equal one tpo_run_host_f32 call per request."""
    import ctypes as C

    import torch

    reqs = (HostRequest * len(requests))()
    keep = []
    for i, r in enumerate(requests):
        kind, x, y, out, L1, L2, L3 = r[:7]
        lt = r[7] if len(r) > 7 else -1
        for t in (x, y, out):
            if t.device.type != "cpu" or not t.is_contiguous() or t.dtype != torch.float32:
                raise ValueError("run_host_batch: host tensors must be contiguous fp32 on the CPU")
        B = x.shape[0]
        Cn = x.shape[1] if x.dim() == 3 else 1
        ys = 1 if (x.dim() == 3 and y.dim() == 2) else 0
        q = reqs[i]
        q.kind, q.L1, q.L2, q.L3, q.l_tilde, q.y_shared = KINDS[kind], L1, L2, L3, lt, ys
        q.batch, q.channels = B, Cn
        q.x, q.y, q.out = x.data_ptr(), y.data_ptr(), out.data_ptr()
        keep.append((x, y, out))
    check(lib().tpo_run_host_batch_f32(context(device).handle, C.cast(reqs, C.c_void_p), len(requests)))
    return [k[2] for k in keep]


def cgtp(x, y, L1: int, L2: int, out=None):
    """Batched tpo::cgtp_mimo (proj/src/cgtp.cpp:145-177); output layout is
    the reference's path order (l1, l2, l3 ascending)."""
    return run("cgtp", x, y, L1, L2, 0, -1, out)


def gtp_grid(x, y, L1: int, L2: int, L3: int, out=None):
    """Batched tpo::gtp_grid (proj/src/gtp.cpp:197-204, 228-260)."""
    return run("gtp_grid", x, y, L1, L2, L3, -1, out)


def gtp_fourier(x, y, L1: int, L2: int, L3: int, out=None):
    """Batched tpo::gtp_fourier (proj/src/gtp.cpp:217-224, 262-327)."""
    return run("gtp_fourier", x, y, L1, L2, L3, -1, out)


def mtp(x, y, L1: int, L2: int, L3: int, l_tilde: int = -1, out=None):
    """Batched tpo::mtp (proj/src/mtp.cpp:99-117)."""
    return run("mtp", x, y, L1, L2, L3, l_tilde, out)


def weighted_gtp(x, y, a, b, c, L1: int, L2: int, L3: int):
    """Batched tpo::weighted_gtp: c (.) gtp(a (.) x, b (.) y) with per-degree
    weights (proj/src/gtp.cpp:206-215)."""
    import ctypes as C

    import numpy as np

    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    if len(c) != L3 + 1:
        raise ValueError("weighted_gtp: c must have L3+1 entries")
    if len(a) < L1 + 1 or len(b) < L2 + 1:
        raise ValueError("weighted_gtp: weight vector shorter than input degrees")
    x, y, o, B, Cc, ys, stream = _prep(x, y, L1, L2, "gtp_grid", L3)
    ctx = context(x.device.index)
    ptr = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
    check(lib().tpo_weighted_gtp_f32(ctx.handle, L1, L2, L3, ptr(a), ptr(b), ptr(c), x.data_ptr(),
                                     y.data_ptr(), o.data_ptr(), B, Cc, ys, stream))
    return o


def backward(kind: str, x, y, grad_out, L1: int, L2: int, L3: int = 0, l_tilde: int = -1,
             need_x: bool = True, need_y: bool = True):
    """Vector-Jacobian products of a product (tpo_backward_f32): returns
    (grad_x, grad_y), each None when not requested.  grad_out has the forward
    output's shape.  With a shared y ([B, Din2] beside x [B, C, Din1]) only
    grad_x is available."""
    import torch

    x, y, o, B, C, ys, stream = _prep(x, y, L1, L2, kind, L3)
    if not isinstance(grad_out, torch.Tensor) or grad_out.shape != o.shape or grad_out.dtype != torch.float32:
        raise ValueError(f"grad_out must be a float32 tensor of shape {tuple(o.shape)}")
    if grad_out.device != x.device:
        raise ValueError("grad_out must be on the inputs' device")
    if ys and need_y:
        raise ValueError("backward: grad_y with a shared y is not supported")
    g = grad_out.contiguous()
    gx = torch.empty_like(x) if need_x else None
    gy = torch.empty_like(y) if need_y else None
    ctx = context(x.device.index)
    check(lib().tpo_backward_f32(ctx.handle, KINDS[kind], L1, L2, L3, l_tilde, x.data_ptr(), y.data_ptr(),
                                 g.data_ptr(), gx.data_ptr() if gx is not None else None,
                                 gy.data_ptr() if gy is not None else None, B, C, ys, stream))
    return gx, gy


_Fn = None


def _autograd_fn():
    global _Fn
    if _Fn is None:
        import torch

        class TensorProductFn(torch.autograd.Function):
            @staticmethod
            def forward(ctx, x, y, kind, L1, L2, L3, l_tilde):
                ctx.save_for_backward(x, y)
                ctx.cfg = (kind, L1, L2, L3, l_tilde)
                return run(kind, x, y, L1, L2, L3, l_tilde)

            @staticmethod
            def backward(ctx, g):
                x, y = ctx.saved_tensors
                kind, L1, L2, L3, l_tilde = ctx.cfg
                gx, gy = backward(kind, x, y, g, L1, L2, L3, l_tilde, ctx.needs_input_grad[0],
                                  ctx.needs_input_grad[1])
                return gx, gy, None, None, None, None, None

        _Fn = TensorProductFn
    return _Fn


def product(kind: str, x, y, L1: int, L2: int, L3: int = 0, l_tilde: int = -1):
    """Differentiable product (torch.autograd): the forward kernel of ``kind``
    and tpo_backward_f32 for the gradients."""
    return _autograd_fn().apply(x, y, kind, L1, L2, L3, l_tilde)
