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


def _prep(x, y, L1, L2, kind, L3, out=None):
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
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=x.device)
    else:  # caller's buffer: must be exactly the output on the inputs' device
        if not isinstance(out, torch.Tensor) or tuple(out.shape) != shape or out.dtype != torch.float32 \
                or not out.is_contiguous():
            raise ValueError("out has the wrong shape/dtype or is not contiguous")
        if out.device != x.device:
            raise ValueError("out must be on the inputs' device")
    stream = torch.cuda.current_stream(x.device).cuda_stream
    return x, y, out, B, C, y_shared, stream


def run(kind: str, x, y, L1: int, L2: int, L3: int = 0, l_tilde: int = -1, out=None):
    """Generic batched dispatch through tpo_run_f32."""
    x, y, o, B, C, ys, stream = _prep(x, y, L1, L2, kind, L3, out)
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
        # the C ABI copies batch x channels rows through raw pointers: every extent must match
        d1, d2 = tower_dim(L1), tower_dim(L2)
        if x.dim() not in (2, 3) or x.shape[-1] != d1:
            raise ValueError(f"run_host_batch: x must be [B, {d1}] or [B, C, {d1}]")
        B = x.shape[0]
        Cn = x.shape[1] if x.dim() == 3 else 1
        ys = 1 if (x.dim() == 3 and y.dim() == 2) else 0
        if ys:
            if tuple(y.shape) != (B, d2):
                raise ValueError(f"run_host_batch: shared y must be [{B}, {d2}]")
        elif tuple(y.shape) != tuple(x.shape[:-1]) + (d2,):
            raise ValueError(f"run_host_batch: y must be {tuple(x.shape[:-1]) + (d2,)}")
        dout = out_dim(kind, L1, L2, L3)
        if out.numel() != B * Cn * dout:
            raise ValueError(f"run_host_batch: out must hold {B} x {Cn} x {dout} floats")
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


# ---------------------------------------------------------------- stage operators (device, batched)
def _dev_check(*ts):
    import torch

    for t in ts:
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError("inputs must be CUDA tensors (no CPU path)")
        if t.device != ts[0].device:
            raise ValueError("all tensors must be on the same device")


def _f32(t):
    import torch

    if t.dtype != torch.float32:
        raise ValueError("tensors must be float32")
    return t.contiguous()


def _ints(v):
    import ctypes as C

    v = [int(a) for a in v]
    return (C.c_int * max(1, len(v)))(*v), len(v)


def _stream(t):
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


def to_sphere(x, L: int, grid_L: int):
    """Batched tpo::to_sphere on make_grid(grid_L) (proj/src/sphere.cpp:105-134): x [B, (L+1)^2]
    -> F [B, grid_L+1, 2 grid_L+1]."""
    import torch

    _dev_check(x)
    x = _f32(x)
    if x.dim() != 2 or x.shape[1] != tower_dim(L):
        raise ValueError(f"x must be [B, {tower_dim(L)}]")
    F = torch.empty((x.shape[0], grid_L + 1, 2 * grid_L + 1), device=x.device)
    check(lib().tpo_to_sphere_f32(context(x.device.index).handle, L, grid_L, x.data_ptr(), F.data_ptr(), x.shape[0],
                                  _stream(x)))
    return F


def from_sphere(F, grid_L: int, degrees):
    """Batched tpo::detail::from_sphere_select (proj/src/sphere.cpp:155-195): F [B, nt, np] ->
    [B, sum(2l+1)] over `degrees` in the given order."""
    import torch

    _dev_check(F)
    F = _f32(F)
    if F.dim() != 3 or tuple(F.shape[1:]) != (grid_L + 1, 2 * grid_L + 1):
        raise ValueError("F must be [B, grid_L+1, 2 grid_L+1]")
    d, n = _ints(degrees)
    out = torch.empty((F.shape[0], sum(2 * l + 1 for l in degrees)), device=F.device)
    check(lib().tpo_from_sphere_f32(context(F.device.index).handle, grid_L, d, n, F.data_ptr(), out.data_ptr(),
                                    F.shape[0], _stream(F)))
    return out


def pointwise_mul(a, b):
    """tpo::pointwise_mul on sphere samples (proj/src/sphere.cpp:145-151)."""
    import torch

    _dev_check(a, b)
    a, b = _f32(a), _f32(b)
    if a.shape != b.shape:
        raise ValueError("pointwise_mul: signals live on different grids")
    out = torch.empty_like(a)
    check(lib().tpo_pointwise_mul_f32(context(a.device.index).handle, a.data_ptr(), b.data_ptr(), out.data_ptr(),
                                      a.numel(), _stream(a)))
    return out


def mtp_embed(x, L: int, l_tilde: int):
    """Batched tpo::mtp_embed (proj/src/mtp.cpp:47-58): x [B, (L+1)^2] -> X [B, dt, dt]."""
    import torch

    _dev_check(x)
    x = _f32(x)
    if x.dim() != 2 or x.shape[1] != tower_dim(L):
        raise ValueError(f"x must be [B, {tower_dim(L)}]")
    dt = 2 * l_tilde + 1
    X = torch.empty((x.shape[0], dt, dt), device=x.device)
    check(lib().tpo_mtp_embed_f32(context(x.device.index).handle, L, l_tilde, x.data_ptr(), X.data_ptr(), x.shape[0],
                                  _stream(x)))
    return X


def mtp_matmul(X, Y):
    """Batched tpo::mtp_matmul (proj/src/mtp.cpp:119-133): Z[b] = X[b] Y[b]."""
    import torch

    _dev_check(X, Y)
    X, Y = _f32(X), _f32(Y)
    if X.dim() != 3 or X.shape != Y.shape or X.shape[1] != X.shape[2]:
        raise ValueError("mtp_matmul: carriers do not match")
    Z = torch.empty_like(X)
    check(lib().tpo_mtp_matmul_f32(context(X.device.index).handle, X.shape[1], X.data_ptr(), Y.data_ptr(),
                                   Z.data_ptr(), X.shape[0], _stream(X)))
    return Z


def mtp_extract(Z, l_tilde: int, degrees):
    """Batched tpo::mtp_extract_select (proj/src/mtp.cpp:60-97): Z [B, dt, dt] -> [B, sum(2l+1)]."""
    import torch

    _dev_check(Z)
    Z = _f32(Z)
    dt = 2 * l_tilde + 1
    if Z.dim() != 3 or tuple(Z.shape[1:]) != (dt, dt):
        raise ValueError("mtp_extract: matrix does not match the carrier degree")
    d, n = _ints(degrees)
    out = torch.empty((Z.shape[0], sum(2 * l + 1 for l in degrees)), device=Z.device)
    check(lib().tpo_mtp_extract_f32(context(Z.device.index).handle, l_tilde, d, n, Z.data_ptr(), out.data_ptr(),
                                    Z.shape[0], _stream(Z)))
    return out


def linear_gtp(x, y, L1: int, L2: int, L3: int, wx, wy, wout):
    """Schur-consistent linear layers around the grid GTP, fused:
    apply_linear(gtp(apply_linear(x, wx), apply_linear(y, wy)), wout) for tower -> tower layers
    (one copy per degree).  Such a layer connects only equal degrees, one weight per degree
    (proj/src/irreps.cpp:95-104), so it is a per-degree scaling and the whole composition is
    weighted_gtp: one launch of the tcgen05 kernel with the weights folded into its input
    conversion and epilogue.  wx, wy, wout: LinearLayer weight vectors of lengths L1+1, L2+1, L3+1
    (linear_connections order)."""
    import numpy as np

    wx, wy, wout = (np.asarray(w, dtype=np.float64) for w in (wx, wy, wout))
    if len(wx) != L1 + 1 or len(wy) != L2 + 1 or len(wout) != L3 + 1:
        raise ValueError("linear_gtp: tower layers take one weight per degree (L+1 each)")
    return weighted_gtp(x, y, wx, wy, wout, L1, L2, L3)


def linear_connections(in_irreps, out_irreps):
    """LinearLayer connections (proj/src/irreps.cpp:95-104): one weight per (input copy, output
    copy) of equal degree, in (input entry, input copy, output entry, output copy) order.  irreps are
    [(mul, l), ...] lists."""
    return [(ei, ci, eo, co) for ei, (mi, li) in enumerate(in_irreps) for ci in range(mi)
            for eo, (mo, lo) in enumerate(out_irreps) if lo == li for co in range(mo)]


def apply_linear(x, in_irreps, out_irreps, weights):
    """Batched tpo::apply_linear (proj/src/irreps.cpp:119-129): the Schur-consistent equivariant
    linear map, x [B, dim(in)] -> [B, dim(out)]."""
    import ctypes as C

    import numpy as np
    import torch

    _dev_check(x)
    x = _f32(x)
    in_mul, n_in = _ints([m for m, _ in in_irreps])
    in_l, _ = _ints([l for _, l in in_irreps])
    out_mul, n_out = _ints([m for m, _ in out_irreps])
    out_l, _ = _ints([l for _, l in out_irreps])
    din = sum(m * (2 * l + 1) for m, l in in_irreps)
    dout = sum(m * (2 * l + 1) for m, l in out_irreps)
    if x.dim() != 2 or x.shape[1] != din:
        raise ValueError("linear layer: input descriptor mismatch")
    w = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
    out = torch.empty((x.shape[0], dout), device=x.device)
    check(lib().tpo_apply_linear_f32(context(x.device.index).handle, in_mul, in_l, n_in, out_mul, out_l, n_out,
                                     w.ctypes.data_as(C.c_void_p), len(w), x.data_ptr(), out.data_ptr(), x.shape[0],
                                     _stream(x)))
    return out


def wigner_d(R, L: int):
    """Real Wigner-D blocks D^0..D^L of a batch of rotations (proj/src/wigner.cpp:288-312) on the
    device, fp64: R [n, 3, 3] -> list of [n, 2l+1, 2l+1]."""
    import torch

    _dev_check(R)
    R = R.to(torch.float64).contiguous()
    n = R.shape[0]
    D = torch.empty((n, int(lib().tpo_wigner_d_size(L))), dtype=torch.float64, device=R.device)
    check(lib().tpo_wigner_d_f64(context(R.device.index).handle, L, R.data_ptr(), D.data_ptr(), n, _stream(R)))
    blocks, off = [], 0
    for l in range(L + 1):
        d = 2 * l + 1
        blocks.append(D[:, off:off + d * d].reshape(n, d, d))
        off += d * d
    return blocks


def rotate(x, R, L: int):
    """Batched tpo::rotate (proj/src/wigner.cpp:314-325): x [B, (L+1)^2] or [B, C, (L+1)^2];
    R [n_rot, 3, 3] with sample b rotated by R[b * n_rot // B]."""
    import torch

    _dev_check(x, R)
    x = _f32(x)
    R = R.to(torch.float64).contiguous()
    B = x.shape[0]
    C = x.shape[1] if x.dim() == 3 else 1
    if x.shape[-1] != tower_dim(L):
        raise ValueError(f"x must end in {tower_dim(L)} components")
    out = torch.empty_like(x)
    check(lib().tpo_rotate_f32(context(x.device.index).handle, L, R.data_ptr(), R.shape[0], x.data_ptr(),
                               out.data_ptr(), B, C, _stream(x)))
    return out


__all__ += ["to_sphere", "from_sphere", "pointwise_mul", "mtp_embed", "mtp_matmul", "mtp_extract", "apply_linear",
            "linear_connections", "wigner_d", "rotate"]


def cgtp_num_paths(L1: int, L2: int) -> int:
    """Number of (l1, l2, l3) paths of cgtp(L1, L2), the reference's order (proj/src/cgtp.cpp:152-163)."""
    return int(lib().tpo_cgtp_num_paths(L1, L2))


def cgtp_weighted(x, y, w, L1: int, L2: int, out=None):
    """Per-path weighted CGTP (MACE "uvu"): path p of sample b scaled by w[b, p] (w [B, n_paths], per
    edge) or w[p] (w [n_paths], shared).  Fused into the shared-y edge kernel (C4 shape)."""
    import torch

    x, y, o, B, C, ys, stream = _prep(x, y, L1, L2, "cgtp", 0, out)
    npth = cgtp_num_paths(L1, L2)
    if not isinstance(w, torch.Tensor) or w.device != x.device or w.dtype != torch.float32:
        raise ValueError("w must be a float32 tensor on the inputs' device")
    if tuple(w.shape) == (B, npth):
        per_edge = 1
    elif tuple(w.shape) == (npth,):
        per_edge = 0
    else:
        raise ValueError(f"w must be [{B}, {npth}] or [{npth}]")
    w = w.contiguous()
    check(lib().tpo_cgtp_weighted_f32(context(x.device.index).handle, L1, L2, w.data_ptr(), per_edge, x.data_ptr(),
                                      y.data_ptr(), o.data_ptr(), B, C, ys, stream))
    return o


__all__ += ["cgtp_num_paths", "cgtp_weighted"]
