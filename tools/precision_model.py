#!/usr/bin/env python
"""Numerical model of the 3xFP16 tcgen05 grid GTP (test/analysis tool, not product code).

Reproduces the fused kernel's arithmetic in numpy on the dense operators of the
S2-grid GTP (built from the fp64 oracle's to_sphere / from_sphere, i.e.
proj/src/sphere.cpp:105-195):

  * inputs scaled by exact powers of two and split into fp16 hi + lo,
  * GEMM 1 / GEMM 2 as three fp16 products (hi*hi + hi*lo + lo*hi) per K-step of 16,
  * the accumulator rounded to fp32 once per MMA instruction, either to nearest
    ("rn") or toward zero ("rz"),
  * GEMM 2 optionally cut into accumulation segments whose partial sums are added
    in fp32 round-to-nearest (the kernel's `seg_chunks`).

On B200 the measured normwise error at L = 12 (1.0385e-5 over a 4096-row sample)
matches the "rz" model (1.04e-5) and not "rn" (1.0e-6): the tensor pipe truncates
its fp32 accumulator once per MMA, so the error grows with the number of MMAs that
accumulate into one TMEM column.  Usage:

    python tools/precision_model.py 10 12      # per L: rn / rz / rz with 2, 3, 4 segments
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import oracle as orc  # noqa: E402  (analysis tool: the oracle builds the reference operators)


def operators(L):
    band = 2 * L
    ls = list(range(L + 1))
    din, dout = (L + 1) ** 2, (2 * L + 1) ** 2
    nth, nph = band + 1, 2 * band + 1
    G = nth * nph
    S = np.zeros((G, din))
    for k in range(din):
        e = np.zeros(din); e[k] = 1
        S[:, k] = orc.to_sphere(ls, e, band).ravel()
    A = np.zeros((dout, G))
    for g in range(G):
        F = np.zeros(G); F[g] = 1
        A[:, g] = orc.from_sphere(F.reshape(nth, nph), band, list(range(2 * L + 1)))
    return S, A


def split(v):
    h = v.astype(np.float16).astype(np.float64)
    return h, (v - h).astype(np.float16).astype(np.float64)


def f32(v, mode):
    f = v.astype(np.float32)
    if mode == "rz":
        over = np.abs(f.astype(np.float64)) > np.abs(v)
        f = np.where(over, np.nextafter(f, np.float32(0)), f)
    return f.astype(np.float64)


def mma3(a, b, mode, segs=1):
    """sum_k a[:, k] b[:, k] as the kernel's 3xFP16 MMA chain (K-steps of 16)."""
    ah, al = split(a); bh, bl = split(b)
    nk = (a.shape[1] + 15) // 16
    bounds = np.linspace(0, nk, segs + 1).astype(int)
    total = np.zeros((a.shape[0], b.shape[0]))
    for s in range(segs):
        D = np.zeros_like(total)
        for kk in range(bounds[s], bounds[s + 1]):
            sl = slice(16 * kk, 16 * kk + 16)
            for p, q in ((ah, bh), (ah, bl), (al, bh)):
                D = f32(D + p[:, sl] @ q[:, sl].T, mode)
        total = f32(total + D, "rn")
    return total


def model_error(L, mode="rz", segs=1, n=512, seed=5):
    S, A = operators(L)
    rng = np.random.default_rng(seed)
    din = S.shape[1]
    x = rng.standard_normal((n, din)).astype(np.float32).astype(np.float64)
    y = rng.standard_normal((n, din)).astype(np.float32).astype(np.float64)
    ref = ((x @ S.T) * (y @ S.T)) @ A.T

    def rowscale(v):
        e = np.floor(np.log2(np.abs(v).max(1))) + 1 + np.ceil(np.log2(din) / 2)
        return v * 2.0 ** (-e[:, None]), e

    xs, ex = rowscale(x); ys, ey = rowscale(y)
    ash = -(np.floor(np.log2(np.abs(A).max())) + 1)
    Fx = f32(mma3(xs, S, mode), "rn"); Fy = f32(mma3(ys, S, mode), "rn")
    P = f32(Fx * Fy, "rn")
    Z = mma3(P, A * 2.0 ** ash, mode, segs)
    out = Z * 2.0 ** (ex + ey - ash)[:, None]
    return float((np.abs(out - ref).max(1) / np.abs(ref).max(1)).max())


if __name__ == "__main__":
    for L in [int(a) for a in sys.argv[1:]] or [10, 12]:
        row = {"rn": model_error(L, "rn"), "rz": model_error(L, "rz")}
        for s in (2, 3, 4):
            row[f"rz_seg{s}"] = model_error(L, "rz", s)
        print(L, {k: f"{v:.2e}" for k, v in row.items()}, flush=True)
