"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/tpo_capi.h declares, and validates arguments / reports errors
without touching a device (no compute calls here)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "tpo_capi.h").read_text()
    return sorted(set(re.findall(r"\b(tpo_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    import paper_2506_13523_b200._lib as L

    lib = ctypes.CDLL(str(L.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(L.EXPORTED)


def test_shapes_without_gpu():
    import paper_2506_13523_b200 as tpo

    assert tpo.out_dim("cgtp", 2, 2) == 81 and tpo.out_dim("cgtp", 3, 3) == 256
    assert tpo.out_dim("gtp_grid", 3, 3, 6) == 49
    assert tpo.out_dim("mtp", 6, 6, 12) == 169
    assert tpo.mtp_l_tilde(4, 4, 8) == 4 and tpo.mtp_l_tilde(2, 1, 3) == 2
    with pytest.raises(ValueError):
        tpo.out_dim("gtp_grid", 2, 2, -1)
    with pytest.raises(ValueError):
        tpo.out_dim("cgtp", -1, 2)


def test_no_silent_cpu_path():
    """Without a usable sm_100 device, context creation fails loudly."""
    import torch

    import paper_2506_13523_b200 as tpo

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises((tpo.TpoError, ValueError)):
        tpo.Context(0)
    x = torch.zeros((2, 9)); y = torch.zeros((2, 9))
    with pytest.raises(ValueError):
        tpo.gtp_grid(x, y, 2, 2, 4)  # CPU tensors are rejected, never computed on host
    with pytest.raises(ValueError):  # the backward too
        tpo.backward("gtp_grid", x, y, torch.zeros((2, 25)), 2, 2, 4)


def test_backward_abi_argument_errors():
    """tpo_backward_f32 validates before touching a device: null context / bad
    kind / shared-y grad_y map to TPO_EINVAL with a message."""
    import ctypes

    import paper_2506_13523_b200 as tpo

    L = tpo.lib()
    rc = L.tpo_backward_f32(None, 1, 2, 2, 4, -1, None, None, None, None, None, 0, 1, 0, None)
    assert rc == 1 and b"null context" in L.tpo_last_error()
    fake = ctypes.c_void_p(1)  # never dereferenced: the argument checks run first
    buf = (ctypes.c_float * 64)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    rc = L.tpo_backward_f32(fake, 1, 2, 2, 4, -1, p, p, p, p, p, 1, 2, 1, None)
    assert rc == 1 and b"shared y" in L.tpo_last_error()


def test_context_first_call_does_not_deadlock():
    """context() before any other library call must not self-deadlock on the
    loader lock (regression: non-reentrant lock in _lib.context -> lib())."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2506_13523_b200 as t\n"
            "try:\n    t.context(0)\nexcept Exception as e:\n    print(type(e).__name__)\n"
            "print('done')" % str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert "done" in r.stdout, r.stderr
