"""C-ABI boundary checks that need no GPU: the library loads, exports every declared symbol, and rejects
invalid arguments before touching the device (include/paradiag.h error contract)."""
import ctypes as C
import os

import pytest

import paper_2005_09158_b200 as pd
from paper_2005_09158_b200 import _lib

LIB = _lib._LIB_PATH


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        pytest.fail("libparadiag.so missing: run __graft_entry__.build()")
    return _lib.load_library()


def test_library_exports_every_declared_symbol(lib):
    decl = _lib.declared_symbols()
    assert len(decl) >= 18
    missing = [n for n, ok in pd.exported_symbols().items() if not ok]
    assert not missing, missing


def _setup(lib, op=0, nx=63, ny=1, length=1.0, dt=1 / 32, nt=32, alpha=1e-2, scheme=0):
    g = _lib.pd_grid(op, nx, ny, length, 0.01, 1.0, 0.0)
    ctx = C.c_void_p()
    st = lib.pd_setup(C.byref(g), dt, nt, alpha, scheme, None, None, C.byref(ctx))
    return st, ctx


@pytest.mark.parametrize("kw,needle", [
    (dict(alpha=0.0), "alpha"), (dict(alpha=1.5), "alpha"), (dict(alpha=-1e-3), "alpha"),
    (dict(nt=48), "power of two"), (dict(nt=0), "power of two"), (dict(dt=0.0), "dt"),
    (dict(scheme=7), "scheme"), (dict(scheme=2, nt=2), "leapfrog"), (dict(op=9), "operator"),
    (dict(op=2, nx=100, ny=100), "power of two"), (dict(op=2, nx=64, ny=32), "N x N"), (dict(nx=0), "nx"),
])
def test_setup_rejects_invalid_arguments(lib, kw, needle):
    st, ctx = _setup(lib, **kw)
    assert st == -1  # PD_EINVAL
    assert not ctx.value
    assert needle in lib.pd_last_error(None).decode()


def test_null_pointers_rejected(lib):
    assert lib.pd_apply_precond(None, None, None) == -1
    assert lib.pd_local_size(None) == -1


def test_host_buffer_checks():
    """The *_host entry points copy Nt * S doubles from / to host memory the library cannot bound-check: the binding
    refuses anything but a contiguous CPU float64 tensor of exactly that many elements."""
    import torch
    ok = torch.zeros(4, 8, dtype=torch.float64)
    assert _lib._hptr(ok, 32, "x").value == ok.data_ptr()
    assert _lib._hptr(None, 32, "x") is None
    with pytest.raises(TypeError):
        _lib._hptr(ok.float(), 32, "x")                 # float32
    with pytest.raises(TypeError):
        _lib._hptr(ok.t(), 32, "x")                     # non-contiguous view
    with pytest.raises(ValueError):
        _lib._hptr(ok[:3], 32, "x")                     # f with Nt rows instead of Nt + 1, etc.
    with pytest.raises(TypeError):
        _lib._hptr(ok.numpy(), 32, "x")                 # not a tensor
