"""ctypes binding of libparadiag.so (include/paradiag.h).  Marshalling only."""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libparadiag.so")
_HEADER = os.path.join(os.path.dirname(_HERE), "include", "paradiag.h")

ADE1D_DIRICHLET, WAVE1D_DIRICHLET, ADE2D_PERIODIC, WAVE2D_DIRICHLET = 0, 1, 2, 3
BE, CN, LEAPFROG = 0, 1, 2
PD_OK, PD_NOT_CONVERGED = 0, 1
SOLVE_ZERO_GUESS = 16  # include/paradiag.h PD_SOLVE_ZERO_GUESS
_STATUS = {0: "PD_OK", 1: "PD_NOT_CONVERGED", -1: "PD_EINVAL", -2: "PD_ESINGULAR", -3: "PD_ECUDA",
           -4: "PD_ENCCL", -5: "PD_ENOMEM", -6: "PD_EBREAKDOWN"}


class ParaDiagError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class pd_grid(C.Structure):
    _fields_ = [("op", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("length", C.c_double),
                ("nu", C.c_double), ("ax", C.c_double), ("ay", C.c_double)]


class pd_dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("size", C.c_int), ("nccl_id", C.c_void_p), ("nccl_comm", C.c_void_p)]


class pd_report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("rel_residual", C.c_double),
                ("wall_ms", C.c_double), ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int),
                ("history_len", C.c_int)]


@dataclasses.dataclass
class Report:
    status: int
    iterations: int
    converged: bool
    rel_residual: float
    wall_ms: float
    history: list


_lib = None


def load_library(path: str | None = None):
    """Load libparadiag.so (built in-tree by __graft_entry__.build()).  Raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or _LIB_PATH
    if not os.path.exists(p):
        raise ImportError(f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(p)
    vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.c_int
    sig = {
        "pd_setup": (ip, [C.POINTER(pd_grid), C.c_double, ip, C.c_double, ip, C.POINTER(pd_dist), vp, C.POINTER(vp)]),
        "pd_destroy": (None, [vp]),
        "pd_last_error": (C.c_char_p, [vp]),
        "pd_nccl_unique_id": (ip, [vp]),
        "pd_local_shape": (ip, [vp, C.POINTER(ip), C.POINTER(ip), C.POINTER(C.c_longlong)]),
        "pd_local_size": (C.c_longlong, [vp]),
        "pd_spectra": (ip, [vp, dp, dp]),
        "pd_apply_precond": (ip, [vp, vp, vp]),
        "pd_residual": (ip, [vp, vp, vp, vp, dp]),
        "pd_matvec": (ip, [vp, vp, vp]),
        "pd_build_rhs": (ip, [vp, vp, vp, vp, vp]),
        "pd_solve_stationary": (ip, [vp, vp, vp, C.c_double, ip, C.POINTER(pd_report)]),
        "pd_solve_gmres": (ip, [vp, vp, vp, C.c_double, ip, ip, C.POINTER(pd_report)]),
        "pd_tail_map": (ip, [vp, vp, vp]),
        "pd_solve_stationary_tail": (ip, [vp, vp, vp, C.c_double, ip, C.POINTER(pd_report)]),
        "pd_solve_gmres_tail": (ip, [vp, vp, vp, C.c_double, ip, ip, C.POINTER(pd_report)]),
        "pd_set_reaction": (ip, [vp, C.c_double, C.c_double]),
        "pd_solve_newton": (ip, [vp, vp, vp, C.c_double, ip, C.POINTER(pd_report)]),
        "pd_solve_ivp_host": (ip, [vp, ip, vp, vp, vp, vp, C.c_double, ip, ip, C.POINTER(pd_report)]),
        "pd_apply_precond_host": (ip, [vp, vp, vp]),
        "pd_solve_host": (ip, [vp, ip, vp, vp, C.c_double, ip, ip, C.POINTER(pd_report)]),
        "pd_solve": (ip, [vp, ip, vp, vp, C.c_double, ip, ip, C.POINTER(pd_report)]),
        "pd_kernel_launches": (C.c_longlong, [vp]),
        "pd_enable_phase_timing": (ip, [vp, ip]),
        "pd_phase_times": (ip, [vp, dp, C.POINTER(C.c_longlong)]),
        "pd_partition": (ip, [ip, ip, ip, ip, ip, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                              C.POINTER(ip), C.POINTER(ip)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def declared_symbols() -> list[str]:
    """Function names declared in include/paradiag.h."""
    with open(_HEADER) as fh:
        return re.findall(r"^PD_API\s+[\w\s\*]+?\b(pd_\w+)\(", fh.read(), flags=re.M)


def exported_symbols(path: str | None = None) -> dict:
    """{name: bool} — whether each declared symbol resolves in the shared library (no GPU needed)."""
    lib = C.CDLL(path or _LIB_PATH)
    out = {}
    for n in declared_symbols():
        try:
            getattr(lib, n)
            out[n] = True
        except AttributeError:
            out[n] = False
    return out


def _check(lib, ctx, st: int, allow=(PD_OK,)):
    if st not in allow:
        msg = lib.pd_last_error(ctx)
        raise ParaDiagError(st, msg.decode() if msg else "")
    return st


def partition(op: int, nx: int, ny: int, nt: int, size: int):
    """Partition plan of the sharded path (pure host): lists s_off, s_cnt, f_off, f_cnt over ranks."""
    lib = load_library()
    so, sc = (C.c_longlong * size)(), (C.c_longlong * size)()
    fo, fc = (C.c_int * size)(), (C.c_int * size)()
    _check(lib, None, lib.pd_partition(op, nx, ny, nt, size, so, sc, fo, fc))
    return list(so), list(sc), list(fo), list(fc)


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    _check(lib, None, lib.pd_nccl_unique_id(buf))
    return buf.raw


def _ptr(t):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError("expected a contiguous CUDA float64 tensor")
    return C.c_void_p(t.data_ptr())


def _hptr(t, numel: int, name: str):
    """HOST buffer of the *_host entry points: a contiguous CPU float64 tensor of exactly `numel` elements (the C side
    copies that many doubles in or out and cannot check host extents).  None passes through (optional inputs)."""
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous CPU float64 tensor (pinned recommended)")
    if t.numel() != numel:
        raise ValueError(f"{name}: expected {numel} elements, got {t.numel()}")
    return C.c_void_p(t.data_ptr())


class ParaDiag:
    """One ParaDiag-II context (pd_ctx) on the current CUDA device and stream.

    op: ADE1D_DIRICHLET | WAVE1D_DIRICHLET | ADE2D_PERIODIC | WAVE2D_DIRICHLET;  scheme: BE | CN | LEAPFROG.
    Vectors are CUDA float64 tensors of shape [Nt, S_local] (S = nx*ny spatial dofs of this rank).
    rank=-1 with size>1 runs `size` virtual ranks of the sharded path on this GPU (global vectors).
    """

    def __init__(self, op: int, nx: int, ny: int, length: float, nu: float, ax: float, ay: float,
                 dt: float, nt: int, alpha: float, scheme: int, stream=None, rank: int = 0, size: int = 1,
                 nccl_id: bytes | None = None, nccl_comm: int | None = None):
        import torch
        self._lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("ParaDiag needs a CUDA device (no CPU fallback)")
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        g = pd_grid(op, nx, ny, length, nu, ax, ay)
        self._idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        d = pd_dist(rank, size, C.cast(self._idbuf, C.c_void_p) if self._idbuf else None,
                    C.c_void_p(nccl_comm) if nccl_comm else None)
        self.rank, self.size = rank, size
        self.scheme = scheme
        ctx = C.c_void_p()
        st = self._lib.pd_setup(C.byref(g), dt, nt, alpha, scheme, C.byref(d),
                                C.c_void_p(self.stream.cuda_stream), C.byref(ctx))
        _check(self._lib, None, st)
        self._ctx = ctx
        self.nt = nt
        nxl, nyl, off = C.c_int(), C.c_int(), C.c_longlong()
        self._lib.pd_local_shape(ctx, C.byref(nxl), C.byref(nyl), C.byref(off))
        self.nx_local, self.ny_local, self.offset = nxl.value, nyl.value, off.value
        self.S = self.nx_local * self.ny_local
        self.shape = (nt, self.S)

    # -- lifecycle
    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.pd_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _new(self):
        import torch
        return torch.empty(self.shape, dtype=torch.float64, device="cuda")

    # -- C ABI mirrors
    def spectra(self):
        import numpy as np
        a = (C.c_double * (2 * self.nt))()
        b = (C.c_double * (2 * self.nt))()
        _check(self._lib, self._ctx, self._lib.pd_spectra(self._ctx, a, b))
        a = np.frombuffer(a, dtype=np.float64)
        b = np.frombuffer(b, dtype=np.float64)
        return a[0::2] + 1j * a[1::2], b[0::2] + 1j * b[1::2]

    def apply_precond(self, r, z=None):
        z = self._new() if z is None else z
        _check(self._lib, self._ctx, self._lib.pd_apply_precond(self._ctx, _ptr(r), _ptr(z)))
        return z

    def residual(self, b, u, r=None, norm: bool = False):
        r = self._new() if r is None else r
        n2 = C.c_double()
        _check(self._lib, self._ctx, self._lib.pd_residual(self._ctx, _ptr(b), _ptr(u), _ptr(r),
                                                           C.byref(n2) if norm else None))
        return (r, n2.value) if norm else r

    def matvec(self, u, w=None):
        w = self._new() if w is None else w
        _check(self._lib, self._ctx, self._lib.pd_matvec(self._ctx, _ptr(u), _ptr(w)))
        return w

    def build_rhs(self, u0, v0=None, f=None, b=None):
        b = self._new() if b is None else b
        _check(self._lib, self._ctx, self._lib.pd_build_rhs(self._ctx, _ptr(u0), _ptr(v0), _ptr(f), _ptr(b)))
        return b

    def _report(self, cap):
        hist = (C.c_double * cap)()
        rep = pd_report(0, 0, 0.0, 0.0, C.cast(hist, C.POINTER(C.c_double)), cap, 0)
        return rep, hist

    @staticmethod
    def _mk(st, rep, hist):
        n = min(rep.history_len, rep.history_cap)
        return Report(st, rep.iterations, bool(rep.converged), rep.rel_residual, rep.wall_ms, list(hist[:n]))

    def solve_stationary(self, b, u=None, tol=1e-10, maxit=100, raise_on_fail=True):
        import torch
        u = torch.zeros(self.shape, dtype=torch.float64, device="cuda") if u is None else u
        rep, hist = self._report(maxit + 2)
        st = self._lib.pd_solve_stationary(self._ctx, _ptr(b), _ptr(u), tol, maxit, C.byref(rep))
        if raise_on_fail:
            _check(self._lib, self._ctx, st, allow=(PD_OK, PD_NOT_CONVERGED))
        return u, self._mk(st, rep, hist)

    def solve_gmres(self, b, u=None, tol=1e-10, m=20, maxit=100, raise_on_fail=True, zero_guess=False):
        """zero_guess: start from u = 0 with u output only (pd_solve with PD_SOLVE_ZERO_GUESS; u not read)."""
        import torch
        if u is None:
            u = torch.empty(self.shape, dtype=torch.float64, device="cuda") if zero_guess else \
                torch.zeros(self.shape, dtype=torch.float64, device="cuda")
        rep, hist = self._report(maxit + 2)
        if zero_guess:
            st = self._lib.pd_solve(self._ctx, 1 | SOLVE_ZERO_GUESS, _ptr(b), _ptr(u), tol, m, maxit, C.byref(rep))
        else:
            st = self._lib.pd_solve_gmres(self._ctx, _ptr(b), _ptr(u), tol, m, maxit, C.byref(rep))
        if raise_on_fail:
            _check(self._lib, self._ctx, st, allow=(PD_OK, PD_NOT_CONVERGED))
        return u, self._mk(st, rep, hist)

    # ---- WR tail form (include/paradiag.h; same iterates as the two solvers above) ----
    @property
    def head_blocks(self) -> int:
        return 2 if self.scheme == LEAPFROG else 1

    def tail_map(self, head, tail=None):
        """tail = last H blocks of P^{-1}(E_H head); head, tail: [H, S] device float64."""
        import torch
        tail = torch.empty_like(head) if tail is None else tail
        _check(self._lib, self._ctx, self._lib.pd_tail_map(self._ctx, _ptr(head), _ptr(tail)))
        return tail

    def solve_stationary_tail(self, b, u=None, tol=1e-10, maxit=100, raise_on_fail=True):
        import torch
        u = torch.zeros(self.shape, dtype=torch.float64, device="cuda") if u is None else u
        rep, hist = self._report(maxit + 2)
        st = self._lib.pd_solve_stationary_tail(self._ctx, _ptr(b), _ptr(u), tol, maxit, C.byref(rep))
        if raise_on_fail:
            _check(self._lib, self._ctx, st, allow=(PD_OK, PD_NOT_CONVERGED))
        return u, self._mk(st, rep, hist)

    def solve_gmres_tail(self, b, u=None, tol=1e-10, m=20, maxit=100, raise_on_fail=True):
        import torch
        u = torch.zeros(self.shape, dtype=torch.float64, device="cuda") if u is None else u
        rep, hist = self._report(maxit + 2)
        st = self._lib.pd_solve_gmres_tail(self._ctx, _ptr(b), _ptr(u), tol, m, maxit, C.byref(rep))
        if raise_on_fail:
            _check(self._lib, self._ctx, st, allow=(PD_OK, PD_NOT_CONVERGED))
        return u, self._mk(st, rep, hist)

    # ---- nonlinear (simplified Newton, include/paradiag.h) ----
    def set_reaction(self, g3: float, g1: float):
        _check(self._lib, self._ctx, self._lib.pd_set_reaction(self._ctx, float(g3), float(g1)))

    def solve_newton(self, b, u=None, tol=1e-10, maxit=50, raise_on_fail=True):
        import torch
        u = torch.zeros(self.shape, dtype=torch.float64, device="cuda") if u is None else u
        rep, hist = self._report(maxit + 2)
        st = self._lib.pd_solve_newton(self._ctx, _ptr(b), _ptr(u), tol, maxit, C.byref(rep))
        if raise_on_fail:
            _check(self._lib, self._ctx, st, allow=(PD_OK, PD_NOT_CONVERGED))
        return u, self._mk(st, rep, hist)

    def apply_precond_host(self, r_host, z_host):
        """r_host, z_host: contiguous CPU float64 tensors (pinned recommended) of shape [Nt, S]."""
        n = self.nt * self.S
        _check(self._lib, self._ctx, self._lib.pd_apply_precond_host(
            self._ctx, _hptr(r_host, n, "r_host"), _hptr(z_host, n, "z_host")))
        return z_host

    def solve_ivp_host(self, solver: int, u0_host, u_host, v0_host=None, f_host=None, tol=1e-10, m=20, maxit=100):
        """End to end from HOST initial data (pinned CPU float64 tensors); u_host [Nt, S] receives the solution.
        solver: 0 stationary, 1 GMRES, 2 / 3 their tail forms, 4 simplified Newton."""
        rep, hist = self._report(maxit + 2)
        S = self.S
        st = self._lib.pd_solve_ivp_host(self._ctx, solver, _hptr(u0_host, S, "u0_host"), _hptr(v0_host, S, "v0_host"),
                                         _hptr(f_host, (self.nt + 1) * S, "f_host"),
                                         _hptr(u_host, self.nt * S, "u_host"), tol, m, maxit, C.byref(rep))
        _check(self._lib, self._ctx, st, allow=(PD_OK, PD_NOT_CONVERGED))
        return u_host, self._mk(st, rep, hist)

    def solve_host(self, solver: int, b_host, u_host, tol, m=20, maxit=100):
        """solver: 0 stationary, 1 GMRES, optionally | SOLVE_ZERO_GUESS; b_host, u_host [Nt, S] CPU float64."""
        rep, hist = self._report(maxit + 2)
        n = self.nt * self.S
        st = self._lib.pd_solve_host(self._ctx, solver, _hptr(b_host, n, "b_host"), _hptr(u_host, n, "u_host"), tol, m,
                                     maxit, C.byref(rep))
        _check(self._lib, self._ctx, st, allow=(PD_OK, PD_NOT_CONVERGED))
        return u_host, self._mk(st, rep, hist)

    def kernel_launches(self) -> int:
        return int(self._lib.pd_kernel_launches(self._ctx))

    def enable_phase_timing(self, on: bool = True):
        _check(self._lib, self._ctx, self._lib.pd_enable_phase_timing(self._ctx, int(on)))

    def phase_times(self):
        ms = (C.c_double * 8)()
        n = (C.c_longlong * 8)()
        _check(self._lib, self._ctx, self._lib.pd_phase_times(self._ctx, ms, n))
        return list(ms), list(n)
