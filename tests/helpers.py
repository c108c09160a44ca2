"""Test helpers: map a workloads.Config to the library's constructor; comparison utilities."""
import numpy as np

import workloads as W

OPS = {W.ADE1D: 0, W.WAVE1D: 1, W.ADE2D: 2, W.WAVE2D: 3}
SCHEMES = {W.BE: 0, W.CN: 1, W.LF: 2}


def ctor_args(cfg):
    nu = cfg.nu if cfg.op != W.WAVE1D else 1.0
    return dict(op=OPS[cfg.op], nx=cfg.nx, ny=cfg.ny, length=cfg.length, nu=nu,
                ax=cfg.ax if cfg.op != W.WAVE1D else 0.0, ay=cfg.ay if cfg.op == W.ADE2D else 0.0,
                dt=cfg.dt, nt=cfg.nt, alpha=cfg.alpha, scheme=SCHEMES[cfg.scheme])


def make_ctx(cfg, **kw):
    from paper_2005_09158_b200 import ParaDiag
    a = ctor_args(cfg)
    a.update(kw)
    return ParaDiag(**a)


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def to_host(t):
    return t.detach().cpu().numpy()
