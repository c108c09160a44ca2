"""World-size-2 gloo test of the sharded path's host logic on CPU (no GPU): the partition plan exported by
libparadiag.so (pd_partition), the all-to-all block layout (frequency rows [f_q, f_q+F_q) of rank p's slab
land in columns [s_off_p, +s_cnt_p) of rank q's frequency shard) and the halo plan of the residual (1D
Dirichlet: no neighbour at the ends; 2D periodic: ring of y-rows) — the same rules dist.cpp executes with
NCCL — with the oracle's Step (a)/(b)/(c) standing in for the kernels.  Result == single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W
from oracle import problems, spectral

OPS = {W.ADE1D: 0, W.WAVE1D: 1, W.ADE2D: 2}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(blocks_out, shapes_in, rank, P):
    """blocks_out[q]: array to send to q; shapes_in[p]: shape of the block coming from p (p2p over gloo)."""
    recv = [None] * P
    reqs = []
    bufs = {}
    for p in range(P):
        if p == rank:
            recv[p] = blocks_out[p]
            continue
        bufs[p] = torch.zeros(tuple(shapes_in[p]) + (2,), dtype=torch.float64)
        reqs.append(dist.irecv(bufs[p], src=p))
    for q in range(P):
        if q != rank:
            t = torch.view_as_real(torch.from_numpy(np.ascontiguousarray(blocks_out[q])))
            reqs.append(dist.isend(t.contiguous(), dst=q))
    for rq in reqs:
        rq.wait()
    for p, t in bufs.items():
        recv[p] = torch.view_as_complex(t).numpy()
    return recv


def _worker(rank, P, port, cfg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        from paper_2005_09158_b200 import partition
        s_off, s_cnt, f_off, f_cnt = partition(OPS[cfg.op], cfg.nx, cfg.ny, cfg.nt, P)
        Sg, F, nt = cfg.S, cfg.nt // 2 + 1, cfg.nt
        r = W.random_vector(cfg, seed=5)
        sl = slice(s_off[rank], s_off[rank] + s_cnt[rank])
        r_loc = r[:, sl]
        # Step (a) on the local slab, half spectrum
        S1_loc = spectral.step_a(cfg, r_loc)[:F]
        # all-to-all: to q the rows of q's frequencies
        out = [S1_loc[f_off[q]:f_off[q] + f_cnt[q]] for q in range(P)]
        inn = _exchange(out, [(f_cnt[rank], s_cnt[p]) for p in range(P)], rank, P)
        Sg_rows = np.zeros((f_cnt[rank], Sg), dtype=np.complex128)
        for p in range(P):
            Sg_rows[:, s_off[p]:s_off[p] + s_cnt[p]] = inn[p]
        lam1, lam2 = spectral.spectra(cfg)
        fs = slice(f_off[rank], f_off[rank] + f_cnt[rank])
        S2_rows = spectral.step_b(cfg, Sg_rows, lam1[fs], lam2[fs])
        # back: to p the columns of p's slab
        back = [S2_rows[:, s_off[p]:s_off[p] + s_cnt[p]] for p in range(P)]
        got = _exchange(back, [(f_cnt[q], s_cnt[rank]) for q in range(P)], rank, P)
        S2_half = np.zeros((F, s_cnt[rank]), dtype=np.complex128)
        for q in range(P):
            S2_half[f_off[q]:f_off[q] + f_cnt[q]] = got[q]
        full = np.zeros((nt, s_cnt[rank]), dtype=np.complex128)
        full[:F] = S2_half
        for n in range(F, nt):
            full[n] = np.conj(S2_half[nt - n])
        z_loc = spectral.step_c(cfg, full)
        # residual with halos (1D: neighbour columns, Dirichlet ends; 2D: ring of rows)
        u = np.random.default_rng(9).standard_normal((nt, Sg))
        u_loc = u[:, sl]
        hw = cfg.nx if cfg.op == W.ADE2D else 1
        first, last = u_loc[:, :hw], u_loc[:, -hw:]
        ring = cfg.op == W.ADE2D
        prev, nxt = (rank - 1) % P, (rank + 1) % P
        sends = [None] * P
        # both neighbours may be the same rank (P = 2 ring): pack (last -> next, first -> prev) as one message
        msgs = {}
        if ring or rank < P - 1:
            msgs.setdefault(nxt, []).append(("last", last))
        if ring or rank > 0:
            msgs.setdefault(prev, []).append(("first", first))
        for q in range(P):
            parts = [m for _, m in msgs.get(q, [])]
            sends[q] = np.concatenate(parts, axis=1).astype(np.complex128) if parts else np.zeros((nt, 0), complex)
        expect = {}
        for p in range(P):
            n_in = 0
            if (ring or p < P - 1) and (p + 1) % P == rank:
                n_in += hw
            if (ring or p > 0) and (p - 1) % P == rank:
                n_in += hw
            expect[p] = (nt, n_in)
        sends[rank] = np.zeros((nt, 0), complex)
        recvd = _exchange(sends, [expect[p] if p != rank else (nt, 0) for p in range(P)], rank, P)
        # parse each peer's message in that peer's send order: (last -> its next), (first -> its prev)
        def parts_from(X):
            names = []
            if (ring or X < P - 1) and (X + 1) % P == rank:
                names.append("last")
            if (ring or X > 0) and (X - 1) % P == rank:
                names.append("first")
            blk = recvd[X].real
            return {nm: blk[:, i * hw:(i + 1) * hw] for i, nm in enumerate(names)}

        hlo = parts_from(prev)["last"] if (ring or rank > 0) else None
        hhi = parts_from(nxt)["first"] if (ring or rank < P - 1) else None
        # local A u with halos, compared column-by-column with the oracle's global residual
        Kloc = np.zeros_like(u_loc)
        if cfg.op == W.ADE2D:
            n = cfg.nx
            h = 2 * np.pi / n
            ny = s_cnt[rank] // n
            U = u_loc.reshape(nt, ny, n)
            lo = hlo.reshape(nt, 1, n) if hlo is not None else U[:, -1:]
            hi = hhi.reshape(nt, 1, n) if hhi is not None else U[:, :1]
            Ue = np.concatenate([lo, U, hi], axis=1)
            c = Ue[:, 1:-1]
            lap = (4 * c - np.roll(c, 1, 2) - np.roll(c, -1, 2) - Ue[:, :-2] - Ue[:, 2:]) / h ** 2
            adv = cfg.ax * (np.roll(c, -1, 2) - np.roll(c, 1, 2)) / (2 * h) + cfg.ay * (Ue[:, 2:] - Ue[:, :-2]) / (2 * h)
            KU = (cfg.nu * lap + adv).reshape(nt, -1)
        else:
            K = problems.K_matrix(cfg)
            sub, dia, sup = K.diagonal(-1)[0], K.diagonal(0)[0], K.diagonal(1)[0]
            lo = hlo if hlo is not None else np.zeros((nt, 1))
            hi = hhi if hhi is not None else np.zeros((nt, 1))
            Ue = np.concatenate([lo, u_loc, hi], axis=1)
            KU = sub * Ue[:, :-2] + dia * Ue[:, 1:-1] + sup * Ue[:, 2:]
        Kloc[:] = KU
        c1, c2 = problems.time_first_columns(cfg)
        Au_loc = problems.apply_time(c1, u_loc, None) + problems.apply_time(c2, Kloc, None)
        gathered = [None] * P if rank == 0 else None
        dist.gather_object((z_loc, Au_loc), gathered, dst=0)
        if rank == 0:
            z = np.concatenate([g[0] for g in gathered], axis=1)
            Au = np.concatenate([g[1] for g in gathered], axis=1)
            e1 = np.linalg.norm(z - spectral.apply_precond(cfg, r)) / np.linalg.norm(z)
            Aref = problems.matvec_A(cfg, u)
            e2 = np.linalg.norm(Au - Aref) / np.linalg.norm(Aref)
            out_q.put((e1, e2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,P", [
    (W.CONFIGS[0].scaled(nx=37, nt=16), 2),
    (W.CONFIGS[2].scaled(nx=30, nt=16), 2),
    (W.CONFIGS[3].scaled(nx=8, ny=8, nt=8), 2),
    (W.CONFIGS[3].scaled(nx=12, ny=12, nt=8), 3),
])
def test_two_rank_plan_matches_oracle(cfg, P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, cfg, q)) for r in range(P)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    e1, e2 = q.get(timeout=10)
    assert e1 < 1e-12 and e2 < 1e-13


def _tail_worker(rank, P, port, cfg, out_q):
    """Sharded tail map (tailform.cpp, NCCL mode): every rank holds the replicated head, solves the shifted systems
    of its plan's half-spectrum frequencies [f_off, f_off + f_cnt), weights the last H rows of Step (c) with the
    half-spectrum multiplicities, and one all-reduce sums the partial tails."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        from paper_2005_09158_b200 import partition
        from oracle import tail
        _, _, f_off, f_cnt = partition(OPS[cfg.op], cfg.nx, cfg.ny, cfg.nt, P)
        nt, H = cfg.nt, tail.head_blocks(cfg)
        g = np.random.default_rng(21).standard_normal((H, cfg.S))
        gam = spectral.gamma(nt, cfg.alpha)
        lam1, lam2 = spectral.spectra(cfg)
        fs = np.arange(f_off[rank], f_off[rank] + f_cnt[rank])
        S1 = sum((gam[t] * np.exp(-2j * np.pi * fs * t / nt))[:, None] * g[t][None, :] for t in range(H))
        S2 = spectral.step_b(cfg, S1, lam1[fs], lam2[fs])
        mult = np.where((fs == 0) | (2 * fs == nt), 1.0, 2.0)
        part = np.zeros((H, cfg.S))
        for a in range(H):
            t = nt - H + a
            w = mult * np.exp(2j * np.pi * fs * t / nt) / nt / gam[t]
            part[a] = (w[:, None] * S2).real.sum(axis=0)
        tt = torch.from_numpy(part)
        dist.all_reduce(tt)
        if rank == 0:
            ref = tail.tail_map(cfg, g)
            out_q.put(float(np.linalg.norm(tt.numpy() - ref) / np.linalg.norm(ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,P", [(W.CONFIGS[1].scaled(nx=31, nt=16), 2), (W.CONFIGS[2].scaled(nx=30, nt=16), 3)])
def test_sharded_tail_map_frequency_split(cfg, P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tail_worker, args=(r, P, port, cfg, q)) for r in range(P)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    assert q.get(timeout=10) < 1e-11
