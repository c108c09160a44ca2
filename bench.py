"""Benchmark of the ParaDiag-II hot path on B200 (see DESIGN.md §6 for the protocol).

A step = one complete ParaDiag-II solve of the workload (all SURVEY §8(a) rows: residuals, Steps (a)-(c)
of every P_alpha^{-1} apply, the Krylov / stationary update) on synthetic seeded data already resident
in HBM.  value = all-at-once dofs (Nt*Nx, all ranks) solved per second.  The apply throughput
(applies/s, apply dofs/s, % of HBM roofline under the 48 B/dof model) is reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "P_alpha^{-1} applies/s and solve time (Nt*Nx dofs/s, % HBM roofline) at 1/2/4/8 GPU"
FALLBACK_HBM = 6650.0
PHASES = ["tfft_fwd", "spatial_solve", "tfft_inv", "residual", "tfft_inv_update", "matvec", "krylov_blas1",
          "residual_norm"]
T_START = time.perf_counter()


def log(msg):
    """Bench stage timestamps on stderr (the JSON line stays alone on stdout)."""
    print(f"[bench {time.perf_counter() - T_START:7.1f}s] {msg}", file=sys.stderr, flush=True)


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def phase_bytes(cfg, S_local):
    """Algorithmic HBM bytes per launch of each timed slot: the time FFTs read or write
    8 B/dof real and the half spectrum (Nt/2+1) S 16 B; Step (b) reads and writes the half spectrum; the residual
    b - A u reads u, b and writes r (24 B/dof), its norm-only form (slot 7, GMRES cycle ends) reads u, b (16 B/dof);
    the matvec reads u and writes A u (16 B/dof).  Slot 6 (Krylov sweeps) has no fixed count."""
    D = cfg.nt * S_local
    spec = (cfg.nt // 2 + 1) * S_local * 16
    return {0: D * 8 + spec, 1: 2 * spec, 2: spec + D * 8, 3: 3 * D * 8, 4: spec + 2 * D * 8, 5: 2 * D * 8,
            7: 2 * D * 8}


def oracle_sample_cfg(cfg):
    """Bounded sample of the workload for the CPU oracle (~10-30 s of CPU work): same recipe, fewer dofs."""
    if cfg.op == W.ADE2D:
        return cfg.scaled(nx=min(cfg.nx, 256), ny=min(cfg.ny, 256), nt=min(cfg.nt, 512))
    return cfg.scaled(nx=min(cfg.nx, 1023), nt=min(cfg.nt, 1024))


def run_oracle_solve(cfg):
    from oracle import problems, solvers
    b = problems.rhs(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
    t0 = time.perf_counter()
    if cfg.solver == "stationary":
        _, rep = solvers.solve_stationary(cfg, b)
    else:
        _, rep = solvers.solve_gmres(cfg, b)
    return time.perf_counter() - t0, rep


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads", 0) for d in threadpool_info() if d.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def host_cpu():
    """nproc and the lscpu model line of the host the CPU legs ran on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def cpu_baseline(cfg, full=False):
    """The oracle (kind "oracle", the contract's key) plus BASELINE.md §3's fair CPU comparisons: the fast CPU
    ParaDiag-II (tools/cpu_fast.py: scipy.fft with workers = nproc, Thomas vectorised over frequencies) on the same
    sample and on the whole workload when it fits the host's memory, and sequential time stepping (the classical
    route, P:l.76-78) on the whole workload."""
    s = oracle_sample_cfg(cfg)
    log(f"cpu: oracle O1 solve on {s.nx}x{s.ny}x{s.nt}")
    sec, rep = run_oracle_solve(s)
    out = {"value": s.D / sec, "unit": "dofs/s", "cores": blas_threads(), "kind": "oracle",
           "sample": f"{cfg.name} recipe at Nx={s.nx}x{s.ny}, Nt={s.nt} ({s.D} dofs): one oracle O1 "
                     f"{s.solver} solve ({rep.iterations} its) in {sec:.2f} s on the host cores",
           "host": host_cpu()}
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import cpu_fast
    log("cpu: fast CPU reference on the oracle's sample")
    t_pd, its, t_seq, err = cpu_fast.timed_solve(s)
    out["fast_cpu_sample"] = {"value": s.D / t_pd, "unit": "dofs/s", "iterations": its, "seconds": round(t_pd, 3),
                              "cores": cpu_fast.NPROC, "kind": "fast CPU ParaDiag-II (tools/cpu_fast.py)",
                              "sample": f"Nx={s.nx}x{s.ny}, Nt={s.nt}"}
    out["sequential_sample"] = {"value": s.D / t_seq, "unit": "dofs/s", "seconds": round(t_seq, 3),
                                "kind": "sequential time stepping (tools/cpu_fast.py)", "rel_diff_vs_paradiag": err}
    if cfg.D > s.D:
        # the whole workload when the host holds it: sequential stepping (one [Nt][S] array) always, the fast
        # ParaDiag-II (GMRES(m): m + 1 vectors plus ~7 work arrays) with --cpu-full (minutes on cfg4)
        try:
            avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        except (ValueError, OSError):
            avail = 0
        if full and (cfg.m + 8) * cfg.D * 8 < 0.6 * avail:
            log("cpu: fast CPU reference on the whole workload")
            t_pd, its, t_seq, err = cpu_fast.timed_solve(cfg)
            out["fast_cpu_full"] = {"value": cfg.D / t_pd, "unit": "dofs/s", "iterations": its,
                                    "seconds": round(t_pd, 3), "cores": cpu_fast.NPROC,
                                    "kind": "fast CPU ParaDiag-II, whole workload"}
            out["sequential_full"] = {"value": cfg.D / t_seq, "unit": "dofs/s", "seconds": round(t_seq, 3),
                                      "kind": "sequential time stepping, whole workload", "rel_diff_vs_paradiag": err}
        elif 3 * cfg.D * 8 < 0.6 * avail:
            log("cpu: sequential stepping on the whole workload")
            t0 = time.perf_counter()
            cpu_fast.sequential(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
            t_seq = time.perf_counter() - t0
            out["sequential_full"] = {"value": cfg.D / t_seq, "unit": "dofs/s", "seconds": round(t_seq, 3),
                                      "kind": "sequential time stepping, whole workload (tools/cpu_fast.py)"}
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md recipe).

    nvidia-smi is started before the region (it needs a few hundred ms to come up) and samples every 20 ms with its
    own timestamps; only samples inside [begin(), end()] (host wall clock) are kept, so a short region still gets
    its own samples.  If none falls inside, the nearest ones are reported and flagged."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.8)
        except Exception:
            self.proc = None
        return self

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        import datetime
        rows = []
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[1]), float(f[2]), f[4:8]))
            except (ValueError, IndexError):
                continue
        if not rows:
            return None
        inside = [r for r in rows if self.t0 is not None and self.t0 <= r[0] <= self.t1]
        flag = None
        if not inside:
            mid = 0.5 * (self.t0 + self.t1) if self.t0 is not None else rows[-1][0]
            inside = sorted(rows, key=lambda r: abs(r[0] - mid))[:3]
            flag = "no sample inside the timed region: the nearest 3"
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, smv, mxv, rs in inside:
            sm.append(smv)
            mx = mxv
            for name, v in zip(names, rs):
                if v.lower().startswith("active"):
                    reasons.add(name)
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if flag:
            out["note"] = flag
        return out



def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--apply-reps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-full", action="store_true", help="also run the fast CPU ParaDiag-II on the whole workload")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torchrun (the driver's own multi-GPU launch sets WORLD_SIZE itself)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"))
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        os.execve(sys.executable, cmd, env)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    cfg = W.BY_NAME[args.config]

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2005_09158_b200 import ParaDiag, nccl_unique_id
    from tests.helpers import ctor_args

    torch.cuda.set_device(local)
    nccl_id = comm_ptr = None
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
        comm_ptr = pg_nccl_comm()
        if comm_ptr is None:  # no handle on the process group's communicator: a second one from a unique id
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
    stream = torch.cuda.current_stream()
    log(f"setup {cfg.name} on {world} rank(s) (communicator: {'process group' if comm_ptr else 'unique id'})")
    ctx = ParaDiag(**ctor_args(cfg), stream=stream, rank=rank, size=world, nccl_id=nccl_id, nccl_comm=comm_ptr)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    # ---- inputs resident in HBM: initial data -> b on device (pd_build_rhs) ----
    u0 = W.initial_u0(cfg)
    v0 = W.initial_v0(cfg)
    f = W.source_samples(cfg)
    sl = slice(ctx.offset, ctx.offset + ctx.S)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    b = ctx.build_rhs(dev(u0[sl]), dev(v0[sl]) if cfg.op == W.WAVE1D else None,
                      None if f is None else dev(np.ascontiguousarray(f[:, sl])))
    u = torch.zeros_like(b)

    def step():  # one full solve from u = 0 (GMRES: pd_solve with PD_SOLVE_ZERO_GUESS, u output only)
        if cfg.solver == "stationary":
            u.zero_()
            return ctx.solve_stationary(b, u, tol=cfg.tol, maxit=cfg.maxit)[1]
        return ctx.solve_gmres(b, u, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit, zero_guess=True)[1]

    log("warm-up")
    for _ in range(args.warmup):
        rep = step()
    barrier()
    log("timed steps")
    launches0 = ctx.kernel_launches()
    ctx.enable_phase_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        clk.begin()
        e0.record(stream)
        its = []
        for _ in range(args.steps):
            rep = step()
            its.append(rep.iterations)
        e1.record(stream)
        barrier()
        clk.end()
    ms = e0.elapsed_time(e1) / args.steps
    launches = ctx.kernel_launches() - launches0
    pms, pn = ctx.phase_times()
    ctx.enable_phase_timing(False)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = cfg.D / (ms / 1e3)

    # ---- the same solve in WR tail form (single GPU): same iterates, reported beside ----
    log("tail form")
    tail_form = None
    if world == 1:
        def step_tail():
            u.zero_()
            if cfg.solver == "stationary":
                return ctx.solve_stationary_tail(b, u, tol=cfg.tol, maxit=cfg.maxit)[1]
            return ctx.solve_gmres_tail(b, u, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)[1]

        for _ in range(max(1, args.warmup)):
            trep = step_tail()
        barrier()
        tl0 = ctx.kernel_launches()
        e0.record(stream)
        for _ in range(args.steps):
            trep = step_tail()
        e1.record(stream)
        barrier()
        tms = e0.elapsed_time(e1) / args.steps
        tail_form = {"ms_per_step": round(tms, 4), "value": cfg.D / (tms / 1e3), "unit": "dofs/s",
                     "iterations": trep.iterations, "rel_residual": trep.rel_residual,
                     "speedup_vs_residual_form": round(ms / tms, 3),
                     "gpu_launches": int(ctx.kernel_launches() - tl0),
                     "note": "pd_solve_*_tail: same iterates/counts as the headline solver; per iteration only the "
                             "last H time blocks are carried (tail map + O(H S) vector work)"}

    # ---- apply throughput (same stream, inputs > L2) ----
    log("apply throughput")
    r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    for _ in range(3):
        ctx.apply_precond(r, z)
    barrier()
    e0.record(stream)
    for _ in range(args.apply_reps):
        ctx.apply_precond(r, z)
    e1.record(stream)
    barrier()
    ams = e0.elapsed_time(e1) / args.apply_reps
    if world > 1:
        t = torch.tensor([ams], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ams = float(t.item())
    del r, z
    peak, peak_src = hbm_peak()
    apply_gbs = 48.0 * cfg.D / (ams / 1e3) / 1e9

    # ---- dominant kernel roofline ----
    pb = phase_bytes(cfg, ctx.S)
    dom = max(pb, key=lambda i: pms[i])  # dominant kernel (largest share) among those with a fixed byte count
    dom_ms = pms[dom] / max(pn[dom], 1)
    achieved = pb[dom] / (dom_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as fh:
                traffic = json.load(fh).get(cfg.name, {}).get(PHASES[dom])
        except Exception:
            traffic = None
    phases = {PHASES[i]: {"ms_per_call": round(pms[i] / pn[i], 4), "calls": int(pn[i]),
                          "share_of_step": round(pms[i] / (ms * args.steps), 4),
                          "GBps": round(pb[i] / (pms[i] / pn[i] / 1e3) / 1e9, 1) if i in pb else None}
              for i in range(8) if pn[i]}

    log("end to end")
    # ---- end to end through the host C ABI (pd_solve_ivp_host): H2D of the step's inputs (the initial data and
    # source samples) from pinned host memory, b built on the device, the solve, D2H of the space-time solution ----
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        u0h = pin(u0[sl])
        v0h = pin(v0[sl]) if cfg.op in (W.WAVE1D, W.WAVE2D) else None
        fh = pin(f[:, sl]) if f is not None else None
        uh = torch.empty(ctx.shape, dtype=torch.float64).pin_memory()
        solver = 0 if cfg.solver == "stationary" else 1

        def step_e2e():
            ctx.solve_ivp_host(solver, u0h, uh, v0h, fh, cfg.tol, cfg.m, cfg.maxit)

        for _ in range(max(1, min(args.warmup, 3))):  # warm-up (pinned staging, graph capture at launch-bound sizes)
            step_e2e()
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        ksteps = max(1, min(args.steps, 3))
        for _ in range(ksteps):
            step_e2e()
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1) / ksteps
        wall = (time.perf_counter() - t0) * 1e3 / ksteps
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = sum(x.numel() * 8 for x in (u0h, v0h, fh) if x is not None)
        e2e = {"value": cfg.D / (ems / 1e3), "unit": "dofs/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": uh.numel() * 8, "ms_per_step": round(ems, 3), "wall_ms_per_step": round(wall, 3),
               "api": "pd_solve_ivp_host (initial data in, space-time solution out)"}
        del uh

    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        del ctx, b, u
        torch.cuda.empty_cache()
        all_host_threads()
        cpu = cpu_baseline(cfg, full=args.cpu_full)
        log("cpu legs done")
    out = {
        "metric": METRIC, "value": value, "unit": "dofs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",  # cfg4 total fixed at every N
        "config": {"workload": cfg.name, "op": cfg.op, "nx": cfg.nx, "ny": cfg.ny, "nt": cfg.nt,
                   "scheme": cfg.scheme, "alpha": cfg.alpha, "solver": f"{cfg.solver}" + (
                       f"({cfg.m})" if cfg.solver == "gmres" else ""), "tol": cfg.tol, "dofs": cfg.D,
                   "iterations": its[-1], "l2": "inputs larger than L2 (vectors %.2f GB > 126 MB)" % (cfg.D * 8 / 1e9)
                   if cfg.D * 8 > 126e6 else "working set fits L2 (no flush); latency regime",
                   "parallelism": f"space/frequency transpose x{world}" if world > 1 else "1 GPU"},
        "apply": {"ms": round(ams, 4), "applies_per_s": 1e3 / ams, "dofs_per_s": cfg.D / (ams / 1e3),
                  "hbm_GBps_48B_model": round(apply_gbs, 1), "hbm_frac": round(apply_gbs / peak, 4)},
        "roofline": {"bound": "hbm", "kernel": PHASES[dom], "achieved": round(achieved, 1), "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "alg_bytes_per_launch": pb[dom], "ms_per_launch": round(dom_ms, 4)},
        "phases": phases,
        "tail_form": tail_form,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "cpu_baseline": cpu,
    }
    clk_s = clk.summary()
    if clk_s:
        out["clocks"] = clk_s
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pg_nccl_comm():
    """ncclComm_t of the default (eagerly connected) ProcessGroupNCCL, or None when torch does not expose it."""
    import torch
    import torch.distributed as dist
    try:
        be = dist.group.WORLD._get_backend(torch.device("cuda"))
        ptr = int(be._comm_ptr())
        return ptr or None
    except Exception:
        return None


def all_host_threads():
    """torchrun sets OMP_NUM_THREADS=1 for every rank; the CPU legs run on rank 0 alone and use all host cores."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count())
    except Exception:
        pass


def run_reference(args, cfg, rank, world):
    """The oracle arm: the CPU oracle as it stands, on bounded samples of the same workload."""
    if rank != 0:
        return
    all_host_threads()
    s = oracle_sample_cfg(cfg)
    for _ in range(args.warmup):
        run_oracle_solve(s)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sec, rep = run_oracle_solve(s)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    value = s.D / (ms / 1e3)
    cores = blas_threads()
    out = {"metric": METRIC, "value": value, "unit": "dofs/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": cfg.name, "sample": f"Nx={s.nx}x{s.ny}, Nt={s.nt}", "dofs": s.D,
                      "solver": cfg.solver, "iterations": rep.iterations},
           "cpu_baseline": {"value": value, "unit": "dofs/s", "cores": cores, "kind": "oracle",
                            "sample": f"{cfg.name} recipe at {s.D} dofs (Nx={s.nx}x{s.ny}, Nt={s.nt}), oracle O1 "
                                      f"{cfg.solver} solve per step"},
           "e2e": {"value": value, "unit": "dofs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
