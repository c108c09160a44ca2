"""Table T4A (P:l.1309-1349): 2D Dirichlet wave, implicit leapfrog, right-preconditioned GMRES with P_alpha,
alpha in {0.1, 1}, zero initial guess, tol 1e-10, no restart (maxit 50).  Oracle only (TEST INFRASTRUCTURE):
the modal O2 apply (DST-I basis, independent of the DFT-in-time O1) inside solvers.solve_gmres, the sequential
march for the converged solution, and the L_inf(0,T; L2) error vs the exact sin(pi x) sin(pi y) e^t.
Writes tests/golden/t4a_oracle.json (argv[1] overrides).  ~1-3 min on 16 host cores."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from oracle import periodic, problems, solvers, stepping

out = {"source": "tools/t4a_oracle.py: solvers.solve_gmres with periodic.apply_precond_modal (O2), m = maxit = 50",
       "paper": "Table T4A, P:l.1333-1349", "labels": list(W.T4A_LABELS), "paper_errors": list(W.T4A_ERRORS),
       "paper_iters": {str(a): list(v) for a, v in W.T4A_ITERS.items()}, "runs": {}}
for L in W.T4A_LABELS:
    for alpha in (0.1, 1.0):
        if L == 256 and alpha == 1.0:
            continue  # > 50 iterations of 16.5M-dof vectors: out of the oracle's budget
        cfg = W.t4a_config(L, alpha)
        b = problems.rhs(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
        t0 = time.time()
        u, rep = solvers.solve_gmres(cfg, b, tol=1e-10, m=50, maxit=50,
                                     apply=lambda r, c=cfg: periodic.apply_precond_modal(c, r))
        ex = W.exact_wave_solution(cfg)
        err = float(np.sqrt(cfg.h ** 2 * np.sum((u - ex) ** 2, axis=1)).max())
        rec = {"iterations": rep.iterations, "converged": bool(rep.converged), "rel_residual": rep.rel_residual,
               "history": [float(h) for h in rep.history], "error": err, "seconds": round(time.time() - t0, 1)}
        out["runs"][f"{L}_{alpha}"] = rec
        print(L, alpha, rec["iterations"], rec["converged"], "err %.3e" % err, "%.1fs" % rec["seconds"], flush=True)
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "tests", "golden", "t4a_oracle.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
