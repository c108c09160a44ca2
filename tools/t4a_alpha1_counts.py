"""Table T4A at alpha = 1 (P:l.1338-1345): is the GMRES iteration count fixed in fp64?  (TEST INFRASTRUCTURE: oracle
only.)  For the meshes L = 32, 64, 128 the same right-preconditioned GMRES (solvers.solve_gmres, tol 1e-10, zero initial
guess, no restart) is run with two independent fp64 oracles of P_1^{-1} -- O1 (time DFT + sparse direct Step (b),
spectral.apply_precond) and O2 (alpha-periodic stepping in the tensor DST-I basis, periodic.apply_precond_modal) -- and
with O2 and the whole GMRES in x87 extended precision (np.longdouble: matvec_A, the Arnoldi process and Givens
rotations).  Writes tests/golden/t4a_alpha1_counts.json (argv[1] overrides); ~8 min on 8 host cores."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from oracle import periodic, problems, solvers, spectral

out = {"source": "tools/t4a_alpha1_counts.py (oracle only)", "paper": "Table T4A alpha = 1 column, P:l.1338-1345",
       "paper_iters": [3, 7, 37], "tol": 1e-10, "runs": {}}
for L in (32, 64, 128):
    cfg = W.t4a_config(L, 1.0)
    b = problems.rhs(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
    arms = {"O1_fp64": (b, lambda r, c=cfg: spectral.apply_precond(c, r)),
            "O2_fp64": (b, lambda r, c=cfg: periodic.apply_precond_modal(c, r)),
            "O2_longdouble": (b.astype(np.longdouble),
                              lambda r, c=cfg: periodic.apply_precond_modal(c, r, precision=np.longdouble))}
    for name, (bb, ap) in arms.items():
        t0 = time.time()
        u, rep = solvers.solve_gmres(cfg, bb, tol=1e-10, m=50, maxit=50, apply=ap)
        rec = {"iterations": rep.iterations, "converged": bool(rep.converged), "rel_residual": float(rep.rel_residual),
               "history": [float(h) for h in rep.history], "seconds": round(time.time() - t0, 1)}
        out["runs"][f"{L}_{name}"] = rec
        print(L, name, rec["iterations"], rec["converged"], ["%.2e" % h for h in rec["history"]], rec["seconds"],
              flush=True)
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "tests", "golden", "t4a_alpha1_counts.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
