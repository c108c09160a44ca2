"""Table ctp-01 (P:l.954-978): which stopping quantity reproduces the printed iteration counts?  Oracle-only
(O1 apply + plain residual), stationary ParaDiag-II (eq 2.10) from u^0 = 0, recording candidate quantities.

Writes tests/golden/ctp01_oracle.json (argv[1] overrides): per (scheme, nu) the per-iteration quantities, the
iteration count under each candidate rule, and the counts printed in the paper.  Only oracle/ and workloads/
are used (TEST INFRASTRUCTURE; takes ~2 min on 16 host cores)."""
import json, math, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from oracle import problems, solvers, spectral

PAPER = {s: list(v) for s, v in W.CTP01_COUNTS.items()}
NUS = list(W.CTP01_NUS)
out = {}
for scheme in ["be", "cn"]:
    for nu in NUS:
        cfg = W.ctp01_config(scheme, nu)
        b = problems.rhs(cfg, W.initial_u0(cfg))
        bn = np.linalg.norm(b)
        u = np.zeros_like(b)
        rows = []
        iters = []
        for k in range(1, 8):
            r = solvers.residual(cfg, b, u)
            u_new = u + spectral.apply_precond(cfg, r)
            d = u_new - u
            rr = np.linalg.norm(solvers.residual(cfg, b, u_new)) / bn
            rows.append({"k": k, "res_rel2": rr, "dif_inf": float(np.abs(d).max()),
                         "dif_rel_inf": float(np.abs(d).max() / np.abs(u_new).max()),
                         "dif_l2h": float(np.linalg.norm(d) / 128.0 / math.sqrt(cfg.nt)),
                         "dif_rel2": float(np.linalg.norm(d) / np.linalg.norm(u_new))})
            u = u_new
            iters.append(u.copy())
        for row, uk in zip(rows, iters):  # error vs the converged solution (the 7th iterate)
            row["err_inf"] = float(np.abs(uk - u).max())
            row["err_rel_inf"] = float(np.abs(uk - u).max() / np.abs(u).max())
        out[f"{scheme}_{nu}"] = rows
        print(scheme, nu, " ".join("%d:%.1e/%.1e" % (r["k"], r["res_rel2"], r["dif_inf"]) for r in rows), flush=True)
rules = ["res_rel2", "dif_inf", "dif_rel_inf", "dif_l2h", "dif_rel2", "err_inf", "err_rel_inf"]
for rule in rules:
    counts = {s: [next((r["k"] for r in out[f"{s}_{nu}"] if r[rule] <= 1e-6), None) for nu in NUS]
              for s in ["be", "cn"]}
    print(rule, counts, "MATCH" if counts == PAPER else "")
golden = {"source": "tools/ctp01_rules.py: oracle O1 (spectral.apply_precond) + solvers.residual, u^0 = 0, tol 1e-6",
          "paper": "Table ctp-01, P:l.954-978 (B-E, TR columns; identical for every np)",
          "paper_counts": {s: list(W.CTP01_COUNTS[s]) for s in ["be", "cn"]}, "nus": list(NUS),
          "counts": {rule: {s: [next((r["k"] for r in out[f"{s}_{nu}"] if r[rule] <= 1e-6), None) for nu in NUS]
                            for s in ["be", "cn"]} for rule in rules},
          "runs": out}
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "tests", "golden", "ctp01_oracle.json")
with open(path, "w") as fh:
    json.dump(golden, fh, indent=1)
