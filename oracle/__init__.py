"""CPU oracle for the ParaDiag-II hot path (arXiv 2005.09158) — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 numpy/scipy implementations of what the
CUDA path computes, each function citing the PAPER.md passage it follows
(``P:l.N`` = /root/reference/PAPER.md line N).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here.  The product package
``paper_2005_09158_b200`` never imports this package, and this package never
imports the product: the two share no code, headers, tables or constants.
Inputs come from ``workloads`` (seeded problem data, no method arithmetic).

Tiers:
  problems  all-at-once system A = B1 (x) M + B2 (x) K (eq 1.1), the alpha-circulant
            P_alpha = C1 (x) M + C2 (x) K (eq 1.2, 2.11b, 3.4), right-hand sides, matvecs.
  dense     O0: dense assembly + numpy.linalg.solve (tiny sizes).
  spectral  O1: spectra (Lemma 1), naive DFT-matrix Steps (a)/(c), pivoted banded LU
            or naive 2D DFT + symbol division for Step (b) (eq 1.3 / 2.12).
  periodic  O2: alpha-periodic time stepping, no DFT at all (WR form, eq 2.10).
  stepping  sequential time stepping (the classical route, P:l.76-78).
  solvers   residual, stationary iteration (eq 5.1), right-preconditioned GMRES(m).

Pins: see tests/test_oracle_*.py (marked not-gpu) and DESIGN.md §4.  No function
here is "parity unpinned".
"""
