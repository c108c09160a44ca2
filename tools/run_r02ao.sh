# r02ao A/B: ld.cg instead of ld.cs for the old values of the accumulating inverse stage 2 (u += P^{-1} r of the stationary
# iteration, libparadiag_acc.so): solve times of the stationary configs
mkdir -p gpurun_out
L=paper_2005_09158_b200
cat > /tmp/st_ab.py <<'P'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2005_09158_b200 import _lib
_lib._LIB_PATH = sys.argv[1]
import workloads as W
from tests.helpers import make_ctx, to_dev
cfg = W.BY_NAME[sys.argv[2]]
ctx = make_ctx(cfg)
b = ctx.build_rhs(to_dev(W.initial_u0(cfg)))
def solve():
    u = torch.zeros_like(b)
    return ctx.solve_stationary(b, u, tol=cfg.tol, maxit=cfg.maxit)
for _ in range(3): solve()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): u, rep = solve()
e1.record(); torch.cuda.synchronize()
print(os.path.basename(sys.argv[1]), sys.argv[2], "solve ms %.4f its %d" % (e0.elapsed_time(e1) / 20, rep.iterations))
P
for rep in 1 2; do for lib in libparadiag.so libparadiag_acc.so; do for c in cfg2 cfg0; do python /tmp/st_ab.py $L/$lib $c 2>&1 | tail -1; done; done; done | tee gpurun_out/r02ao_acc_ab.txt
