"""Tuning helper: time apply phases of a config with an alternative libparadiag build (argv: lib config [reps])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_09158_b200 import _lib
_lib._LIB_PATH = sys.argv[1]
import workloads as W
from tests.helpers import make_ctx
name = sys.argv[2]
cfg = W.t4a_config(int(name[4:])) if name.startswith("t4a_") else W.BY_NAME[name]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
ctx = make_ctx(cfg)
r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); z = torch.empty_like(r)
for _ in range(2): ctx.apply_precond(r, z)
torch.cuda.synchronize()
ctx.enable_phase_timing(True)
for _ in range(reps): ctx.apply_precond(r, z)
torch.cuda.synchronize()
ms, cnt = ctx.phase_times()
print(os.path.basename(sys.argv[1]), name, " ".join("%d:%.3f" % (i, ms[i] / max(cnt[i], 1)) for i in range(3)))
