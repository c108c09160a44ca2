"""Debug helper: apply parity of the tfx (x-folded time FFT) cases against the oracle with a given library (argv[1])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_09158_b200 import _lib
_lib._LIB_PATH = sys.argv[1]
import workloads as W
from oracle import spectral
from tests.helpers import make_ctx, rel, to_dev, to_host
for nx, nt, P in ((32, 1024, 0), (64, 1024, 0), (32, 2048, 0), (32, 2048, 4), (128, 1024, 0)):
    cfg = W.CONFIGS[4].scaled(nx=nx, ny=nx, nt=nt, alpha=1e-3)
    ctx = make_ctx(cfg, rank=-1, size=P) if P else make_ctx(cfg)
    r = W.random_vector(cfg, seed=11)
    z = to_host(ctx.apply_precond(to_dev(r)))
    print(os.path.basename(sys.argv[1]), nx, nt, P, "rel", rel(z, spectral.apply_precond(cfg, r)), flush=True)
