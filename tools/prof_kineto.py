"""Per-kernel durations of cfg4 applies in the default stream-pipelined regime, via torch.profiler (CUPTI activity
records; unlike ncu it does not serialise the streams).  Prints count, mean and total per kernel and the wall
time per apply (argv: config, applies)."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from tests.helpers import make_ctx
cfg = W.BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = make_ctx(cfg)
r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); z = torch.empty_like(r)
for _ in range(2): ctx.apply_precond(r, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA], acc_events=True) as prof:
    e0.record()
    for _ in range(n): ctx.apply_precond(r, z)
    e1.record()
    torch.cuda.synchronize()
tot = collections.Counter(); cnt = collections.Counter()
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:60]
        tot[k] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        cnt[k] += 1
print("wall ms per apply %.3f" % (e0.elapsed_time(e1) / n))
for k, v in tot.most_common(12):
    print("%-60s %6d  mean %8.2f us  per-apply %8.3f ms" % (k, cnt[k], v / cnt[k], v / n / 1e3))
