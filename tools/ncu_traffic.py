"""Per-call DRAM traffic of the cfg4 apply phases from ncu --set full reports (argv: reports...).

Writes profiles/ncu_traffic.json {cfg: {phase: bytes per call}} used by bench.py's roofline.traffic.  Per-launch
dram__bytes_read.sum + dram__bytes_write.sum of each kernel, times the launches one phase call makes at cfg4
(time FFTs: 4 chunks of 32768 pairs; y-pass: 4 chunks of 256 slabs + 1 slab)."""
import csv, json, os, subprocess, sys, collections
per = collections.defaultdict(list)
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    iK, iR, iW = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in data:
        b = float(r[iR]) * scale[units[iR]] + float(r[iW]) * scale[units[iW]]
        per[r[iK].split("(")[0].replace("void ", "").strip()].append(b)
big = {k: max(v) for k, v in per.items()}
def get(*prefixes, pick=max):
    for prefix in prefixes:  # first pattern present in the reports
        ks = [k for k in per if k.startswith(prefix) or prefix in k]
        if ks:
            return pick(per[ks[0]])
    return None
# the x-first tfx kernels (default since r01 v11), else the t1-first ones
fwd = 4 * (get("tf4_fwd_s1<2048") + get("tfx_fwd_s2x<2048", "tfx_fwd_s2<2048"))
inv = 4 * (get("tfx_inv_s1x<2048", "tfx_inv_s1<2048") + get("tf4_inv_s2<2048, 256, 16, 1, 0"))
cols = get("slab_ytri_kernel<512>") / 256 * 1025  # y-pass: per-slab bytes of a 256-slab chunk x F = 1025 slabs
out = {"cfg4": {"tfft_fwd": fwd, "spatial_solve": cols, "tfft_inv": inv},
       "source": "ncu --set full --clock-control none, tools/prof_apply.py --config cfg4 (r01); per call = per-launch "
                 "dram read+write x launches per call",
       "per_launch_bytes": big}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out["cfg4"]))
