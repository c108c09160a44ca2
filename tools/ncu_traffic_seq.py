"""Per-call DRAM traffic of the cfg4 time FFTs in their natural launch sequence (argv: ncu CSV log, calls).

The chunked 2D time FFT (3 streams of 16 MB four-step chunks) relies on L2 between stage 1 and
stage 2 of a chunk, which the per-kernel cold-cache captures cannot see.  Input: the CSV of
  ncu --replay-mode application --cache-control none --clock-control none
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
      -k regex:"tf4_fwd_s1|tfx_fwd_s2x|tfx_inv_s1x|tf4_inv_s2" --csv python tools/prof_apply.py --config cfg4
(ncu serialises the streams, so each chunk's stage 2 directly follows its stage 1).  Sums every launch of the
forward pair and of the inverse pair and divides by the number of calls of each (argv[2], prof_apply: 2);
updates profiles/ncu_traffic.json (tfft_fwd / tfft_inv) keeping the cold-capture numbers under "cold"."""
import collections, csv, json, os, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
iK, iM, iU, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= iV:
        continue
    name = r[iK].split("(")[0].replace("void ", "").strip()
    key = "fwd" if ("tf4_fwd_s1" in name or "tfx_fwd_s2x" in name) else "inv" if ("tfx_inv_s1x" in name or "tf4_inv_s2<2048, 256, 16, 1, 0" in name) else None
    if key is None:
        continue
    v = float(r[iV].replace(",", "")) * scale.get(r[iU], 1)
    if r[iM].startswith("dram__bytes"):
        tot[key + "_bytes"] += v
    elif r[iM] == "gpu__time_duration.sum":
        tot[key + "_s"] += v
        cnt[key] += 1
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
doc = json.load(open(path))
doc.setdefault("cold", dict(doc["cfg4"]))
doc["cfg4"]["tfft_fwd"] = tot["fwd_bytes"] / calls
doc["cfg4"]["tfft_inv"] = tot["inv_bytes"] / calls
doc["sequence"] = {"source": "ncu --replay-mode application --cache-control none (tools/ncu_traffic_seq.py); "
                             "serialised launches in program order", "launches_per_call": {k: v / calls for k, v in cnt.items()},
                   "bytes_per_call": {"tfft_fwd": tot["fwd_bytes"] / calls, "tfft_inv": tot["inv_bytes"] / calls},
                   "serialised_ms_per_call": {"tfft_fwd": 1e3 * tot["fwd_s"] / calls, "tfft_inv": 1e3 * tot["inv_s"] / calls}}
json.dump(doc, open(path, "w"), indent=1)
print(json.dumps(doc["sequence"]))
