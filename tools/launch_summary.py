"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel count, total and share."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    name = r[iK].split("(")[0].replace("void ", "").strip()
    tot[name] += float(r[iV].replace(",", "")); cnt[name] += 1
T = sum(tot.values())
print("%-60s %6s %12s %7s" % ("kernel", "calls", "total_ms", "share"))
for k, v in tot.most_common():
    print("%-60s %6d %12.3f %6.1f%%" % (k[:60], cnt[k], v / 1e6, 100 * v / T))
print("launches", sum(cnt.values()))
