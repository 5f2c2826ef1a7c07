"""Kernel-time shares of an ncu launch list (ncu --metrics gpu__time_duration.sum --csv)."""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = {}
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).split("::")[-1].split("<")[0]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[ix["Metric Value"]].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{sys.argv[2] if len(sys.argv) > 2 else ''}")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:34s} launches={c:5d} total={t:14.1f} share={100 * t / tot:5.1f}%")
