"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list.
python tools/ncu_launches.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {x: i for i, x in enumerate(h)}
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    u = r[ix["Metric Unit"]]
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[u]
    k = r[ix["Kernel Name"]]
    tot[k] += v
    cnt[k] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.3f} ms {100 * v / s:5.1f}% n={cnt[k]:4d} {k[:100]}")
