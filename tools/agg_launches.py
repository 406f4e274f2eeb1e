"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel:
python tools/agg_launches.py FILE.csv [skip_first_n_launches]"""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
rows = rows[int(sys.argv[2]) if len(sys.argv) > 2 else 0:]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.OrderedDict()
for r in rows:
    n = r["Kernel Name"].split("(")[0].split("::")[-1][:36]
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:38s} {c:6d} {t:11.1f} us {t / c:9.2f} us/launch {100 * t / tot:5.1f}%")
print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
