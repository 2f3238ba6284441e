"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel count, total, share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
data = data[skip:]
agg = collections.OrderedDict()
for d in data:
    k = d["Kernel Name"].split("(")[0][:70]
    unit = d["Metric Unit"]
    v = float(d["Metric Value"].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                                                        "nsecond": 1e-3}.get(unit, 1.0)
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':72s} {'n':>5s} {'total us':>10s} {'us/launch':>10s} {'share':>7s}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:72s} {c:5d} {t:10.1f} {t / c:10.2f} {100 * t / tot:6.1f}%")
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
