"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel name, launches and mean / total device time (us)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        agg.setdefault(d["Kernel Name"].split("(")[0][:48], []).append(v)
tot = sum(sum(v) for v in agg.values())
for n, v in agg.items():
    print(f"{n:48s} n={len(v):4d} mean={sum(v) / len(v):10.1f} us  total={sum(v):10.1f} us  {100 * sum(v) / tot:5.1f}%")
