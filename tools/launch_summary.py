"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", "")) * {"ms": 1e3, "us": 1, "ns": 1e-3, "usecond": 1,
                                                             "msecond": 1e3, "nsecond": 1e-3}.get(d["Metric Unit"], 1)
            k = d["Kernel Name"][:70]
            agg[k][0] += 1
            agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"  {n:4d} {t / 1e3:9.2f} ms {100 * t / tot:5.1f}% {k}")
