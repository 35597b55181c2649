"""Summarise an ncu --page source --csv dump: hottest SASS lines by stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[idx[key]] or 0) for r in data)
data.sort(key=lambda r: -float(r[idx[key]] or 0))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for r in data[:n]:
    s = float(r[idx[key]] or 0)
    print(f"{100*s/tot:5.1f}%  {r[idx['Address']]:>6}  {r[idx['Source']][:110]}")
