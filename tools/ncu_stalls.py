"""Per-CUDA-line stall samples with the dominant stall reasons, from
`ncu -i rep --page source --csv --print-source cuda,sass` (SASS rows are
aggregated onto the CUDA line that precedes them)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
cur = None
fname = None
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path' or r[0] == 'File Name':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No' or r[0] == '#':
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    if len(r) > 2 and r[2] == '-':      # CUDA source row
        cur = (fname, int(r[0]))
        src[cur] = r[1][:90].strip()
        for i, h in enumerate(hdr):
            if h.startswith('stall_') and '(Not Issued)' not in h:
                try:
                    agg[cur][h[6:]] += float(r[i] or 0)
                except ValueError:
                    pass
tot = sum(sum(c.values()) for c in agg.values())
print('total', tot)
for k, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:n]:
    s = sum(c.values())
    top = ', '.join(f"{a} {100*b/s:.0f}%" for a, b in c.most_common(3))
    print(f"{100*s/tot:5.1f}%  {k[0]}:{k[1]}  [{top}]  {src[k]}")
