"""Per-CUDA-line stall samples / executed instructions from
`ncu --page source --csv --print-source cuda,sass`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
cur = None
agg = {}
tot_s = tot_i = 0.0
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if not r[0].isdigit() or len(r) < 8 or r[2] != '-':
        continue
    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    s, i = f(r[4]), f(r[7])
    agg[(cur, int(r[0]))] = (s, i, r[1][:95])
    tot_s += s
    tot_i += i
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print('total stall samples', tot_s, 'inst', tot_i)
for (fn, ln), (s, i, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{100*s/tot_s:5.1f}% st {100*i/max(tot_i,1):5.1f}% in  {fn}:{ln}  {src.strip()}")
