"""Match gpurun_out/energy.log windows with nvidia-smi power samples."""
import datetime, re, statistics
rows = []
for l in open("gpurun_out/energy_smi.csv"):
    ts, p, c = [x.strip() for x in l.split(",")]
    t = datetime.datetime.strptime(ts, "%Y/%m/%d %H:%M:%S.%f").replace(tzinfo=datetime.timezone.utc).timestamp()
    rows.append((t, float(p.split()[0]), float(c.split()[0])))
idle = None
for l in open("gpurun_out/energy.log"):
    m = re.match(r"(\S+)\s+t0 (\S+) t1 (\S+)\s+(\d+) GB/s", l)
    n, t0, t1, bw = m.group(1), float(m.group(2)), float(m.group(3)), float(m.group(4))
    s = [r for r in rows if t0 + 0.8 < r[0] < t1 - 0.1]
    p, c = statistics.median(r[1] for r in s), statistics.median(r[2] for r in s)
    if idle is None:
        idle = p
    e = (p - idle) / bw * 1e3 if bw else 0.0
    print(f"{n:16s} {bw:6.0f} GB/s  {p:6.0f} W  clk {c:5.0f}  pJ/B above idle {e:6.1f}")
