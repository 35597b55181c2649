"""Pinned host <-> device copy bandwidth: H2D alone, D2H alone, both at once
(the e2e path's bound).  Development aid."""
import torch, time
n = 2 << 30
dev = torch.device("cuda")
hs = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hd = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, chunks=1):
    torch.cuda.synchronize()
    t = time.perf_counter()
    c = n // chunks
    for i in range(chunks):
        if h2d:
            with torch.cuda.stream(s1):
                d1[i*c:(i+1)*c].copy_(hs[i*c:(i+1)*c], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                hd[i*c:(i+1)*c].copy_(d2[i*c:(i+1)*c], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t
for chunks in (1, 8):
    run(True, True, chunks)
    for name, a, b in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
        dt = min(run(a, b, chunks) for _ in range(3))
        print(f"chunks={chunks} {name:5s} {n / dt / 1e9:6.1f} GB/s per direction", flush=True)
