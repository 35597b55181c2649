"""Effective SM clock and board power of the fused cfg3 kernel under several
XL_FUSED_* settings (development aid).  For each setting: run the kernel in a
loop for ~3 s sampling NVML power / clock, then one traced launch whose
clock64 / globaltimer ratio gives the effective SM clock.
The XL_FUSED_* settings need the development-hooks build
(build_ext.py --out variants/dev.so -DXL_DEV_HOOKS=1; run via tools/with_lib.sh).
"""
import os, sys, subprocess, threading, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
import paper_2305_13925_b200 as X
from paper_2305_13925_b200 import batched as BT

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
wl = X.CONFIGS["cfg3"]
B = int(os.environ.get("B", 32768))
H = X.generate_channels(wl.model, seed=0, first=0, B=B, dtype=wl.dtype)
out = BT.alloc_outputs(H, want_gamma=True)
f = lambda: BT.rzf_batched(H, wl.alpha(), wl.power(), T=int(os.environ.get("T", wl.T)), out=out, check=False)
settings = sys.argv[1:] or ["-"]
print("power limit W", pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1e3, flush=True)
for s in settings:
    env = {}
    if s != "-":
        for kv in s.split(","):
            k, v = kv.split("=")
            env[k] = v
    for k in ("XL_FUSED_DEBUG", "XL_FUSED_L2", "XL_FUSED_GRID", "T"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    pw, ck, stop = [], [], threading.Event()

    def samp():
        while not stop.is_set():
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1e3)
            ck.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.02)
    th = threading.Thread(target=samp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    th.start()
    e0.record()
    t0 = time.time()
    while time.time() - t0 < 3.0:
        for _ in range(5):
            f()
        n += 5
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / n
    os.environ["XL_FUSED_TRACE"] = "1"
    f(); f()
    torch.cuda.synchronize()
    os.environ.pop("XL_FUSED_TRACE")
    print(f"{s:40s} {B / ms * 1e3 / 1e6:6.3f} M/s {ms:8.3f} ms  power med {statistics.median(pw):6.0f} W  E {statistics.median(pw) * ms * 1e3 / B:6.1f} uJ/real max {max(pw):6.0f}  nvml clk {statistics.median(ck):5.0f}", flush=True)
