"""Time on-device channel generation (chan_kernel) for a config: realizations/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_13925_b200 as X
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
wl = X.CONFIGS[cfg]
H = X.generate_channels(wl.model, seed=0, first=0, B=B, dtype=wl.dtype)
f = lambda i: X.generate_channels(wl.model, seed=0, first=i * B, B=B, dtype=wl.dtype, out=H, check=False)
for i in range(2):
    f(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(5):
    f(i)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"{cfg} channel generation: {B / ms * 1e3:.0f} realizations/s ({ms:.3f} ms per {B}; "
      f"{B * wl.M * wl.K * (8 if wl.dtype == torch.complex64 else 16) / ms / 1e6:.0f} GB/s written)")
