"""Channel generation only (for ncu / timing): python tools/gen_only.py cfg4 2048 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_13925_b200 as X  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl = X.CONFIGS[cfg]
H = torch.empty(B, wl.M, wl.K, dtype=wl.dtype, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
for i in range(reps):
    ev[2 * i].record()
    X.generate_channels(wl.model, seed=0, first=i * B, B=B, dtype=wl.dtype, out=H, check=False)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
print(cfg, B, [round(ev[2 * i].elapsed_time(ev[2 * i + 1]), 3) for i in range(reps)], "ms",
      f"{B / (ev[-2].elapsed_time(ev[-1]) / 1e3):.4g} realizations/s")
