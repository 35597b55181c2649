"""One batched precoder call of a config (for ncu launch lists / captures):
    python tools/one_call.py cfg5 [B] [repeats] [method]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_13925_b200 as X  # noqa: E402
from paper_2305_13925_b200 import batched as BT  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
wl = X.CONFIGS[cfg]
B = int(sys.argv[2]) if len(sys.argv) > 2 else min(wl.B, 2048)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
method = sys.argv[4] if len(sys.argv) > 4 else "jacpcg"
H = X.generate_channels(wl.model, seed=0, first=0, B=B, dtype=wl.dtype)
out = BT.alloc_outputs(H)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
for i in range(reps):
    ev[2 * i].record()
    BT.rzf_batched(H, wl.alpha(), wl.power(), method=method, T=wl.T, out=out, check=False)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
X._lib.raise_status(out.status.cpu().numpy(), cfg) if hasattr(X, "_lib") else None
print(cfg, B, method, [round(ev[2 * i].elapsed_time(ev[2 * i + 1]), 3) for i in range(reps)], "ms",
      f"{B / (ev[-2].elapsed_time(ev[-1]) / 1e3):.4g} precoders/s")
