"""Time the fused cfg3 call (check=False) under the current XL_FUSED_* env;
prints precoders/s.  Development aid for A/B experiments.
The XL_FUSED_* settings need the development-hooks build
(build_ext.py --out variants/dev.so -DXL_DEV_HOOKS=1; run via tools/with_lib.sh).
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_13925_b200 as X
from paper_2305_13925_b200 import batched as BT
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
wl = X.CONFIGS[cfg]
H = X.generate_channels(wl.model, seed=0, first=0, B=B, dtype=wl.dtype)
out = BT.alloc_outputs(H, want_gamma=True)
T = int(os.environ.get("T", wl.T))
f = lambda: BT.rzf_batched(H, wl.alpha(), wl.power(), T=T, out=out, check=False)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"dbg={os.environ.get('XL_FUSED_DEBUG', '-')} T={T}: {B / ms * 1e3 / 1e6:.3f} M/s  {ms:.3f} ms")
