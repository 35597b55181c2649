"""Phase timeline of the K = 256 cluster solver (cluster 0, CTA 0): clock64
stamps via xl_debug_lk_trace.  python tools/lk_trace.py [B] [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_13925_b200 as X  # noqa: E402
from paper_2305_13925_b200 import _lib as L  # noqa: E402
from paper_2305_13925_b200 import batched as BT  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
T = int(sys.argv[2]) if len(sys.argv) > 2 else 6
wl = X.CONFIGS["cfg5"]
H = X.generate_channels(wl.model, seed=0, first=0, B=B, dtype=wl.dtype)
BT.rzf_batched(H, wl.alpha(), wl.power(), T=T, check=False)
buf = torch.zeros(256, dtype=torch.int64, device="cuda")
L.lib().xl_debug_lk_trace(L.ptr(buf))
BT.rzf_batched(H, wl.alpha(), wl.power(), T=T, check=False)
torch.cuda.synchronize()
L.lib().xl_debug_lk_trace(None)
t = buf.cpu().tolist()
n = next((i for i, v in enumerate(t) if v == 0), len(t))
labels = ["top", "synced", "built", "slot ready"]
for it in range(T):
    labels += [f"it{it + 1} start", "scaled", "product", "update+rz"]
labels += ["gx start", "gx loaded", "gx computed", "X written", "GX written"]
per = len(labels)
for i in range(1, min(n, 2 * per)):
    print(f"{labels[i % per]:>12s} +{t[i] - t[i - 1]:8d} cycles")
print("realization:", t[per] - t[0] if n > per else None, "cycles")

# per-chunk: producer issue time (after its empty wait) and consumer landing time
iss = t[128:192]
lnd = t[192:256]
print("chunk  issue->land  land gap")
for n in range(1, 48):
    if iss[n] and lnd[n]:
        print(f"{n:5d} {lnd[n] - iss[n]:10d} {lnd[n] - lnd[n - 1]:9d}")
