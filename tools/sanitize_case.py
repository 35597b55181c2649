"""Small precoder calls for compute-sanitizer (one tool per run):
fused K<=64 (cfg3 shape), K = 128 chain (cluster PCG), K = 256 chain
(cluster solver with multicast), complex128 DMMA GEMM (K = 96)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_13925_b200 as X  # noqa: E402
from paper_2305_13925_b200 import batched as BT  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
cases = {"cfg3": ("cfg3", 4), "cfg4": ("cfg4", 2), "cfg5": ("cfg5", 2)}
for name, (cfg, B) in cases.items():
    if which not in ("all", name):
        continue
    wl = X.CONFIGS[cfg]
    H = X.generate_channels(wl.model, seed=0, first=0, B=B, dtype=wl.dtype)
    out = BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T)
    torch.cuda.synchronize()
    print(name, "ok", float(out.sum_se[0]))
if which in ("all", "c128"):
    m = X.ChannelModel(S=2, K=96, p=1.0, r=0.5)
    H = X.generate_channels(m, seed=0, first=0, B=2, dtype=torch.complex128)
    out = BT.rzf_batched(H, 9.6, 10.0, T=3)
    torch.cuda.synchronize()
    print("c128 ok", float(out.sum_se[0]))
