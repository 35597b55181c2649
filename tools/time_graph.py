"""Direct rzf_batched calls vs GraphedRzf replay (device time per call, and
host wall time per call) for small batches.  Development aid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_13925_b200 as X
from paper_2305_13925_b200 import batched as BT
for cfg, B in (("cfg1", 100), ("cfg2", 256), ("cfg3", 148)):
    wl = X.CONFIGS[cfg]
    H = X.generate_channels(wl.model, seed=0, first=0, B=B, dtype=wl.dtype)
    out = BT.alloc_outputs(H)
    f = lambda: BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T, out=out, check=False)
    g = BT.GraphedRzf(B, wl.M, wl.K, wl.dtype, wl.alpha(), wl.power(), T=wl.T)
    res = {}
    for name, fn in (("direct", f), ("graph", lambda: g.run(H, check=False))):
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0) / 200 * 1e6
    print(f"{cfg} B={B}: direct {res['direct']:.1f} us/call ({B / res['direct']:.2f} M/s), "
          f"graph {res['graph']:.1f} us/call ({B / res['graph']:.2f} M/s)", flush=True)
