"""Quick fused-kernel vs general-path / oracle check (development tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_13925_b200 as X
from paper_2305_13925_b200 import batched as BT, _lib as L
from oracle import xlmimo_oracle as O

def relf(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
lib = L.lib()
for (S, K) in [(16, 64), (4, 32), (4, 16)]:
    m = X.ChannelModel(S=S, K=K, p=0.4, r=0.7)
    B = 8
    H = X.generate_channels(m, seed=3, first=0, B=B, dtype=torch.complex64)
    alpha, power = K / 10.0, 10.0
    print("shape", S * 64, K, "tc:", X.uses_tensor_cores(torch.complex64, "jacpcg", S * 64, K), flush=True)
    Adbg = torch.zeros(B, K, K, dtype=torch.complex64, device="cuda")
    lib.xl_debug_set_gram_out(Adbg.data_ptr())
    t0 = time.time()
    f = BT.rzf_batched(H, alpha, power, T=4, want_X=True, check=False)
    torch.cuda.synchronize()
    lib.xl_debug_set_gram_out(None)
    print("  fused done in %.3fs status" % (time.time() - t0), f.status.cpu().tolist(), flush=True)
    g = BT.rzf_batched(H, alpha, power, T=4, want_X=True, check=False, general=True)
    Ag = BT.gram_batched(H, alpha)
    torch.cuda.synchronize()
    print("  gram rel err", relf(Adbg.cpu().numpy(), Ag.cpu().numpy()))
    print("  X rel err", relf(f.X.cpu().numpy(), g.X.cpu().numpy()))
    print("  beta", f.beta.cpu().numpy()[:3], g.beta.cpu().numpy()[:3])
    print("  W rel err", relf(f.W.cpu().numpy(), g.W.cpu().numpy()))
    print("  sumse", f.sum_se.cpu().numpy()[:3], g.sum_se.cpu().numpy()[:3])
    Hn = H.cpu().numpy().astype(np.complex128)
    for b in range(2):
        Gr, beta, gam, s = O.precoder_and_se(Hn[b], alpha, power, 1.0, "jacpcg", 4, "textbook")
        print("  oracle b=%d W err %.2e SE err %.2e" % (b, relf(f.W[b].cpu().numpy(), Gr), abs(float(f.sum_se[b]) - s) / s))
