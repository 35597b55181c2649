import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_13925_b200 as X
from paper_2305_13925_b200 import batched as BT
K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B = int(sys.argv[3]) if len(sys.argv) > 3 else 2
m = X.ChannelModel(S=S, K=K, p=0.4, r=0.7)
H = X.generate_channels(m, seed=3, first=0, B=B, dtype=torch.complex64)
torch.cuda.synchronize()
f = BT.rzf_batched(H, K / 10.0, 10.0, T=4, check=False)
torch.cuda.synchronize()
st = f.status.cpu(); print("status nonzero", int((st != 0).sum()), "sumse mean", float(f.sum_se.mean()))
