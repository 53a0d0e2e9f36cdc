"""Each forward path of a named config at a few batch sizes (debug helper)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
for path in sys.argv[2].split(","):
    for B in [int(b) for b in sys.argv[3:]]:
        L.reserve(B)
        x = torch.randn(B, L.in_dim, device="cuda")
        y = L.forward(x, path=path)
        torch.cuda.synchronize()
        print(f"{path} B={B} ok finite={bool(torch.isfinite(y).all())}", flush=True)
