"""One forward per batch size (for an ncu launch list)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
name = sys.argv[1]
Bs = [int(b) for b in sys.argv[2:]]
L = tq.Layer(synth.ensure_config(name))
for B in Bs:
    L.reserve(B)
    x = torch.randn(B, L.in_dim, device="cuda")
    for _ in range(2):
        y = L.forward(x)
    torch.cuda.synchronize()
print("done")
