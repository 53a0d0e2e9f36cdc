"""A few router launches at one batch size (for ncu)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config("c2"))
B = int(sys.argv[1])
L.reserve(B)
x = torch.randn(B, L.in_dim, device="cuda")
for _ in range(3):
    L.route(x)
torch.cuda.synchronize()
print("ok")
