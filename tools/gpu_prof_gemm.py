"""Run a few forwards of one config/batch (for ncu --set full on the expert GEMM)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
name, B = sys.argv[1], int(sys.argv[2])
L = tq.Layer(synth.ensure_config(name))
L.reserve(B)
x = torch.randn(B, L.in_dim, device="cuda")
for _ in range(3):
    y = L.forward(x)
torch.cuda.synchronize()
print("ok")
