"""One routed forward of a named config at batch B (debug helper: CUDA_LAUNCH_BLOCKING=1
pins a failing launch), output checked for finiteness."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
for B in [int(b) for b in sys.argv[2:]]:
    L.reserve(B)
    x = torch.randn(B, L.in_dim, device="cuda")
    for it in range(3):
        y = L.forward(x)
        torch.cuda.synchronize()
    print(f"B={B} ok finite={bool(torch.isfinite(y).all())}", flush=True)
