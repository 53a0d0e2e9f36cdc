"""Forward sequence on one layer: python tools/gpu_mix.py <config> B1 B2 ... (graphs on unless TQ_GRAPHS=0)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
for B in [int(b) for b in sys.argv[2:]]:
    x = torch.from_numpy(np.random.default_rng(B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
    y = L.forward(x)
    torch.cuda.synchronize()
    print(f"B={B} ok {float(y.abs().mean()):.4f}", flush=True)
