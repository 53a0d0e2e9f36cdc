"""Device time of the router kernel alone (Layer.route) per batch size."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1] if len(sys.argv) > 1 else "c2"))
for B in (1, 8, 64, 512, 4096):
    L.reserve(B)
    x = torch.randn(B, L.in_dim, device="cuda")
    for _ in range(3):
        L.route(x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); L.route(x); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"route B={B}: {np.median(ts) * 1e3:.1f} us", flush=True)
