"""Decode forwards over many batch sizes / paths, then prefill forwards (the stress test's sequence)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config("c2"))
batches = [int(b) for b in os.environ.get("SR_B", "1 8 64 65 128 256").split()]
paths = os.environ.get("SR_PATHS", "full qmoe lotile").split()
reps = int(os.environ.get("SR_REPS", "3"))
xs = {B: torch.from_numpy(np.random.default_rng(1000 + B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda() for B in batches}
for rep in range(reps):
    for B in batches:
        for p in paths:
            L.forward(xs[B], path=p)
torch.cuda.synchronize()
print("decode ok", flush=True)
xp = torch.from_numpy(np.random.default_rng(5).standard_normal((int(os.environ.get("SR_P", "4096")), L.in_dim), dtype=np.float32)).cuda()
for i in range(int(os.environ.get("SR_PN", "4"))):
    y = L.forward(xp)
    torch.cuda.synchronize()
    if i % 10 == 9 or i == int(os.environ.get("SR_PN", "4")) - 1: print(f"prefill {i} ok", flush=True)
