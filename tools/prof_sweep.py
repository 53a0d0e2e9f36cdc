"""Two forwards per batch size (graphs off) for ncu captures of the kernels."""
import os, sys
os.environ.setdefault("TQ_GRAPHS", "0")
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
name = sys.argv[1]
Bs = [int(b) for b in sys.argv[2:]]
L = tq.Layer(synth.ensure_config(name))
L.reserve(max(Bs))
for B in Bs:
    x = torch.from_numpy(np.random.default_rng(B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
    for _ in range(2):
        L.forward(x)
    torch.cuda.synchronize()
print("ok")
