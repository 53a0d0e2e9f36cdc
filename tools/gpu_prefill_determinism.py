"""Grouped (prefill) path run-to-run reproducibility: 20 forwards of 300 / 1000 / 4096
tokens on the c2 layer must be bitwise identical."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config("c2", tier="folded"))
for B in (300, 1000, 4096):
    x = torch.from_numpy(np.random.default_rng(B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
    y0 = L.forward(x).clone()
    same = all(torch.equal(L.forward(x), y0) for _ in range(20))
    print(B, "bitwise reproducible over 20 runs:", same, flush=True)
