"""Repeat forwards of one batch size and report bitwise / max differences vs the first output."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
for B in [int(b) for b in sys.argv[2:]]:
    x = torch.from_numpy(np.random.default_rng(1000 + B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
    ref = L.forward(x).clone()
    bad = 0
    worst = 0.0
    rows = set()
    for rep in range(50):
        y = L.forward(x)
        d = (y - ref).abs()
        if d.max().item() > 0:
            bad += 1
            worst = max(worst, d.max().item() / ref.abs().max().item())
            rows |= set(torch.nonzero(d.amax(1) > 0).flatten().tolist()[:5])
    print(f"B={B}: {bad}/50 reps differ, worst rel {worst:.2e}, tokens {sorted(rows)[:10]}", flush=True)
