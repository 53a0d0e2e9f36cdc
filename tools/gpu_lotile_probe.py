"""Probe the lotile-only path on synthetic shapes (units per CTA, ext width)."""
import os, sys, tempfile
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
d = tempfile.mkdtemp()
for (o, i, r, B) in [(128 * 148, 256, 8, 1), (128 * 300, 256, 8, 1), (128 * 300, 256, 32, 1), (128 * 300, 4096, 32, 1), (128 * 112, 4096, 32, 1)]:
    art = synth.write_synthetic(os.path.join(d, f"a{o}_{i}_{r}"), K=8, top_k=2, i=i, o=o, S=0, bits=3, r=r, group=128,
                                tier="folded", seed=3)
    L = tq.Layer(art)
    L.reserve(B)
    x = torch.randn(B, i, device="cuda")
    try:
        y = L.forward(x, path="lotile")
        torch.cuda.synchronize()
        print(f"o={o} i={i} r={r} B={B}: ok", flush=True)
    except Exception as e:
        print(f"o={o} i={i} r={r} B={B}: FAIL {e}", flush=True)
        break
    L.close()
