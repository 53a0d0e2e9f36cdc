"""One forward per batch size (graphs off, synchronous launches) on a named config; prints progress."""
import os, sys
os.environ.setdefault("TQ_GRAPHS", "0")
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
L.reserve(64)
for B in [int(b) for b in sys.argv[2:]]:
    x = torch.from_numpy(np.random.default_rng(100 + B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
    for rep in range(3):
        y = L.forward(x)
        torch.cuda.synchronize()
    print(f"B={B} ok, |y| {float(y.abs().mean()):.4f}", flush=True)
