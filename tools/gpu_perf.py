"""Quick timing of the engine on BASELINE shapes (synthetic artifacts)."""
import os, sys, time, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth

def bench(L, B, iters=20, path="full"):
    x = torch.randn(B, L.in_dim, device="cuda")
    y = torch.empty(B, L.out_dim, device="cuda")
    L.reserve(B)
    for _ in range(3):
        L.forward(x, out=y, path=path)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); L.forward(x, out=y, path=path); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))

cfgs = sys.argv[1:] or ["c2"]
for name in cfgs:
    t = time.time(); d = synth.ensure_config(name); L = tq.Layer(d); print(name, "load", round(time.time() - t, 2), "s", flush=True)
    for B in (1, 4, 16, 64, 256, 1024, 4096):
        ms = bench(L, B)
        print(f"{name} B={B}: {ms*1e3:.1f} us  {B/ms*1e3:.0f} tok/s", flush=True)
