"""Forward device time under three cache regimes: L2 flushed between forwards,
no flush (same layer re-run: weights partly L2 resident), and R distinct layer
replicas run round-robin (weights of the step always cold, code/tables warm)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
name = sys.argv[1]
Bs = [int(b) for b in sys.argv[2:]] or [1, 8, 64]
R = int(os.environ.get("REPLICAS", "4"))
Ls = [tq.Layer(synth.ensure_config(name)) for _ in range(R)]
for L in Ls:
    L.reserve(max(Bs))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for B in Bs:
    x = torch.from_numpy(np.random.default_rng(B).standard_normal((B, Ls[0].in_dim), dtype=np.float32)).cuda()
    y = torch.empty(B, Ls[0].out_dim, device="cuda")
    for L in Ls:
        for _ in range(3):
            L.forward(x, out=y)
    torch.cuda.synchronize()
    for mode in ("flush", "none", "replicas"):
        ts = []
        for it in range(40):
            L = Ls[it % R] if mode == "replicas" else Ls[0]
            if mode == "flush":
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); L.forward(x, out=y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        print(f"{name} B={B} {mode}: {np.median(ts) * 1e3:.1f} us", flush=True)
