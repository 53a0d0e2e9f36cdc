"""Full-forward device time per batch size (events around each forward, L2 flushed)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
name = sys.argv[1]
Bs = [int(b) for b in sys.argv[2:]] or [1, 2, 4, 8, 16, 32, 64]
L = tq.Layer(synth.ensure_config(name))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
L.reserve(max(Bs))
tot = 0.0
for B in Bs:
    x = torch.from_numpy(np.random.default_rng(B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
    y = torch.empty(B, L.out_dim, device="cuda")
    for _ in range(3):
        L.forward(x, out=y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); L.forward(x, out=y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    tot += ms
    print(f"graphs={os.environ.get('TQ_GRAPHS', '1')} {name} B={B}: forward {ms * 1e3:.1f} us", flush=True)
print(f"sweep total {tot * 1e3:.1f} us -> {sum(Bs) / tot * 1e3:.0f} tok/s")
L.close()
