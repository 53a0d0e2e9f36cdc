"""Time forward() under TQ_DEBUG variants (isolates GEMM pipeline stages)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
for B in [int(b) for b in sys.argv[2:]]:
    L.reserve(B)
    x = torch.randn(B, L.in_dim, device="cuda")
    y = torch.empty(B, L.out_dim, device="cuda")
    for _ in range(3): L.forward(x, out=y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); L.forward(x, out=y); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    print(f"TQ_DEBUG={os.environ.get('TQ_DEBUG','0')} B={B}: forward {np.median(ts)*1e3:.1f} us", flush=True)
