"""Expert-GEMM device time (CUDA events around the launch) per batch size; L2 flushed."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
name = sys.argv[1]
Bs = [int(b) for b in sys.argv[2:]] or [1, 8, 64]
L = tq.Layer(synth.ensure_config(name))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tag = os.environ.get("TQ_DEBUG", "0")
for B in Bs:
    L.reserve(B)
    x = torch.randn(B, L.in_dim, device="cuda")
    y = torch.empty(B, L.out_dim, device="cuda")
    for _ in range(3):
        L.forward(x, out=y)
    torch.cuda.synchronize()
    L.gemm_timing(True)
    for _ in range(20):
        flush.zero_()
        L.forward(x, out=y)
    torch.cuda.synchronize()
    ms, n = L.gemm_time()
    L.gemm_timing(False)
    print(f"dbg={tag} {name} B={B}: gemm {ms / n * 1e3:.1f} us", flush=True)
