"""Expert-GEMM time after a write-flush vs a read-flush of L2 (dirty-line write-back effect)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config("c2"))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, device="cuda")
for B in (1, 8, 64):
    L.reserve(B)
    x = torch.randn(B, L.in_dim, device="cuda")
    y = torch.empty(B, L.out_dim, device="cuda")
    for mode in ("write", "read", "none"):
        for _ in range(3):
            L.forward(x, out=y)
        torch.cuda.synchronize()
        L.gemm_timing(True)
        for _ in range(20):
            if mode == "write":
                flush.zero_()
            elif mode == "read":
                sink += flush.view(torch.int32).sum(dtype=torch.int64).float()
            L.forward(x, out=y)
        torch.cuda.synchronize()
        ms, n = L.gemm_time()
        L.gemm_timing(False)
        print(f"B={B} flush={mode}: gemm {ms / n * 1e3:.1f} us", flush=True)
