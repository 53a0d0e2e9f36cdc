"""Run forwards with TQ_DEBUG=8 and save CTA-0 pipeline traces (last expert GEMM launch)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
for B in [int(b) for b in sys.argv[2:]]:
    L.reserve(B)
    x = torch.randn(B, L.in_dim, device="cuda")
    os.environ["TQ_TRACE_FILE"] = f"gpurun_out/trace_B{B}{os.environ.get('TRACE_TAG', '')}.bin"
    for _ in range(3):
        L.forward(x)
    torch.cuda.synchronize()
print("ok")
