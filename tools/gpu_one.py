"""One forward of a synthetic config (graphs off) -- localise faults with CUDA_LAUNCH_BLOCKING=1.
    python tools/gpu_one.py <config> <tier> <B>"""
import os, sys
os.environ.setdefault("TQ_GRAPHS", "0")
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
name, tier, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
L = tq.Layer(synth.ensure_config(name, tier=tier))
x = np.random.default_rng(B).standard_normal((B, L.in_dim), dtype=np.float32)
y = L.forward_host(x)
print("ok", float(np.abs(y).mean()))
