"""The decode stress pattern of tests/test_gpu_shapes.py::test_decode_stress_c2 with
knobs to narrow a fault down (diagnostic): SCAN_PATHS, SCAN_BATCHES, SCAN_REPS."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config("c2", tier="folded"))
batches = [int(b) for b in os.environ.get("SCAN_BATCHES", "1,2,3,4,5,7,8,12,16,24,31,32,33,48,63,64,65,100,128,200,256").split(",")]
paths = tuple(os.environ.get("SCAN_PATHS", "full,qmoe,lotile").split(","))
reps = int(os.environ.get("SCAN_REPS", "30"))
xs = {B: torch.from_numpy(np.random.default_rng(1000 + B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
      for B in batches}
ref = {(B, p): L.forward(xs[B], path=p).clone() for B in batches for p in paths}
torch.cuda.synchronize()
print("ref ok", flush=True)
bad = 0
for rep in range(reps):
    for B in batches:
        p = paths[(rep + B) % len(paths)]
        y = L.forward(xs[B], path=p)
        if rep % 5 == 0:
            torch.cuda.synchronize()
            if not torch.equal(y, ref[(B, p)]):
                d = (y - ref[(B, p)]).abs()
                bad += 1
                if bad < 6:
                    print(f"rep {rep} B={B} {p}: max diff {float(d.max()):.3e} in {int((d > 0).sum())} elems, rows {sorted(set((d > 0).nonzero()[:, 0].tolist()))[:8]}", flush=True)
    torch.cuda.synchronize()
print(f"done, {bad} mismatches", flush=True)
