"""After every decode forward: the self-resetting counters (slot counts, router
tickets, split-segment arrivals) must be back to zero (diagnostic)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config("c2", tier="folded"))
n = L.num_experts + 256 + (L.num_experts + L.num_shared) * ((L.out_dim + 127) // 128)
buf = np.zeros(n, np.int32)
batches = [int(b) for b in os.environ.get("SCAN_BATCHES", "12,16,24,31,32").split(",")]
path = os.environ.get("SCAN_PATH", "full")
xs = {B: torch.from_numpy(np.random.default_rng(1000 + B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
      for B in batches}
for rep in range(int(os.environ.get("SCAN_REPS", "4"))):
    for B in batches:
        L.forward(xs[B], path=path)
        tq.check(tq.lib().tq_debug_decode_counters(L._h, buf.ctypes.data, n))
        K = L.num_experts
        cnt, tick, seg = buf[:K], buf[K:K + 256], buf[K + 256:]
        if cnt.any() or tick.any() or seg.any():
            print(f"rep {rep} B={B}: cnt {np.nonzero(cnt)[0][:8]} tickets {np.nonzero(tick)[0][:8]} "
                  f"(vals {tick[tick != 0][:8]}) segcnt {np.nonzero(seg)[0][:8]} (vals {seg[seg != 0][:8]})", flush=True)
print("done", flush=True)
