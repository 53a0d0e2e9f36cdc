"""Per-launch device time of a forward (TQ_KTIME=1): 30 forwards enqueued back to
back (host far ahead of the GPU, so event gaps are device time), L2 flushed
between forwards."""
import os, sys
os.environ["TQ_KTIME"] = "1"
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
B = int(sys.argv[2])
L.reserve(B)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
x = torch.from_numpy(np.random.default_rng(B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
y = torch.empty(B, L.out_dim, device="cuda")
for _ in range(3):
    L.forward(x, out=y)
torch.cuda.synchronize()
# a long kernel first so the host runs ahead
torch.cuda._sleep(20_000_000)
for _ in range(30):
    flush.zero_()
    L.forward(x, out=y)
torch.cuda.synchronize()
L.close()
