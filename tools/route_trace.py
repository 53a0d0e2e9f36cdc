"""dec_route_kernel phase timeline (TQ_ROUTE_TRACE builds):
    TQ_LIB_PATH=...tq_route_trace.so python tools/route_trace.py c2 1"""
import os, sys
os.environ["TQ_GRAPHS"] = "0"
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
L = tq.Layer(synth.ensure_config(sys.argv[1]))
for B in [int(b) for b in sys.argv[2:]]:
    x = torch.randn(B, L.in_dim, device="cuda")
    for _ in range(3):
        L.forward(x)
    torch.cuda.synchronize()
    f = f"/tmp/route_trace_{B}.bin"
    if os.path.exists(f):
        os.remove(f)
    os.environ["TQ_ROUTE_TRACE_FILE"] = f
    L.forward(x)
    torch.cuda.synchronize()
    del os.environ["TQ_ROUTE_TRACE_FILE"]
    t = np.fromfile(f, dtype=np.uint64).reshape(-1, 64 * 128, 16)[-1].astype(np.int64)
    used = t[:, 0] > 0
    t0 = t[used, 0].min()
    print(f"B={B}: {used.sum()} CTAs; phases (us after first entry): 0 entry 1 work done 2 last-CTA 3 picked+x 4 dests 5 lowrank 6 sx 7 x16 8 end 9-10 proj 11 pick(w0) 12 x pass(w1)")
    for c in np.nonzero(used)[0][:24]:
        print(f"  cta {c:4d}: " + " ".join(f"{(v - t0) / 1000:7.2f}" if v else "      -" for v in t[c, :13]))
