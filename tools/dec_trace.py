"""Decode GEMM event trace (TQ_DEC_TRACE builds): run forwards at the given batch
sizes with graphs off and print per-step timelines of one CTA.
    TQ_LIB_PATH=...tq_dec_trace.so python tools/dec_trace.py c2 1 64 [cta]"""
import os, sys
os.environ["TQ_GRAPHS"] = "0"
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
name = sys.argv[1]
Bs = [int(b) for b in sys.argv[2:4]]
cta = sys.argv[4] if len(sys.argv) > 4 else "0"
os.environ["TQ_DEC_TRACE_CTA"] = cta
L = tq.Layer(synth.ensure_config(name))
names = ["code_iss", "x_iss", "dq_data", "dq_done", "mma_a", "mma_x", "commit0", "epi_part", "dq_afree", "commit3"]
for B in Bs:
    x = torch.randn(B, L.in_dim, device="cuda")
    for _ in range(3):
        L.forward(x)
    torch.cuda.synchronize()
    f = f"/tmp/dec_trace_{B}.bin"
    if os.path.exists(f):
        os.remove(f)
    os.environ["TQ_DEC_TRACE_FILE"] = f
    L.forward(x)
    torch.cuda.synchronize()
    del os.environ["TQ_DEC_TRACE_FILE"]
    raw = np.fromfile(f, dtype=np.uint64).reshape(-1, 16 * 1024)[-1].astype(np.int64)
    t = raw[:10240].reshape(10, 1024)
    ct = raw[12288:12288 + 148 * 4].reshape(148, 4)
    ok = ct[:, 0] > 0
    base = ct[ok, 0].min()
    rel = (ct[ok] - base) / 1000.0
    print(f"B={B} per-CTA (us from first entry): entry max {rel[:, 0].max():.1f}, prologue done med {np.median(rel[:, 1]):.1f} "
          f"max {rel[:, 1].max():.1f}, roles done med {np.median(rel[:, 2]):.1f} min {rel[:, 2].min():.1f} max {rel[:, 2].max():.1f}")
    print("  roles-done per CTA (us):", " ".join(f"{v:.0f}" for v in rel[:, 2]))
    valid = t[0] > 0
    n = int(valid.sum())
    t0 = t[t > 0].min()
    print(f"B={B} cta {cta}: {n} steps, span {(t[t > 0].max() - t0)} cycles")
    print("step " + " ".join(f"{s:>10}" for s in names))
    for j in range(min(n, 80)):
        print(f"{j:4d} " + " ".join(f"{(t[s, j] - t0) if t[s, j] else -1:10d}" for s in range(10)))
