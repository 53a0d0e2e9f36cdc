"""Routing vs oracle on a layer created after the device memory was filled with garbage (diagnostic)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from paper_2605_09281_b200 import synth
from oracle.oracle import Oracle, read_artifact_np
name, tier, B, reps = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
path = synth.ensure_config(name, tier=tier)
art = read_artifact_np(path)
# poison: fill a large chunk of device memory with NaN bit patterns, then free it
g = torch.full((4 << 28,), float("nan"), device="cuda")
del g
torch.cuda.synchronize()
torch.cuda.empty_cache()
L = tq.Layer(path)
x = np.random.default_rng(7 + B).standard_normal((B, art["i"]), dtype=np.float32)
idr, gr = Oracle().route(x, art["gate"], art["top_k"])
bad = 0
for rep in range(reps):
    y, ids, gates = L.forward_host(x, with_routing=True)
    d = np.argwhere(np.abs(gates.view(np.int32).astype(np.int64) - gr.view(np.int32).astype(np.int64)) > 1)
    di = np.argwhere(ids != idr)
    if len(d) or len(di):
        bad += 1
        rows = sorted(set(int(r) for r, _ in d))
        print(f"rep {rep}: {len(d)} gate mismatches in {len(rows)} tokens, {len(di)} id mismatches; first tokens {rows[:8]}")
        for r in rows[:3]:
            print("   tok", r, "ids", ids[r], idr[r], "gates", gates[r], gr[r])
print(f"poisoned {name}/{tier} B={B}: {bad}/{reps} bad reps")
