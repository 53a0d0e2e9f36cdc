"""First-light check on a B200: small reference artifact, engine vs reference."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import RefLib
import paper_2605_09281_b200 as tq

ref = RefLib()
for spec in [dict(K=4, top_k=2, i=256, o=256, r=8, bits=3, g=128, calib="signs", seed=1),
             dict(K=8, top_k=2, i=512, o=640, r=16, bits=3, g=128, calib="gauss", seed=2)]:
    d = f"/tmp/first_{spec['K']}_{spec['calib']}"
    ref.make_artifact(d, **spec)
    t = time.time()
    L = tq.Layer(d)
    print("load", time.time() - t, L.info, flush=True)
    R = ref.load(d)
    for B in (1, 5, 40):
        x = np.random.default_rng(B).standard_normal((B, spec["i"])).astype(np.float32)
        for path, mode in (("qmoe", 1), ("lotile", 2), ("full", 0)):
            y, ids, g = L.forward_host(x, path=path, with_routing=True)
            yr, idr, gr = R.forward(x, mode=mode)
            err = np.linalg.norm(y - yr) / max(np.linalg.norm(yr), 1e-30)
            print(f"B={B} {path}: ids_equal={bool((ids == idr).all())} gates_maxdiff={np.abs(g - gr).max():.3g} "
                  f"rel_frob={err:.3g} |y|={np.linalg.norm(yr):.3g}", flush=True)
