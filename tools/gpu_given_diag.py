"""Given-routing forwards (device and host-ids entries) vs self-routed ones on tiny layers (diagnostic)."""
import sys, os, ctypes as C
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq
from oracle.oracle import RefLib
R = RefLib()
lib = tq.lib()
lib.tq_forward_host_ids.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
for bits in (2, 3, 4, 8, 3, 2):
    d = f"/tmp/given_b{bits}"
    R.make_artifact(d, K=6, top_k=2, i=64, o=48, S=1, r=8, bits=bits, g=32, calib="gauss", seed=130 + bits)
    L = tq.Layer(d)
    x = np.random.default_rng(1).standard_normal((5, 64)).astype(np.float32)
    yr, idr, gr = R.load(d).forward(x)
    for path, pi in (("qmoe", 1), ("full", 0), ("lotile", 2)):
        y1, ids, gates = L.forward_host(x, path=path, with_routing=True)
        xd = torch.from_numpy(x).cuda()
        y2 = L.forward(xd, torch.from_numpy(ids.astype(np.int32)).cuda(), torch.from_numpy(gates).cuda(), path=path).cpu().numpy()
        y3 = np.zeros_like(y1)
        ids64 = ids.astype(np.int64)
        tq.check(lib.tq_forward_host_ids(L._h, x.ctypes.data, 5, ids64.ctypes.data, gates.ctypes.data, y3.ctypes.data, pi))
        e = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
        extra = f" ref {e(y1, yr):.2e}" if path == "full" else ""
        print(f"bits {bits} {path:6s}: dev-given {e(y2, y1):.2e}  host-ids {e(y3, y1):.2e}{extra}")
