"""The paper's layout bench (infer.cpp:345-426) on B200 and on the host CPU.

    python tools/layouts_bench.py [config] [--cpu] > layouts.csv

For each layout (fused_2d, shared_1d, element_wise, dequant_only) and batch
B, one call on the same synthetic tokens and the reference's routing is
timed REPEATS times after WARMUP calls with CUDA events on the launching
stream (synchronised on both sides; host-orchestrated layouts include their
launch overhead, as the reference's steady_clock brackets include its loops).
CSV columns follow the reference bench CLI (tileq_main.cpp:553-587):
device,layout,batch,median_ns,p10_ns,p90_ns,dispatch_count,launches.
--cpu adds the reference's own bench() (oracle/_ref, 1 thread) rows.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_09281_b200 as tq  # noqa: E402
from paper_2605_09281_b200 import synth  # noqa: E402

LAYOUTS = ("fused_2d", "shared_1d", "element_wise", "dequant_only")
BATCHES = [1, 2, 4, 8, 16, 32, 64]
REPEATS, WARMUP = 20, 3


def pct(v, p):
    v = sorted(v)
    return v[min(len(v) - 1, int(round(p / 100.0 * (len(v) - 1))))]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name = args[0] if args else "c2"
    art = synth.ensure_config(name)
    L = tq.Layer(art)
    L.reserve(max(BATCHES))
    for lay in LAYOUTS:
        L.layout_prepare(lay)
    print("device,layout,batch,median_ns,p10_ns,p90_ns,dispatch_count,launches")
    for B in BATCHES:
        x = torch.from_numpy(np.random.default_rng(B).standard_normal((B, L.in_dim), dtype=np.float32)).cuda()
        _, ids, gates = L.forward_routed(x)
        for lay in LAYOUTS:
            for _ in range(WARMUP):
                L.layout_forward(lay, x, ids, gates)
            torch.cuda.synchronize()
            ts = []
            for _ in range(REPEATS):
                L.reset_launch_count()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                _, disp = L.layout_forward(lay, x, ids, gates)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e6)
            print(f"b200,{lay},{B},{pct(ts, 50):.0f},{pct(ts, 10):.0f},{pct(ts, 90):.0f},{disp},{L.launch_count()}",
                  flush=True)
    if "--cpu" in sys.argv:
        from oracle.oracle import RefLib, ref_available
        if ref_available():
            R = RefLib().load(art)
            for lay in LAYOUTS:
                bs = BATCHES if lay != "dequant_only" else [1]
                rep = R.bench(lay, bs, repeats=5, warmup=1, seed=1)
                for B, (med, p10, p90, d) in rep.items():
                    print(f"cpu-ref-1t,{lay},{B},{med:.0f},{p10:.0f},{p90:.0f},{int(d)},0", flush=True)
    L.close()


if __name__ == "__main__":
    main()
