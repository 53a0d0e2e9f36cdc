"""Artifact load time at a BASELINE shape: the engine's
tq_layer_load (parallel blob reads + CRC32 + unpack on host threads, repack,
upload, graph-free) against the reference's read_artifact (io.cpp:679-813, one
thread) on the same directory, page cache warm for both.

    python tools/load_bench.py [--config c2] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2605_09281_b200 as tq
    from paper_2605_09281_b200 import synth
    path = synth.ensure_config(a.config)
    nbytes = sum(os.path.getsize(os.path.join(path, f)) for f in os.listdir(path))
    torch.cuda.init()
    tq.Layer(path)   # warm: page cache, CUDA context, module load
    times = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L = tq.Layer(path)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        del L
    out = {"config": a.config, "artifact_bytes": nbytes, "engine_load_s": min(times),
           "engine_gbs": nbytes / min(times) / 1e9, "engine_threads": min(16, os.cpu_count() or 1)}
    if not a.no_ref:
        from oracle.oracle import RefLib
        ref = RefLib()
        ref.load(path)
        t0 = time.perf_counter()
        ref.load(path)
        out["reference_read_artifact_s"] = time.perf_counter() - t0
        out["reference_gbs"] = nbytes / out["reference_read_artifact_s"] / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
