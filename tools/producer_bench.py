"""Time the GPU artifact-producer stages at the Mixtral (c2) expert
shape and the reference's CPU implementation on bounded samples.

    python tools/producer_bench.py [--rows 14336] [--dim 4096] [--tokens 512] [--cpu-rows 8]

GPU: CUDA events around each stage (best of 3 after a warm-up call) (estimate_hessian over `tokens` calibration
rows; spd_inverse; quantize_rtn; quantize_gptq = spd_inverse + grids + the
column sweep + RTN + two proxy losses; proxy_loss).  CPU: the reference
(oracle/_ref) on the same dim with `cpu-rows` residual rows, one thread, and
the per-row cost scaled to `rows` (the row loops are independent; spd_inverse
is paid once per call and reported separately).  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=14336)
    ap.add_argument("--dim", type=int, default=4096)
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--gs", type=int, default=128)
    ap.add_argument("--cpu-rows", type=int, default=8)
    ap.add_argument("--cpu-dim", type=int, default=0, help="dim of the CPU sample (default: --dim)")
    ap.add_argument("--cpu-rows2", type=int, default=0,
                    help="second GPTQ sample size: per-row cost = difference of the two runs (same spd_inverse)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sketch", default="43008x12288", help="sketch_lowrank shape (the c2 3x3 mosaic), '' to skip")
    ap.add_argument("--sketch-rank", type=int, default=32)
    ap.add_argument("--sketch-iters", type=int, default=4)
    a = ap.parse_args()
    import torch
    from paper_2605_09281_b200 import producer as P

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    calib = torch.randn((a.tokens, a.dim), device=dev, generator=g)
    r = torch.randn((a.rows, a.dim), device=dev, generator=g) * 0.02
    out = {"config": {"rows": a.rows, "dim": a.dim, "tokens": a.tokens, "bits": a.bits, "group_size": a.gs}}

    def timed(fn, reps=3):
        fn()   # warm-up (allocator, module load, clocks)
        torch.cuda.synchronize()
        best, res = float("inf"), None
        for _ in range(reps):   # best of `reps` (each call synchronizes where the API returns host values)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best, res

    t_h, hp = timed(lambda: P.estimate_hessian(calib, 0.01))
    t_inv, _ = timed(lambda: P.spd_inverse(hp))
    t_rtn, q_rtn = timed(lambda: P.quantize_rtn(r, a.bits, a.gs))
    t_gptq, q = timed(lambda: P.quantize_gptq(r, hp, a.bits, a.gs))
    t_proxy, loss = timed(lambda: P.proxy_loss(r, q, hp))
    gpu = {"estimate_hessian_ms": t_h, "spd_inverse_ms": t_inv, "quantize_rtn_ms": t_rtn,
           "quantize_gptq_ms": t_gptq, "proxy_loss_ms": t_proxy, "gptq_used_rtn": q.used_rtn,
           "proxy_loss": loss}
    # FP64 work per stage (mul + add or mul + div + sub counted as one element op)
    d, R, T = a.dim, a.rows, a.tokens
    gpu["proxy_loss_f64_macs"] = R * d * d + R * d
    gpu["proxy_loss_gmac_per_s"] = gpu["proxy_loss_f64_macs"] / (t_proxy * 1e6)
    gpu["gptq_sweep_updates"] = R * d * (d - 1) // 2
    if a.sketch:
        sr, sc = (int(v) for v in a.sketch.split("x"))
        wm = torch.randn((sr, sc), device=dev, generator=g)
        t_sk, f = timed(lambda: P.sketch_lowrank(wm, a.sketch_rank, a.sketch_iters, 7))
        passes = (2 * a.sketch_iters + 2) + 2   # mat-vecs + deflate (read + write) per triple
        gpu["sketch_lowrank_ms"] = t_sk
        gpu["sketch_shape"] = [sr, sc, a.sketch_rank, a.sketch_iters]
        gpu["sketch_gbs"] = a.sketch_rank * passes * sr * sc * 8 / (t_sk * 1e6)
    out["gpu"] = gpu

    if not a.no_cpu:
        from oracle.oracle import RefLib
        ref = RefLib()
        cd = a.cpu_dim or a.dim
        cn = a.cpu_rows
        rs = r[:cn, :cd].float().cpu().numpy()
        cs = calib[:, :cd].float().cpu().numpy()
        t0 = time.perf_counter()
        h_ref, _ = ref.estimate_hessian(cs, 0.01)
        t_h_cpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        c, s, z = ref.quantize("rtn", rs, None, a.bits, a.gs)
        t_rtn_cpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref.proxy_loss(rs, c, s, z, a.bits, a.gs, h_ref)
        t_proxy_cpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref.quantize("gptq", rs, h_ref, a.bits, a.gs)
        t_gptq_cpu = time.perf_counter() - t0
        # quantize_gptq = spd_inverse (once per call) + per-row work (sweep, RTN, two
        # proxy losses); spd_inverse alone is timed on the C restatement of the
        # same loops (oracle/tileq_oracle.c, quant.cpp:72-112, -O2 like the reference)
        from oracle.oracle import Oracle
        t0 = time.perf_counter()
        Oracle().spd_inverse(h_ref)
        t_inv_cpu = time.perf_counter() - t0
        scale = a.rows / cn
        if a.sketch:
            # one triple of the sketch on the full mosaic: every triple streams the
            # same working copy the same number of times, so rank x this is the stage
            t0 = time.perf_counter()
            ref.sketch_lowrank(wm.cpu().numpy(), 1, a.sketch_iters, 7)
            t_sk1 = time.perf_counter() - t0
        per_row = None
        if a.cpu_rows2 > cn:
            rs2 = r[:a.cpu_rows2, :cd].float().cpu().numpy()
            t0 = time.perf_counter()
            ref.quantize("gptq", rs2, h_ref, a.bits, a.gs)
            t_gptq2 = time.perf_counter() - t0
            per_row = (t_gptq2 - t_gptq_cpu) / (a.cpu_rows2 - cn)
        out["cpu_reference"] = {
            "threads": 1, "sample": f"{cn} residual rows x dim {cd}, {T} calibration tokens",
            "estimate_hessian_s": t_h_cpu, "proxy_loss_s_sample": t_proxy_cpu, "quantize_rtn_s_sample": t_rtn_cpu,
            "quantize_gptq_s_sample": t_gptq_cpu, "spd_inverse_s": t_inv_cpu,
            "proxy_loss_s_scaled_to_rows": t_proxy_cpu * scale,
            "quantize_gptq_per_row_s": per_row,
            "sketch_lowrank_rank1_s": t_sk1 if a.sketch else None,
            "sketch_lowrank_s_scaled_to_rank": t_sk1 * a.sketch_rank if a.sketch else None,
            "quantize_gptq_s_scaled_to_rows": (t_gptq_cpu + per_row * (a.rows - cn)
                                               if per_row is not None and cd == a.dim else None),
        }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
