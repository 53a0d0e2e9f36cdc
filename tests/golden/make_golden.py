"""Regenerate the committed golden fixtures from the REFERENCE itself.

    make -C oracle ref && python tests/golden/make_golden.py

Every expected value here is produced by the unmodified reference library
(oracle/_ref/libtileq_ref.so compiled from /root/reference/proj/src): its
quantization pipeline writes the artifacts (pipeline.cpp quantize_moe stages
+ io.cpp write_artifact), and its route / qmoe_forward / lotile_forward /
tileq_forward / pack_codes produce the outputs.  The fixtures travel to the
GPU box (which has no /root/reference), so the GPU tests can check the engine
against the reference there, and the CPU tests pin our C restatement
(oracle/tileq_oracle.c) against them here.
"""
from __future__ import annotations

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle.oracle import RefLib  # noqa: E402

# small artifacts covering the tiers, widths, shared experts and ragged dims
ARTIFACTS = {
    "folded_b3": dict(K=4, top_k=2, i=256, o=96, r=8, bits=3, g=128, calib="signs", seed=21),
    "general_b2_shared": dict(K=6, top_k=3, i=256, o=80, S=1, r=8, bits=2, g=128, calib="gauss", seed=22),
    "scalar_b4_ragged": dict(K=5, top_k=2, i=192, o=72, r=4, bits=4, g=64, calib="none", noise=0.0, seed=23),
    "general_b8": dict(K=3, top_k=1, i=128, o=40, r=4, bits=8, g=32, calib="gauss", seed=24),
}
BATCHES = (1, 7, 33)


def main():
    ref = RefLib()
    out = {}
    for name, spec in ARTIFACTS.items():
        d = os.path.join(HERE, name)
        if os.path.exists(d):
            shutil.rmtree(d)
        ref.make_artifact(d, **spec)
        R = ref.load(d)
        for B in BATCHES:
            x = np.random.default_rng(1000 + B).standard_normal((B, R.i)).astype(np.float32)
            out[f"{name}/x{B}"] = x
            for mode, tag in ((0, "tileq"), (1, "qmoe"), (2, "lotile")):
                y, ids, gates = R.forward(x, mode=mode)
                out[f"{name}/{tag}{B}"] = y
            out[f"{name}/ids{B}"] = ids
            out[f"{name}/gates{B}"] = gates
        for e in range(R.K + R.S):
            if e < 2:
                out[f"{name}/dequant{e}"] = R.dequantize(e)
    # routing known answers (moe.cpp:43-89), incl. forced underflow ties
    rng = np.random.default_rng(11)
    for t, (B, i, K, k, scale) in enumerate([(33, 10, 7, 1, 1.0), (33, 10, 7, 3, 1.0), (33, 10, 7, 7, 1.0),
                                             (64, 64, 8, 2, 100.0), (5, 3, 4, 4, 30.0)]):
        x = (rng.standard_normal((B, i)) * scale).astype(np.float32)
        g = rng.standard_normal((K, i)).astype(np.float32)
        ids, gates = ref.route(x, g, k)
        out[f"route{t}/x"], out[f"route{t}/g"] = x, g
        out[f"route{t}/ids"], out[f"route{t}/gates"] = ids, gates
    # codec known answers (codec.cpp:150-195)
    for bits in (2, 3, 4, 8):
        for count in (1, 5, 7, 64, 129, 1000):
            codes = rng.integers(0, 1 << bits, size=count).astype(np.uint32)
            out[f"pack{bits}_{count}/codes"] = codes
            out[f"pack{bits}_{count}/bytes"] = ref.pack(codes, bits)
    halves = np.arange(1 << 16, dtype=np.uint16)
    out["f16/decode"] = ref.f16_to_f32(halves)
    vals = np.concatenate([rng.standard_normal(4096).astype(np.float32) * 10.0 ** rng.integers(-8, 5, 4096),
                           np.array([65520.0, 65519.996, 1e30, -1e30, 2.0 ** -25, 2.0 ** -24 * 1.5], np.float32)])
    out["f16/encode_in"] = vals.astype(np.float32)
    out["f16/encode_out"] = ref.f32_to_f16(vals.astype(np.float32))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
