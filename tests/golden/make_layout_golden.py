"""Golden outputs of the paper's bench layouts, written by the REFERENCE itself.

    make -C oracle ref && python tests/golden/make_layout_golden.py

For every committed golden artifact and the committed B=7 / B=33 inputs of
golden.npz, the unmodified reference library (oracle/_ref/libtileq_ref.so)
runs, on the reference's own routing of those inputs:
baseline_1d_forward on shared_1d_from_tiled_representative,
baseline_elementwise_forward on elementwise_factors_from_tiled
(infer.cpp:187-335) and lotile_forward (the fused 2D layout), recording the
outputs and dispatch_count() -- the contract the GPU ports are checked
against on the GPU box (which has no /root/reference).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle.oracle import RefLib  # noqa: E402

ARTS = ["folded_b3", "general_b2_shared", "scalar_b4_ragged", "general_b8"]


def main():
    ref = RefLib()
    gold = np.load(os.path.join(HERE, "golden.npz"))
    out = {}
    for name in ARTS:
        R = ref.load(os.path.join(HERE, name))
        for B in (7, 33):
            x = gold[f"{name}/x{B}"]
            ids, gates = gold[f"{name}/ids{B}"], gold[f"{name}/gates{B}"]
            for lay in ("fused_2d", "shared_1d", "element_wise"):
                y, d = R.layout(lay, x, ids, gates)
                out[f"{name}/{lay}{B}"] = y
                out[f"{name}/{lay}{B}_dispatches"] = np.array(d, np.int64)
            _, d = R.layout("dequant_only", x, ids, gates)
            out[f"{name}/dequant_only{B}_dispatches"] = np.array(d, np.int64)
    np.savez_compressed(os.path.join(HERE, "layouts.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
