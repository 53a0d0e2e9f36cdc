"""GPU parity at the BASELINE.json configuration shapes (VERDICT r1 missing item 4).

Synthetic artifacts of the named shapes in the reference wire format
(paper_2605_09281_b200.synth; the reference's own read_artifact accepts them,
tests/test_cpu_oracle.py), checked against the C restatement of route /
qmoe_forward / lotile_forward (oracle/tileq_oracle.c, pinned to the reference's
golden vectors in tests/test_cpu_oracle.py) on output row slices:

  * routing ids bit-exact and gates within 1 f32 ulp (moe.cpp:43-89),
  * layer output within the north_star 2e-3 relative Frobenius error,

for the decode configurations (B in {1, 8, 64}: the 3-launch decode path with
split segments, shared experts, 32- and 64-token tiles) and prefill-sized
batches (the grouped tcgen05 path), folded and general descale tiers.
"""
import os

import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(scope="module")
def tq():
    import paper_2605_09281_b200 as tq
    return tq


_ART = {}


def _artifact(name, tier):
    from oracle.oracle import read_artifact_np
    from paper_2605_09281_b200 import synth
    key = (name, tier)
    if key not in _ART:
        path = synth.ensure_config(name, tier=tier)
        _ART[key] = (path, read_artifact_np(path))
    return _ART[key]


_LAYERS = {}


def _layer(tq, name, tier):
    key = (name, tier)
    if key not in _LAYERS:
        path, _ = _artifact(name, tier)
        _LAYERS[key] = tq.Layer(path)
    return _LAYERS[key]


def _x(B, i, seed):
    return np.random.default_rng(seed).standard_normal((B, i), dtype=np.float32)


def _check(tq, oracle, name, tier, B, slices, seed=7):
    path, art = _artifact(name, tier)
    L = _layer(tq, name, tier)
    x = _x(B, art["i"], seed + B)
    y, ids, gates = L.forward_host(x, with_routing=True)
    idr, gr = oracle.route(x, art["gate"], art["top_k"])
    np.testing.assert_array_equal(ids, idr)
    np.testing.assert_array_max_ulp(gates, gr, maxulp=1)
    errs = []
    for r0, r1 in slices:
        yr, _, _ = oracle.tileq_forward(art, x, r0, r1)
        e = rel_frob(y[:, r0:r1], yr)
        errs.append(e)
        assert e <= TOL, (name, tier, B, (r0, r1), e)
    print(f"\n{name}/{tier} B={B}: rel_frob {' '.join(f'{e:.2e}' for e in errs)} (rows {slices})")
    return errs


# (config, tier, batches, row slices) -- slices cover the first and the last m-blocks
DECODE = [
    ("c2", "folded", [1, 8, 64], [(0, 256), (14336 - 256, 14336)]),
    ("c2", "general", [1, 64], [(0, 128), (14336 - 128, 14336)]),
    ("c4", "folded", [1, 8, 64], [(0, 256), (1408 - 256, 1408)]),
    ("c4", "general", [8], [(0, 1408)]),
    ("c5", "folded", [1, 8, 64], [(0, 256), (1408 - 256, 1408)]),
    ("c1", "general", [1, 17, 64, 200], [(0, 2816)]),
    ("c2", "folded", [256], [(14336 - 128, 14336)]),
]


@pytest.mark.parametrize("case", DECODE, ids=lambda c: f"{c[0]}-{c[1]}")
def test_decode_shapes_match_oracle(tq, oracle, case):
    name, tier, batches, slices = case
    for B in batches:
        _check(tq, oracle, name, tier, B, slices)


PREFILL = [
    ("c2", "folded", 1024, [(14336 - 128, 14336)]),
    ("c2", "general", 600, [(0, 128)]),
    ("c4", "folded", 700, [(0, 256)]),
    ("c4", "general", 700, [(0, 256)]),
    ("c5", "general", 700, [(0, 256)]),
    ("c5", "folded", 2000, [(0, 128)]),
    ("c1", "folded", 700, [(0, 512)]),
]


@pytest.mark.parametrize("case", PREFILL, ids=lambda c: f"{c[0]}-{c[1]}")
def test_prefill_shapes_match_oracle(tq, oracle, case):
    name, tier, B, slices = case
    _check(tq, oracle, name, tier, B, slices)


def test_decode_stress_c2(tq):
    """>= 5000 c2-shape forwards over B = 1..256 (every decode tile / split shape)
    on all three paths (tileq / qmoe / lotile, infer.cpp:40-185) plus prefill
    4096: no device fault; a batch whose experts fit one 64-token tile (B <= 64)
    reproduces its first output bit for bit (fixed reduction orders), larger
    ones within float rounding (an expert's slots may then straddle two tiles
    in the router's atomic slot order, changing the split-segment rounding)."""
    import torch
    path, art = _artifact("c2", "folded")
    L = _layer(tq, "c2", "folded")
    batches = [1, 2, 3, 4, 5, 7, 8, 12, 16, 24, 31, 32, 33, 48, 63, 64, 65, 100, 128, 200, 256]
    xs = {B: torch.from_numpy(_x(B, art["i"], 1000 + B)).cuda() for B in batches}
    paths = ("full", "qmoe", "lotile")
    ref = {(B, p): L.forward(xs[B], path=p).clone() for B in batches for p in paths}

    def same(y, r, B):
        if B <= 64:
            return torch.equal(y, r)
        return float((y - r).abs().max()) <= 1e-5 * float(r.abs().max())

    n = 0
    reps = int(os.environ.get("TQ_STRESS_REPS", "240"))
    for rep in range(reps):
        for B in batches:
            p = paths[(rep + B) % 3]
            y = L.forward(xs[B], path=p)
            n += 1
            if rep % 25 == 0:
                torch.cuda.synchronize()
                assert same(y, ref[(B, p)], B), (rep, B, p)
    torch.cuda.synchronize()
    for B in batches:
        for p in paths:
            assert same(L.forward(xs[B], path=p), ref[(B, p)], B), (B, p)
    assert n >= 5000
    xp = torch.from_numpy(_x(4096, art["i"], 5)).cuda()
    yp = L.forward(xp).clone()
    for _ in range(10):
        assert torch.equal(L.forward(xp), yp)
    assert L.sync() is None
    print(f"\nstress: {n} decode forwards + 10 prefill forwards, no fault")
