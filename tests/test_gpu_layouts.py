"""GPU ports of the paper's bench layouts against the
reference's own outputs (tests/golden/layouts.npz, written by
tests/golden/make_layout_golden.py from the unmodified reference library):

* element_wise  == baseline_elementwise_forward(elementwise_factors_from_tiled)  (infer.cpp:187-225, 271-289)
* shared_1d     == baseline_1d_forward(shared_1d_from_tiled_representative)      (infer.cpp:227-269, 320-335)
* fused_2d      == lotile_forward through the engine's fused path               (infer.cpp:53-180)
* dequant_only  == dequantize() of every expert (golden.npz dequant0/1)          (quant.cpp:285-323)

plus the dispatch-count contract of each layout (reference dispatch_count()).
Tolerances: the f32 GPU ports vs the f64 reference 1e-4 relative Frobenius;
the fused path and fp16 weights the north_star 2e-3.
"""
import os

import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ARTS = ["folded_b3", "general_b2_shared", "scalar_b4_ragged", "general_b8"]


@pytest.fixture(scope="module")
def tq():
    import paper_2605_09281_b200 as tq
    return tq


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(GOLD, "golden.npz")))


@pytest.fixture(scope="module")
def lay():
    return dict(np.load(os.path.join(GOLD, "layouts.npz")))


@pytest.mark.parametrize("name", ARTS)
def test_layouts_match_reference(tq, gold, lay, name):
    import torch
    L = tq.Layer(os.path.join(GOLD, name))
    for B in (7, 33):
        x = torch.from_numpy(gold[f"{name}/x{B}"]).cuda()
        ids = torch.from_numpy(gold[f"{name}/ids{B}"]).cuda()
        gates = torch.from_numpy(gold[f"{name}/gates{B}"]).cuda()
        for layout, tol in (("element_wise", 1e-4), ("shared_1d", 1e-4), ("fused_2d", 2e-3)):
            y, disp = L.layout_forward(layout, x, ids, gates)
            torch.cuda.synchronize()
            want = lay[f"{name}/{layout}{B}"]
            assert rel_frob(y.cpu().numpy(), want) <= tol, (layout, B)
            assert disp == int(lay[f"{name}/{layout}{B}_dispatches"]), (layout, B, disp)
        _, disp = L.layout_forward("dequant_only", x, ids, gates)
        assert disp == int(lay[f"{name}/dequant_only{B}_dispatches"])
    L.close()


@pytest.mark.parametrize("name", ARTS)
def test_dequantize_experts_matches_reference(tq, gold, name):
    L = tq.Layer(os.path.join(GOLD, name))
    W = L.dequantize_experts().float().cpu().numpy()
    for e in range(2):
        want = gold[f"{name}/dequant{e}"]
        assert W[e].shape == want.shape
        assert rel_frob(W[e], want) <= 2e-3, e
    L.close()


def test_layout_dispatch_structure(tq):
    """Dispatches: fused 2 for any B, 1D 1 + B*k, element-wise 2*B*k (test_infer.cpp:204-231)."""
    import torch
    L = tq.Layer(os.path.join(GOLD, "folded_b3"))
    k = L.top_k
    for B in (1, 5, 16):
        x = torch.randn(B, L.in_dim, device="cuda")
        ids = torch.stack([torch.randperm(L.num_experts)[:k] for _ in range(B)]).cuda()
        gates = torch.full((B, k), 1.0 / k, device="cuda")
        assert L.layout_forward("fused_2d", x, ids, gates)[1] == 2
        assert L.layout_forward("shared_1d", x, ids, gates)[1] == 1 + B * k
        assert L.layout_forward("element_wise", x, ids, gates)[1] == 2 * B * k
    torch.cuda.synchronize()
    L.close()


def test_layout_errors(tq):
    """Out-of-range expert ids raise ParamError (infer.cpp:203-207 / 252-255)."""
    import torch
    L = tq.Layer(os.path.join(GOLD, "folded_b3"))
    x = torch.randn(2, L.in_dim, device="cuda")
    ids = torch.tensor([[0, 1], [L.num_experts, 0]], dtype=torch.int32, device="cuda")
    gates = torch.full((2, 2), 0.5, device="cuda")
    for layout in ("element_wise", "shared_1d"):
        with pytest.raises(tq.TileqError, match="out of range"):
            L.layout_forward(layout, x, ids, gates)
    L.close()
