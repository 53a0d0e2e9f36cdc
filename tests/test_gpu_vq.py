"""Vector-quantized (codebook) residuals -- TileQ_v, SURVEY 8(f) row 2.

Artifacts come from the reference's own pipeline (quantize_moe with the vq
quantizer, quant.cpp:223-283, through oracle/_ref) and are read by the engine's
loader (io.cpp:464-480 semantics: codes o x ceil(i / sub_dim), codebook
2^bits x sub_dim binary16).  Every codebook entry is f16-snapped
(quant.cpp:262-266), so the loader resolves each code to its exact fp16 weights
and the dense-weight GEMM path serves the layer.  Checked against the reference
(route ids bit-exact, outputs within the north_star 2e-3), plus the
dequantized weights bit-exact against dequantize() (quant.cpp:303-321).
"""
import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu

SPECS = [
    dict(K=6, top_k=2, i=256, o=128, S=1, r=8, bits=2, g=128, calib="gauss", seed=21, quantizer="vq", sub_dim=2),
    dict(K=8, top_k=2, i=320, o=200, S=0, r=16, bits=3, g=128, calib="signs", seed=22, quantizer="vq", sub_dim=2),
    dict(K=5, top_k=3, i=192, o=96, S=0, r=8, bits=4, g=128, calib="gauss", seed=23, quantizer="vq", sub_dim=1),
    dict(K=4, top_k=1, i=256, o=64, S=1, r=4, bits=2, g=128, calib="none", seed=24, quantizer="vq", sub_dim=4),
]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"b{s['bits']}sd{s['sub_dim']}")
def test_vq_forward_matches_reference(ref, make_artifact, spec):
    import paper_2605_09281_b200 as tq
    d = make_artifact(**spec)
    L = tq.Layer(d)
    assert L.bits == spec["bits"]
    R = ref.load(d)
    for B in (1, 7, 64, 300):
        x = np.random.default_rng(B).standard_normal((B, spec["i"])).astype(np.float32)
        y, ids, gates = L.forward_host(x, with_routing=True)
        yr, idr, gr = R.forward(x)
        np.testing.assert_array_equal(ids, idr)
        np.testing.assert_array_max_ulp(gates, gr, maxulp=1)
        e = rel_frob(y, yr)
        assert e <= 2e-3, (B, e)


@pytest.mark.parametrize("spec", SPECS[:2], ids=lambda s: f"b{s['bits']}sd{s['sub_dim']}")
def test_vq_dequantize_bit_exact(ref, make_artifact, spec):
    import torch
    import paper_2605_09281_b200 as tq
    d = make_artifact(**spec)
    L = tq.Layer(d)
    R = ref.load(d)
    w = L.dequantize_experts().float().cpu().numpy()
    for e in range(spec["K"]):
        np.testing.assert_array_equal(w[e], R.dequantize(e))   # codebook entries are exact in fp16


def test_vq_export_codes_is_refused(ref, make_artifact):
    import paper_2605_09281_b200 as tq
    L = tq.Layer(make_artifact(**SPECS[0]))
    with pytest.raises(tq.ParamError):
        L.export_codes(0)
