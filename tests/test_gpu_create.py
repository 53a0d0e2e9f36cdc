"""In-memory layers (tq_layer_create, the C++ shim's entry) against the
artifact loader (tq_layer_load): the same layer through either door gives
the same engine state, so forwards agree bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPECS = [
    dict(K=6, top_k=2, i=64, o=48, S=1, r=8, bits=2, g=32, calib="gauss", seed=11),
    dict(K=6, top_k=2, i=64, o=48, S=1, r=8, bits=3, g=32, calib="gauss", seed=12),
    dict(K=6, top_k=2, i=64, o=48, S=1, r=8, bits=4, g=32, calib="gauss", seed=13),
    dict(K=6, top_k=2, i=64, o=48, S=1, r=8, bits=8, g=32, calib="gauss", seed=14),
    dict(K=8, top_k=2, i=512, o=640, r=16, bits=3, g=128, calib="signs", seed=15),
]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"i{s['i']}b{s['bits']}")
def test_create_matches_load(ref, make_artifact, spec):
    import paper_2605_09281_b200 as tq
    from oracle.oracle import read_artifact_np
    from conftest import rel_frob
    d = make_artifact(**spec)
    a = read_artifact_np(d)
    for q in a["experts"] + a["shared"]:
        q["zeros"] = q["zeros"].astype(np.uint8)
    La = tq.Layer(d)
    Lm = tq.Layer.from_arrays(a)
    for B in (1, 5, 40, 300):
        x = np.random.default_rng(B).standard_normal((B, spec["i"])).astype(np.float32)
        ya, ida, ga = La.forward_host(x, with_routing=True)
        ym, idm, gm = Lm.forward_host(x, with_routing=True)
        np.testing.assert_array_equal(ida, idm)
        np.testing.assert_array_equal(ga, gm)
        np.testing.assert_array_equal(ya, ym)
        yr, _, _ = ref.load(d).forward(x)
        assert rel_frob(ym, yr) <= 2e-3, (B, rel_frob(ym, yr))
