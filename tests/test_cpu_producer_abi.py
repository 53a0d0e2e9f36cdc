"""Host-side argument checks of the producer C-ABI entries, on a machine without a
GPU: every domain error the reference raises before touching data
(quant.cpp:18-22,116-122,152-155,177-185; lowrank.cpp:64-73,196-197) comes back
with the reference's error class and message, before any device call."""
import ctypes as C

import pytest


@pytest.fixture(scope="module")
def tq():
    import paper_2605_09281_b200 as tq
    return tq


def _err(tq, status):
    with pytest.raises(tq.TileqError) as e:
        tq.check(status)
    return e.value


def test_estimate_hessian_domain_errors(tq):
    L = tq.lib()
    lam = C.c_double()
    e = _err(tq, L.tq_estimate_hessian(None, 0, 4, 0.01, None, C.byref(lam), None))
    assert isinstance(e, tq.DataError) and str(e) == "estimate_hessian: empty calibration set"
    e = _err(tq, L.tq_estimate_hessian(None, 3, 4, -1.0, None, C.byref(lam), None))
    assert isinstance(e, tq.ParamError) and str(e) == "estimate_hessian: damping_fraction must be >= 0"


def test_quantizer_domain_errors(tq):
    L = tq.lib()
    e = _err(tq, L.tq_quantize_rtn(None, 2, 8, 5, 4, None, None, None, None))
    assert isinstance(e, tq.ParamError) and str(e) == "quantizer bits must be in {2,3,4,8}, got 5"
    e = _err(tq, L.tq_quantize_rtn(None, 2, 8, 3, 0, None, None, None, None))
    assert str(e) == "quantize_rtn: group_size must be >= 1"
    e = _err(tq, L.tq_quantize_rtn(None, 0, 8, 3, 4, None, None, None, None))
    assert str(e) == "quantize_rtn: empty input"
    e = _err(tq, L.tq_quantize_gptq(None, 2, 8, None, 7, 4, None, None, None, None, None))
    assert str(e) == "quantizer bits must be in {2,3,4,8}, got 7"
    e = _err(tq, L.tq_quantize_gptq(None, 2, 8, None, 3, 0, None, None, None, None, None))
    assert str(e) == "quantize_gptq: group_size must be >= 1"
    out = C.c_double()
    e = _err(tq, L.tq_proxy_loss(None, 2, 8, None, None, None, 1, 4, None, C.byref(out), None))
    assert isinstance(e, tq.ParamError) and "got 1" in str(e)


def test_sketch_domain_errors(tq):
    L = tq.lib()
    e = _err(tq, L.tq_sketch_lowrank(None, 0, 4, 1, 1, 0, None, None, None, None))
    assert str(e) == "sketch_lowrank: input matrix is empty"
    e = _err(tq, L.tq_sketch_lowrank(None, 6, 4, 5, 1, 0, None, None, None, None))
    assert str(e) == "sketch_lowrank: rank 5 outside [1, 4] for a 6x4 matrix"
    e = _err(tq, L.tq_sketch_lowrank(None, 6, 4, 2, -1, 0, None, None, None, None))
    assert str(e) == "sketch_lowrank: power_iters must be >= 0"


def test_messages_match_the_reference(tq, ref):
    """The same calls on the reference library raise the same messages."""
    import numpy as np
    r = np.ones((2, 8), np.float32)
    for bits, gs, want in ((5, 4, "quantizer bits must be in {2,3,4,8}, got 5"),
                           (3, 0, "quantize_rtn: group_size must be >= 1")):
        with pytest.raises(Exception) as e:
            ref.quantize("rtn", r, None, bits, gs)
        assert e.value.msg == want
    with pytest.raises(Exception) as e:
        ref.sketch_lowrank(np.ones((6, 4), np.float32), 5, 1, 0)
    assert e.value.msg == "sketch_lowrank: rank 5 outside [1, 4] for a 6x4 matrix"
