"""Pinning the producer's checkers on CPU: a numpy restatement of make_grids +
the GPTQ column sweep (quant.cpp:28-70,177-213) driven by the C restatement of
spd_inverse (oracle/tileq_oracle.c, quant.cpp:72-112) must reproduce the
reference's quantize_gptq codes bit for bit (oracle/_ref) -- which pins the
spd_inverse restatement the GPU H^-1 test compares against."""
import numpy as np
import pytest


def _grids(r, bits, gs):
    rows, cols = r.shape
    G = (cols + gs - 1) // gs
    levels = float((1 << bits) - 1)
    scales = np.zeros((rows, G), np.float32)
    zeros = np.zeros((rows, G), np.int32)
    for row in range(rows):
        for g in range(G):
            v = r[row, g * gs:min(cols, (g + 1) * gs)]
            vmin, vmax = float(v.min()), float(v.max())
            rmin, rmax = min(vmin, 0.0), max(vmax, 0.0)
            scale = (rmax - rmin) / levels
            if scale <= 0.0:
                scale = 1e-8
            s = np.float32(np.float16(np.float32(scale)))
            if s <= 0.0:
                s = np.float32(2.0 ** -24)
            z = np.rint(-rmin / float(s))
            z = min(levels, max(0.0, z))
            scales[row, g], zeros[row, g] = s, int(z)
    return scales, zeros


def _gptq(r, hinv, bits, gs, scales, zeros):
    rows, dim = r.shape
    levels = float((1 << bits) - 1)
    codes = np.zeros((rows, dim), np.uint32)
    for row in range(rows):
        work = r[row].astype(np.float64)
        for j in range(dim):
            s = float(scales[row, j // gs])
            z = int(zeros[row, j // gs])
            code = min(levels, max(0.0, np.rint(work[j] / s) + z))
            codes[row, j] = int(code)
            err = work[j] - (code - z) * s
            work[j + 1:] = work[j + 1:] - (err * hinv[j, j + 1:]) / hinv[j, j]
    return codes


@pytest.mark.parametrize("rows,dim,bits,gs", [(6, 24, 3, 8), (4, 40, 2, 16), (5, 33, 4, 5), (3, 64, 8, 32)])
def test_gptq_restatement_matches_reference(oracle, ref, rows, dim, bits, gs):
    rng = np.random.default_rng(rows * dim + bits)
    r = (rng.standard_normal((rows, dim)) * 0.1).astype(np.float32)
    h, _ = ref.estimate_hessian(rng.standard_normal((3 * dim, dim)).astype(np.float32), 0.01)
    hinv, bad = oracle.spd_inverse(h)
    assert bad is None
    scales, zeros = _grids(r, bits, gs)
    codes = _gptq(r, hinv, bits, gs, scales, zeros)
    c, s, z = ref.quantize("gptq", r, h, bits, gs)
    np.testing.assert_array_equal(scales.view(np.uint32), s.view(np.uint32))
    np.testing.assert_array_equal(zeros, z)
    # these cases keep GPTQ over plain rounding (quant.cpp:216-219), so the codes
    # compared are the column sweep's
    c_rtn, _, _ = ref.quantize("rtn", r, None, bits, gs)
    assert not np.array_equal(c, c_rtn)
    np.testing.assert_array_equal(codes, c)


def test_spd_inverse_restatement_is_an_inverse(oracle, ref):
    rng = np.random.default_rng(3)
    h, _ = ref.estimate_hessian(rng.standard_normal((200, 50)).astype(np.float32), 0.01)
    hinv, bad = oracle.spd_inverse(h)
    assert bad is None
    assert np.abs(hinv @ h.astype(np.float64) - np.eye(50)).max() < 1e-9
