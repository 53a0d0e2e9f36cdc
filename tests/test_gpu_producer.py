"""GPU artifact-producer hot spots against the reference, bit for bit.

estimate_hessian, quantize_rtn, quantize_gptq and proxy_loss are compared with
the reference library compiled from its sources (oracle/_ref, through
oracle/ref_shim.cpp); spd_inverse, internal to quant.cpp, with the C
restatement (oracle/tileq_oracle.c), which the GPTQ comparison pins in turn
(GPTQ codes depend on every Hinv entry they touch).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def prod():
    from paper_2605_09281_b200 import producer
    return producer


def _calib(T, d, seed):
    return np.random.default_rng(seed).standard_normal((T, d)).astype(np.float32)


def _resid(rows, cols, seed, scale=0.05):
    r = np.random.default_rng(seed).standard_normal((rows, cols)) * scale
    return r.astype(np.float32)


@pytest.mark.parametrize("T,d,damp", [(100, 80, 0.01), (37, 130, 0.0), (256, 64, 0.1), (1, 3, 0.01)])
def test_estimate_hessian_bit_exact(prod, ref, T, d, damp):
    x = _calib(T, d, T + d)
    hp = prod.estimate_hessian(x, damp)
    h_ref, lam_ref = ref.estimate_hessian(x, damp)
    np.testing.assert_array_equal(hp.h.cpu().numpy().view(np.uint32), h_ref.view(np.uint32))
    assert hp.damping == lam_ref
    assert hp.sample_count == T


@pytest.mark.parametrize("n", [1, 2, 5, 63, 64, 65, 130, 200])
def test_spd_inverse_bit_exact(prod, ref, oracle, n):
    h, _ = ref.estimate_hessian(_calib(max(2 * n, 8), n, n), 0.01)
    got = prod.spd_inverse(h).cpu().numpy()
    want, bad = oracle.spd_inverse(h)
    assert bad is None
    np.testing.assert_array_equal(got.view(np.uint64), want.view(np.uint64))


def test_spd_inverse_singular_matches_reference(prod, ref, oracle):
    import paper_2605_09281_b200 as tq
    h, _ = ref.estimate_hessian(_calib(40, 20, 1), 0.0)
    h[7, :] = 0.0
    h[:, 7] = 0.0
    _, bad = oracle.spd_inverse(h)
    assert bad is not None and bad[0] == 7
    with pytest.raises(tq.NumericError) as ei:
        prod.spd_inverse(h)
    r = np.zeros((3, 20), np.float32)
    with pytest.raises(Exception) as er:      # the reference's own message, via quantize_gptq
        ref.quantize("gptq", r, h, 3, 8)
    assert str(ei.value) == er.value.msg


SHAPES = [(33, 100, 3, 16), (20, 48, 2, 5), (64, 256, 4, 128), (17, 130, 8, 32), (5, 7, 3, 128), (1, 64, 2, 64)]


@pytest.mark.parametrize("rows,cols,bits,gs", SHAPES)
def test_quantize_rtn_bit_exact(prod, ref, rows, cols, bits, gs):
    r = _resid(rows, cols, rows * cols + bits)
    r[0, :3] = 0.0                                  # an all-zero start of a group
    q = prod.quantize_rtn(r, bits, gs)
    c, s, z = ref.quantize("rtn", r, None, bits, gs)
    np.testing.assert_array_equal(q.codes.cpu().numpy().astype(np.uint32), c)
    np.testing.assert_array_equal(q.scales.cpu().numpy().view(np.uint32), s.view(np.uint32))
    np.testing.assert_array_equal(q.zeros.cpu().numpy(), z)


@pytest.mark.parametrize("rows,cols,bits,gs", SHAPES)
def test_quantize_gptq_bit_exact(prod, ref, rows, cols, bits, gs):
    r = _resid(rows, cols, rows + cols * bits)
    h, _ = ref.estimate_hessian(_calib(3 * cols, cols, cols), 0.01)
    q = prod.quantize_gptq(r, h, bits, gs)
    c, s, z = ref.quantize("gptq", r, h, bits, gs)
    np.testing.assert_array_equal(q.codes.cpu().numpy().astype(np.uint32), c)
    np.testing.assert_array_equal(q.scales.cpu().numpy().view(np.uint32), s.view(np.uint32))
    np.testing.assert_array_equal(q.zeros.cpu().numpy(), z)
    # and GPTQ actually changed codes relative to plain rounding on a correlated Hessian
    if not q.used_rtn and rows * cols > 100:
        c_rtn, _, _ = ref.quantize("rtn", r, None, bits, gs)
        assert (c != c_rtn).any()


def test_quantize_gptq_identity_hessian_equals_rtn(prod, ref):
    """With H = I the feedback vanishes (Hinv off-diagonal is 0): GPTQ == RTN."""
    r = _resid(24, 96, 5)
    h = np.eye(96, dtype=np.float32)
    q = prod.quantize_gptq(r, h, 3, 32)
    c, _, _ = ref.quantize("rtn", r, None, 3, 32)
    np.testing.assert_array_equal(q.codes.cpu().numpy().astype(np.uint32), c)


@pytest.mark.parametrize("rows,cols,bits,gs", SHAPES[:4])
def test_proxy_loss_bit_exact(prod, ref, rows, cols, bits, gs):
    r = _resid(rows, cols, 11 * rows + cols)
    h, _ = ref.estimate_hessian(_calib(2 * cols, cols, 3), 0.01)
    for method in ("rtn", "gptq"):
        c, s, z = ref.quantize(method, r, h, bits, gs)
        want = ref.proxy_loss(r, c, s, z, bits, gs, h)
        q = prod.QuantizedExpert(c.astype(np.uint8), s, z, bits, gs)
        import torch
        q.codes, q.scales, q.zeros = (torch.from_numpy(a).cuda() for a in (c.astype(np.uint8), s, z))
        got = prod.proxy_loss(r, q, h)
        assert got == want, (method, got, want)


def test_errors_match_reference(prod, ref):
    import paper_2605_09281_b200 as tq
    r = _resid(4, 16, 1)
    h = np.eye(16, dtype=np.float32)
    cases = [(lambda: prod.quantize_rtn(r, 5, 8), lambda: ref.quantize("rtn", r, None, 5, 8)),
             (lambda: prod.quantize_rtn(r, 3, 0), lambda: ref.quantize("rtn", r, None, 3, 0)),
             (lambda: prod.quantize_gptq(r, h, 3, 0), lambda: ref.quantize("gptq", r, h, 3, 0)),
             (lambda: prod.quantize_rtn(np.zeros((0, 16), np.float32), 3, 8),
              lambda: ref.quantize("rtn", np.zeros((0, 16), np.float32), None, 3, 8)),
             (lambda: prod.quantize_gptq(np.zeros((0, 16), np.float32), h, 3, 8),
              lambda: ref.quantize("gptq", np.zeros((0, 16), np.float32), h, 3, 8))]
    for ours, theirs in cases:
        with pytest.raises(tq.TileqError) as e1:
            ours()
        with pytest.raises(Exception) as e2:
            theirs()
        assert str(e1.value) == e2.value.msg
        assert tq._STATUS[e2.value.code] is type(e1.value)
    with pytest.raises(tq.DataError):
        prod.estimate_hessian(np.zeros((0, 4), np.float32), 0.01)
    with pytest.raises(tq.ParamError):
        prod.estimate_hessian(np.ones((2, 4), np.float32), -1.0)


SKETCH = [(30, 20, 5, 2, 7), (64, 200, 8, 4, 11), (257, 33, 6, 0, 3), (100, 100, 12, 4, 5), (1, 40, 1, 3, 9)]


@pytest.mark.parametrize("rows,cols,rank,iters,seed", SKETCH)
def test_sketch_lowrank_bit_exact(prod, ref, rows, cols, rank, iters, seed):
    w = np.random.default_rng(rows * cols + seed).standard_normal((rows, cols)).astype(np.float32)
    f = prod.sketch_lowrank(w, rank, iters, seed)
    l, s, r = ref.sketch_lowrank(w, rank, iters, seed)
    np.testing.assert_array_equal(f.singulars.cpu().numpy().view(np.uint32), s.view(np.uint32))
    np.testing.assert_array_equal(f.left.cpu().numpy().view(np.uint32), l.view(np.uint32))
    np.testing.assert_array_equal(f.right.cpu().numpy().view(np.uint32), r.view(np.uint32))


def test_sketch_lowrank_rank_deficient_and_zero(prod, ref):
    """Exhausted directions become basis triples (sigma 0), sorted last, as in the reference."""
    rng = np.random.default_rng(4)
    w = (rng.standard_normal((40, 2)) @ rng.standard_normal((2, 24))).astype(np.float32)   # rank 2
    for m in (w, np.zeros((12, 9), np.float32)):
        f = prod.sketch_lowrank(m, 5, 2, 21)
        l, s, r = ref.sketch_lowrank(m, 5, 2, 21)
        np.testing.assert_array_equal(f.singulars.cpu().numpy().view(np.uint32), s.view(np.uint32))
        np.testing.assert_array_equal(f.left.cpu().numpy().view(np.uint32), l.view(np.uint32))
        np.testing.assert_array_equal(f.right.cpu().numpy().view(np.uint32), r.view(np.uint32))


def test_sketch_lowrank_errors_match_reference(prod, ref):
    import paper_2605_09281_b200 as tq
    w = np.ones((6, 4), np.float32)
    for rank, iters in ((0, 1), (5, 1), (2, -1)):
        with pytest.raises(tq.ParamError) as e1:
            prod.sketch_lowrank(w, rank, iters, 1)
        with pytest.raises(Exception) as e2:
            ref.sketch_lowrank(w, max(rank, 0), iters, 1)
        assert str(e1.value) == e2.value.msg


def test_producer_at_c1_dims(prod, ref):
    """c1's in_dim (1024) and group size (128): the staged GPTQ sweep (R = 4 rows per
    CTA, 512 threads dealing 1024 columns) and a 1024-wide H^-1, on 36 residual rows
    (9 CTAs, the last one partial), against the reference; proxy losses equal."""
    d = 1024
    h, _ = ref.estimate_hessian(_calib(384, d, 77), 0.01)
    hp = prod.estimate_hessian(_calib(384, d, 77), 0.01)
    np.testing.assert_array_equal(hp.h.cpu().numpy().view(np.uint32), h.view(np.uint32))
    r = _resid(36, d, 78, scale=0.02)
    q = prod.quantize_gptq(r, hp, 3, 128)
    c, s, z = ref.quantize("gptq", r, h, 3, 128)
    np.testing.assert_array_equal(q.codes.cpu().numpy().astype(np.uint32), c)
    np.testing.assert_array_equal(q.scales.cpu().numpy().view(np.uint32), s.view(np.uint32))
    assert prod.proxy_loss(r, q, hp) == ref.proxy_loss(r, c, s, z, 3, 128, h)


def test_sketch_at_mosaic_like_dims(prod, ref):
    """A 2-row x 3-column mosaic of 768 x 512 blocks, rank 8, 4 power iterations
    (the decompose stage's defaults), against the reference."""
    w = np.random.default_rng(91).standard_normal((1536, 1536)).astype(np.float32)
    f = prod.sketch_lowrank(w, 8, 4, 1234)
    l, s, r = ref.sketch_lowrank(w, 8, 4, 1234)
    np.testing.assert_array_equal(f.singulars.cpu().numpy().view(np.uint32), s.view(np.uint32))
    np.testing.assert_array_equal(f.left.cpu().numpy().view(np.uint32), l.view(np.uint32))
    np.testing.assert_array_equal(f.right.cpu().numpy().view(np.uint32), r.view(np.uint32))
