"""The routers' f64 exp against glibc's (SURVEY hard part 1).

route() takes prob_k = std::exp(s_k - mx) in f64 (moe.cpp:72) -- glibc on the
reference's host.  The engine's routers run the same algorithm (csrc/tq_exp.h,
a restatement of glibc's table-driven exp), so the contract is bit-identity on
every argument: a dense log-uniform sweep of [-745, 0] (the softmax's range),
differences of f32 scores (the form s - mx takes), the over/underflow range,
and the edges.
"""
import ctypes
import ctypes.util

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _glibc_exp(xs):
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.exp.restype = ctypes.c_double
    libm.exp.argtypes = [ctypes.c_double]
    return np.array([libm.exp(float(v)) for v in xs], np.float64)


def _ulps(a, b):
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    return np.abs(ia - ib)


def test_router_exp_matches_glibc():
    import torch
    import paper_2605_09281_b200 as tq
    rng = np.random.default_rng(0)
    n = 400_000
    sweep = -np.exp(rng.uniform(np.log(1e-12), np.log(745.0), n))          # log-uniform magnitudes
    s = rng.standard_normal((n // 2, 2)).astype(np.float32) * 8.0            # f32 scores
    diffs = (s.min(axis=1).astype(np.float64) - s.max(axis=1).astype(np.float64))
    edges = np.array([0.0, -0.0, -1e-300, -5e-324, -1.0, -0.5, -708.39, -708.40, -744.44, -745.0, -745.13,
                      -745.2, -746.0], np.float64)
    wide = rng.uniform(-1100.0, 800.0, n // 4)
    x = np.concatenate([sweep, diffs, wide, edges, -edges])
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    tq.check(tq.lib().tq_exp_f64(xd.data_ptr(), x.size, yd.data_ptr(), None))
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    want = _glibc_exp(x)
    u = _ulps(y, want)
    exact = float((u == 0).mean())
    print(f"\nexp vs glibc: {x.size} arguments, {exact * 100:.4f}% bit-identical, max {int(u.max())} ulp")
    assert int(u.max()) == 0
