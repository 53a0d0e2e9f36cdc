"""The artifact producer's hot spots on the GPU.

Mirrors the reference's quantizer API (include/tileq/quant.hpp) for the
stages that dominate the CPU pipeline's time (PAPER: Mixtral takes ~1 h,
mostly proxy_loss):

    estimate_hessian(calib, damping_fraction)  quant.hpp:67,   quant.cpp:116-150
    quantize_rtn(r, bits, group_size)          quant.hpp:74,   quant.cpp:152-175
    quantize_gptq(r, h, bits, group_size)      quant.hpp:85,   quant.cpp:177-221
    proxy_loss(original, q, h)                 quant.hpp:104,  quant.cpp:325-343
    spd_inverse(h)                             quant.cpp:72-112 (internal there)
    sketch_lowrank(w, rank, power_iters, seed) lowrank.hpp:21-30, lowrank.cpp:194-247

Results are bit-identical to the reference's (same f64 operations in the same
order per element; tq_producer.cu).  Matrices may be numpy arrays or CUDA
tensors; outputs are CUDA tensors.  Errors raise the reference's exception
classes with its messages.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import DataError, ParamError, ShapeError, _stream_ptr, _torch, check, lib


def _dev():
    torch = _torch()
    return torch.device("cuda", torch.cuda.current_device())


def _as_dev(x, dtype):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(device=_dev(), dtype=dtype).contiguous()
    npdt = {torch.float32: np.float32, torch.uint8: np.uint8, torch.int32: np.int32}[dtype]
    return torch.from_numpy(np.ascontiguousarray(x, npdt)).to(_dev())


@dataclass
class HessianProxy:
    """quant.hpp:16-20: h (dim x dim f32), the damping lambda actually added, the sample count."""
    h: object
    damping: float = 0.0
    sample_count: int = 0


@dataclass
class QuantizedExpert:
    """A scalar-mode quantized matrix, unpacked: codes (rows x cols uint8), per-group
    scales (f32) and zero points (int32), rows x ceil(cols / group_size) (quant.hpp:37-63)."""
    codes: object
    scales: object
    zeros: object
    bits: int
    group_size: int
    used_rtn: bool = False

    @property
    def out_dim(self) -> int:
        return int(self.codes.shape[0])

    @property
    def in_dim(self) -> int:
        return int(self.codes.shape[1])

    def dequantize(self):
        """dequantize (quant.cpp:285-302): float(double(code - zero) * scale)."""
        torch = _torch()
        g = self.group_size
        idx = torch.arange(self.in_dim, device=self.codes.device) // g
        q = self.codes.to(torch.int64) - self.zeros.to(torch.int64)[:, idx]
        return (q.to(torch.float64) * self.scales.to(torch.float64)[:, idx]).to(torch.float32)


def estimate_hessian(calib, damping_fraction: float) -> HessianProxy:
    torch = _torch()
    x = _as_dev(calib, torch.float32)
    if x.ndim != 2:
        raise ParamError("estimate_hessian: calibration inputs must be 2-D")
    T, d = x.shape
    if T == 0 or d == 0:
        raise DataError("estimate_hessian: empty calibration set")
    h = torch.empty((d, d), dtype=torch.float32, device=_dev())
    import ctypes as C
    lam = C.c_double(0.0)
    check(lib().tq_estimate_hessian(x.data_ptr(), T, d, float(damping_fraction), h.data_ptr(), C.byref(lam),
                                    _stream_ptr(_dev())))
    return HessianProxy(h=h, damping=lam.value, sample_count=T)


def identity_hessian(dim: int) -> HessianProxy:
    torch = _torch()
    return HessianProxy(h=torch.eye(dim, dtype=torch.float32, device=_dev()), damping=0.0, sample_count=0)


def spd_inverse(h):
    torch = _torch()
    hd = _as_dev(h.h if isinstance(h, HessianProxy) else h, torch.float32)
    n = hd.shape[0]
    out = torch.empty((n, n), dtype=torch.float64, device=_dev())
    check(lib().tq_spd_inverse(hd.data_ptr(), n, out.data_ptr(), _stream_ptr(_dev())))
    return out


def _alloc_q(rows, cols, group_size):
    torch = _torch()
    G = (cols + group_size - 1) // group_size if group_size >= 1 else 0
    return (torch.empty((rows, cols), dtype=torch.uint8, device=_dev()),
            torch.empty((rows, max(G, 0)), dtype=torch.float32, device=_dev()),
            torch.empty((rows, max(G, 0)), dtype=torch.int32, device=_dev()))


def quantize_rtn(r, bits: int, group_size: int) -> QuantizedExpert:
    torch = _torch()
    rd = _as_dev(r, torch.float32)
    rows, cols = rd.shape
    codes, scales, zeros = _alloc_q(rows, cols, max(group_size, 1))
    check(lib().tq_quantize_rtn(rd.data_ptr(), rows, cols, int(bits), int(group_size), codes.data_ptr(),
                                scales.data_ptr(), zeros.data_ptr(), _stream_ptr(_dev())))
    return QuantizedExpert(codes, scales, zeros, int(bits), int(group_size))


def quantize_gptq(r, h, bits: int, group_size: int) -> QuantizedExpert:
    import ctypes as C
    torch = _torch()
    rd = _as_dev(r, torch.float32)
    hd = _as_dev(h.h if isinstance(h, HessianProxy) else h, torch.float32)
    rows, cols = rd.shape
    if hd.shape[0] != cols or hd.shape[1] != cols:
        raise ShapeError(f"quantize_gptq: Hessian is {hd.shape[0]}x{hd.shape[1]}, residual has in_dim {cols}")
    codes, scales, zeros = _alloc_q(rows, cols, max(group_size, 1))
    used = C.c_int32(0)
    check(lib().tq_quantize_gptq(rd.data_ptr(), rows, cols, hd.data_ptr(), int(bits), int(group_size),
                                 codes.data_ptr(), scales.data_ptr(), zeros.data_ptr(), C.byref(used),
                                 _stream_ptr(_dev())))
    return QuantizedExpert(codes, scales, zeros, int(bits), int(group_size), used_rtn=bool(used.value))


def proxy_loss(original, q: QuantizedExpert, h) -> float:
    import ctypes as C
    torch = _torch()
    od = _as_dev(original, torch.float32)
    hd = _as_dev(h.h if isinstance(h, HessianProxy) else h, torch.float32)
    rows, cols = od.shape
    if q.codes.shape[0] != rows or q.codes.shape[1] != cols:
        raise ShapeError("sub: shape mismatch")
    if hd.shape[0] != cols or hd.shape[1] != cols:
        raise ShapeError("proxy_loss: Hessian does not match in_dim")
    out = C.c_double(0.0)
    check(lib().tq_proxy_loss(od.data_ptr(), rows, cols, _as_dev(q.codes, torch.uint8).data_ptr(),
                              _as_dev(q.scales, torch.float32).data_ptr(), _as_dev(q.zeros, torch.int32).data_ptr(),
                              int(q.bits), int(q.group_size), hd.data_ptr(), C.byref(out), _stream_ptr(_dev())))
    return out.value


@dataclass
class LowRankFactor:
    """lowrank.hpp:15-19: left (rows x r), singulars (r, nonincreasing), right (r x cols); f32 CUDA tensors."""
    left: object
    singulars: object
    right: object


def sketch_lowrank(w, rank: int, power_iters: int, seed: int) -> LowRankFactor:
    torch = _torch()
    wd = _as_dev(w, torch.float32)
    if wd.ndim != 2:
        raise ParamError("sketch_lowrank: input must be 2-D")
    rows, cols = wd.shape
    r = max(int(rank), 0)
    left = torch.empty((rows, r), dtype=torch.float32, device=_dev())
    right = torch.empty((r, cols), dtype=torch.float32, device=_dev())
    sing = torch.empty((r,), dtype=torch.float32, device=_dev())
    check(lib().tq_sketch_lowrank(wd.data_ptr(), rows, cols, int(rank), int(power_iters), int(seed) & (2**64 - 1),
                                  left.data_ptr(), right.data_ptr(), sing.data_ptr(), _stream_ptr(_dev())))
    return LowRankFactor(left, sing, right)


__all__ = ["HessianProxy", "LowRankFactor", "sketch_lowrank", "QuantizedExpert", "estimate_hessian", "identity_hessian", "spd_inverse",
           "quantize_rtn", "quantize_gptq", "proxy_loss"]
