"""B200-native fused low-rank MoE inference engine for TileQ artifacts.

Python mirror of the reference's Python API for the hot path
(/root/reference/proj/bindings/py_module.cpp, python/tileq/__init__.py):

    route(x, gate_weights, top_k) -> (int64 ids [B,k], float32 gates [B,k])
    forward_from_artifact(artifact_dir, x) -> float32 [B, o]
    TileqError (base of ShapeError, ParamError, ... like errors.hpp:13-50)

plus the device-tensor entry points (``Layer``) a serving stack uses.  All
compute runs in libtileq_b200.so (sm_100a kernels behind the C-ABI in
include/tileq_b200.h); there is no CPU fallback -- if the library cannot be
loaded or no B200 is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TQ_LIB_PATH") or os.path.join(HERE, "libtileq_b200.so")

PATH_FULL, PATH_QMOE, PATH_LOTILE = 0, 1, 2
_PATHS = {"full": PATH_FULL, "tileq": PATH_FULL, "qmoe": PATH_QMOE, "lotile": PATH_LOTILE}


# ---------------------------------------------------------------------------
# errors: the reference taxonomy (errors.hpp:13-50) + device failures
# ---------------------------------------------------------------------------

class TileqError(RuntimeError):
    """Base of every engine error (the reference binding's TileqError)."""


class ShapeError(TileqError):
    pass


class ParamError(TileqError):
    pass


class SizeError(TileqError):
    pass


class FormatError(TileqError):
    pass


class IoError(TileqError):
    pass


class NumericError(TileqError):
    pass


class DataError(TileqError):
    pass


class CudaError(TileqError):
    pass


class NcclError(TileqError):
    pass


_STATUS = {1: ShapeError, 2: ParamError, 3: SizeError, 4: FormatError, 5: IoError,
           6: NumericError, 7: DataError, 8: CudaError, 9: NcclError}


class _LayerInfo(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "num_experts", "top_k", "in_dim", "out_dim", "num_shared", "rank", "grid_rows",
        "grid_cols", "bits", "group_size", "expert_begin", "expert_end", "device",
        "device_bytes", "tier_folded", "tier_scalar", "tier_general")]


class _QMatDesc(C.Structure):
    _fields_ = [("out_dim", C.c_int64), ("in_dim", C.c_int64), ("bits", C.c_int), ("mode", C.c_int),
                ("packed", C.c_void_p), ("packed_bytes", C.c_int64), ("group_size", C.c_int64),
                ("scale_bits", C.c_void_p), ("zeros", C.c_void_p), ("sub_dim", C.c_int64),
                ("codebook_bits", C.c_void_p)]


class _LayerDesc(C.Structure):
    _fields_ = [("num_experts", C.c_int64), ("top_k", C.c_int64), ("in_dim", C.c_int64), ("out_dim", C.c_int64),
                ("num_shared", C.c_int64), ("gate_weights", C.c_void_p), ("grid_rows", C.c_int64),
                ("grid_cols", C.c_int64), ("rank", C.c_int64), ("placement", C.c_void_p),
                ("scaling", C.c_void_p), ("singular_bits", C.c_void_p), ("u_codes", C.c_void_p),
                ("u_absmax", C.c_void_p), ("v_codes", C.c_void_p), ("v_absmax", C.c_void_p),
                ("experts", C.c_void_p), ("shared", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load libtileq_b200.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    L = C.CDLL(LIB_PATH)
    p, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    L.tq_last_error.restype = C.c_char_p
    L.tq_version.restype = C.c_char_p
    L.tq_layer_load.argtypes = [C.c_char_p, i32, i32, i64, i64, C.POINTER(p)]
    L.tq_layer_free.argtypes = [p]
    L.tq_artifact_check.argtypes = [C.c_char_p, i32]
    L.tq_exp_f64.argtypes = [p, i64, p, p]
    L.tq_layer_create.argtypes = [p, i32, i64, i64, C.POINTER(p)]
    L.tq_layer_info_get.argtypes = [p, C.POINTER(_LayerInfo)]
    L.tq_layer_reserve.argtypes = [p, i64]
    L.tq_route.argtypes = [p, p, i64, p, p, p]
    L.tq_route_raw.argtypes = [p, i64, i64, p, i64, i64, p, p, p]
    L.tq_permute.argtypes = [p, p, i64, p, p, p, p]
    L.tq_forward.argtypes = [p, p, i64, p, p, p, i32, p]
    L.tq_forward_routed.argtypes = [p, p, i64, p, p, p, i32, p]
    L.tq_forward_host.argtypes = [p, p, i64, p, p, p, i32]
    L.tq_sync.argtypes = [p, p]
    L.tq_debug_decode_counters.argtypes = [p, p, i64]
    L.tq_unpack_codes.argtypes = [p, i64, i32, i64, p, p]
    L.tq_layer_export_codes.argtypes = [p, i64, p, p]
    L.tq_launch_count.restype = C.c_uint64
    L.tq_launch_count.argtypes = [p]
    L.tq_reset_launch_count.argtypes = [p]
    L.tq_ep_dispatch_rows.argtypes = [p, p, i64, p, p, p, p, i32, p]
    L.tq_ep_expert_rows.argtypes = [p, p, p, i64, p, i64, p, i32, p]
    L.tq_ep_combine.argtypes = [p, p, i64, p, p, p, p, i32, p]
    L.tq_ep_expert_rows_slab.argtypes = [p, p, i64, i64, i64, p, i64, p, i32, p]
    L.tq_gemm_timing_enable.argtypes = [p, i32]
    L.tq_gemm_time_get.argtypes = [p, C.POINTER(C.c_double), C.POINTER(i64)]
    L.tq_layout_prepare.argtypes = [p, i32]
    L.tq_layout_forward.argtypes = [p, i32, p, i64, p, p, p, C.POINTER(i64), p]
    L.tq_dequantize_experts.argtypes = [p, p, p]
    L.tq_ep_xrow_elems.restype = i64
    L.tq_ep_xrow_elems.argtypes = [p]
    L.tq_ep_extrow_elems.restype = i64
    L.tq_ep_extrow_elems.argtypes = [p]
    L.tq_estimate_hessian.argtypes = [p, i64, i64, C.c_double, p, p, p]
    L.tq_spd_inverse.argtypes = [p, i64, p, p]
    L.tq_quantize_rtn.argtypes = [p, i64, i64, i32, i64, p, p, p, p]
    L.tq_quantize_gptq.argtypes = [p, i64, i64, p, i32, i64, p, p, p, p, p]
    L.tq_proxy_loss.argtypes = [p, i64, i64, p, p, p, i32, i64, p, p, p]
    L.tq_sketch_lowrank.argtypes = [p, i64, i64, i64, i32, C.c_uint64, p, p, p, p]
    for name in ("tq_layer_load", "tq_artifact_check", "tq_exp_f64", "tq_layer_create", "tq_layer_free", "tq_layer_info_get", "tq_layer_reserve", "tq_route",
                 "tq_route_raw", "tq_permute", "tq_forward", "tq_forward_routed", "tq_forward_host",
                 "tq_sync", "tq_debug_decode_counters", "tq_unpack_codes", "tq_layer_export_codes", "tq_ep_dispatch_rows",
                 "tq_ep_expert_rows", "tq_ep_expert_rows_slab", "tq_ep_combine", "tq_gemm_timing_enable", "tq_gemm_time_get",
                 "tq_estimate_hessian", "tq_spd_inverse", "tq_quantize_rtn", "tq_quantize_gptq", "tq_proxy_loss", "tq_sketch_lowrank"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def check(status: int) -> None:
    if status != 0:
        msg = lib().tq_last_error().decode(errors="replace")
        raise _STATUS.get(status, TileqError)(msg)


def _torch():
    import torch  # plumbing only: device memory and streams
    return torch


def _stream_ptr(device) -> int:
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


def _dptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


# ---------------------------------------------------------------------------
# the layer
# ---------------------------------------------------------------------------

class Layer:
    """A TileQ artifact resident on one B200 (read_artifact + the runtime).

    expert_range=(begin, end) keeps only those routed experts resident
    (expert parallel); the router, factor blocks and shared experts always are.
    """

    def __init__(self, artifact_dir: str, device: int = 0, verify_crc: bool = True,
                 expert_range: Optional[tuple] = None):
        b, e = expert_range if expert_range is not None else (0, -1)
        h = C.c_void_p()
        check(lib().tq_layer_load(os.fsencode(artifact_dir), int(device), int(verify_crc), int(b), int(e),
                                  C.byref(h)))
        self._init_handle(h, device, artifact_dir)

    def _init_handle(self, h, device, artifact_dir):
        self._h = h
        self.device = int(device)
        info = _LayerInfo()
        check(lib().tq_layer_info_get(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in _LayerInfo._fields_}
        for k in ("num_experts", "top_k", "in_dim", "out_dim", "num_shared", "rank", "bits", "group_size"):
            setattr(self, k, self.info[k])
        self.artifact_dir = artifact_dir

    @classmethod
    def from_arrays(cls, t: dict, device: int = 0, expert_range: Optional[tuple] = None) -> "Layer":
        """An in-memory layer (TileQLayer, infer.hpp:22-28) through tq_layer_create.

        `t` holds numpy arrays: K, top_k, i, o, S, M, N, r; gate (K x i f32),
        scaling (K x i f32), placement (K x 2), singulars (r binary16 bits),
        u_codes (M x o x r int8), u_absmax (M), v_codes (N x r x i int8),
        v_absmax (N); experts / shared: lists of dicts with packed (u8),
        bits, and either group_size, scales (binary16 bits), zeros, or
        sub_dim, codebook (binary16 bits)."""
        keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data

        def qm(q):
            d = _QMatDesc()
            d.out_dim, d.in_dim, d.bits = int(t["o"]), int(t["i"]), int(q["bits"])
            d.packed = arr(q["packed"], np.uint8)
            d.packed_bytes = int(np.asarray(q["packed"]).size)
            if "codebook" in q:
                d.mode, d.sub_dim = 1, int(q["sub_dim"])
                d.codebook_bits = arr(q["codebook"], np.uint16)
            else:
                d.mode, d.group_size = 0, int(q["group_size"])
                d.scale_bits = arr(q["scales"], np.uint16)
                d.zeros = arr(q["zeros"], np.uint8)
            return d

        ex = (_QMatDesc * max(1, len(t["experts"])))(*[qm(q) for q in t["experts"]])
        sh = (_QMatDesc * max(1, len(t["shared"])))(*[qm(q) for q in t["shared"]])
        d = _LayerDesc()
        for k, f in (("num_experts", "K"), ("top_k", "top_k"), ("in_dim", "i"), ("out_dim", "o"),
                     ("num_shared", "S"), ("grid_rows", "M"), ("grid_cols", "N"), ("rank", "r")):
            setattr(d, k, int(t[f]))
        d.gate_weights = arr(t["gate"], np.float32)
        d.scaling = arr(t["scaling"], np.float32)
        d.placement = arr(t["placement"], np.uint32)
        d.singular_bits = arr(t["singulars"], np.uint16)
        d.u_codes, d.u_absmax = arr(t["u_codes"], np.int8), arr(t["u_absmax"], np.float32)
        d.v_codes, d.v_absmax = arr(t["v_codes"], np.int8), arr(t["v_absmax"], np.float32)
        d.experts = C.cast(ex, C.c_void_p)
        d.shared = C.cast(sh, C.c_void_p) if len(t["shared"]) else None
        b, e = expert_range if expert_range is not None else (0, -1)
        h = C.c_void_p()
        check(lib().tq_layer_create(C.byref(d), int(device), int(b), int(e), C.byref(h)))
        self = cls.__new__(cls)
        self._init_handle(h, device, "<memory>")
        return self

    def close(self):
        if getattr(self, "_h", None):
            lib().tq_layer_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device-tensor API ----------------------------------------------------
    def _check_x(self, x):
        torch = _torch()
        if x.dim() != 2 or x.shape[1] != self.in_dim:
            raise ShapeError(f"token width {x.shape[-1]} vs in_dim {self.in_dim}")
        if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
            raise ParamError("x must be a contiguous float32 CUDA tensor")

    def reserve(self, max_tokens: int) -> None:
        check(lib().tq_layer_reserve(self._h, int(max_tokens)))

    def route(self, x):
        """route() on the GPU: (int32 ids [B,k], float32 gates [B,k]) CUDA tensors."""
        torch = _torch()
        self._check_x(x)
        B = x.shape[0]
        ids = torch.empty((B, self.top_k), dtype=torch.int32, device=x.device)
        gates = torch.empty((B, self.top_k), dtype=torch.float32, device=x.device)
        check(lib().tq_route(self._h, x.data_ptr(), B, ids.data_ptr(), gates.data_ptr(), _stream_ptr(x.device)))
        return ids, gates

    def permute(self, ids):
        torch = _torch()
        B = ids.shape[0]
        perm = torch.empty(B * self.top_k, dtype=torch.int32, device=ids.device)
        inv = torch.empty(B * self.top_k, dtype=torch.int32, device=ids.device)
        offsets = torch.empty(self.num_experts + 1, dtype=torch.int32, device=ids.device)
        check(lib().tq_permute(self._h, ids.contiguous().data_ptr(), B, perm.data_ptr(), offsets.data_ptr(),
                               inv.data_ptr(), _stream_ptr(ids.device)))
        return perm, offsets, inv

    def forward(self, x, ids=None, gates=None, path: str = "full", out=None):
        """tileq_forward (path='full'), qmoe_forward ('qmoe') or lotile_forward
        ('lotile').  With ids/gates None the layer routes the batch itself."""
        torch = _torch()
        self._check_x(x)
        B = x.shape[0]
        y = out if out is not None else torch.empty((B, self.out_dim), dtype=torch.float32, device=x.device)
        st = _stream_ptr(x.device)
        if ids is None:
            check(lib().tq_forward_routed(self._h, x.data_ptr(), B, y.data_ptr(), None, None, _PATHS[path], st))
        else:
            ids32 = ids.to(torch.int32).contiguous()
            if ids32.shape != (B, self.top_k):
                raise ShapeError(f"routing batch {ids32.shape[0]} vs input batch {B}")
            g = gates.to(torch.float32).contiguous()
            if B and (int(ids32.min()) < 0 or int(ids32.max()) >= self.num_experts):
                raise ParamError(f"reference_forward: expert id out of range [0, {self.num_experts})")
            check(lib().tq_forward(self._h, x.data_ptr(), B, ids32.data_ptr(), g.data_ptr(), y.data_ptr(),
                                   _PATHS[path], st))
        return y

    # the paper's bench layouts (infer.cpp:345-426), in BenchLayout order
    LAYOUTS = ("fused_2d", "shared_1d", "element_wise", "dequant_only")

    def layout_prepare(self, layout: str):
        """Build a comparison layout's factors once (outside timed regions)."""
        check(lib().tq_layout_prepare(self._h, self.LAYOUTS.index(layout)))

    def layout_forward(self, layout: str, x, ids, gates, out=None):
        """One call of a bench layout on a given routing (device tensors):
        fused_2d = lotile_forward, shared_1d = baseline_1d_forward,
        element_wise = baseline_elementwise_forward, dequant_only = dequantize
        every resident expert.  Returns (y or None, dispatch count)."""
        torch = _torch()
        self._check_x(x)
        B = x.shape[0]
        ids32 = ids.to(torch.int32).contiguous()
        if ids32.shape != (B, self.top_k):
            raise ShapeError(f"routing batch {ids32.shape[0]} vs input batch {B}")
        g = gates.to(torch.float32).contiguous()
        y = out if out is not None else torch.empty((B, self.out_dim), dtype=torch.float32, device=x.device)
        disp = C.c_int64(0)
        check(lib().tq_layout_forward(self._h, self.LAYOUTS.index(layout), x.data_ptr(), B, ids32.data_ptr(),
                                      g.data_ptr(), y.data_ptr(), C.byref(disp), _stream_ptr(x.device)))
        return (None if layout == "dequant_only" else y), int(disp.value)

    def dequantize_experts(self):
        """fp16 [n_experts, out_dim, in_dim]: every resident expert's residual
        dequantized (quant.cpp:285-323) from the engine's repacked layout."""
        torch = _torch()
        n = self.info["expert_end"] - self.info["expert_begin"]
        out = torch.empty((n, self.out_dim, self.in_dim), dtype=torch.float16, device=f"cuda:{self.device}")
        check(lib().tq_dequantize_experts(self._h, out.data_ptr(), _stream_ptr(out.device)))
        return out

    def forward_routed(self, x, path: str = "full"):
        """(y, ids int32, gates) in one call."""
        torch = _torch()
        self._check_x(x)
        B = x.shape[0]
        y = torch.empty((B, self.out_dim), dtype=torch.float32, device=x.device)
        ids = torch.empty((B, self.top_k), dtype=torch.int32, device=x.device)
        gates = torch.empty((B, self.top_k), dtype=torch.float32, device=x.device)
        check(lib().tq_forward_routed(self._h, x.data_ptr(), B, y.data_ptr(), ids.data_ptr(), gates.data_ptr(),
                                      _PATHS[path], _stream_ptr(x.device)))
        return y, ids, gates

    def sync(self):
        check(lib().tq_sync(self._h, _stream_ptr(self.device)))

    # -- host-buffer API (the reference binding's numpy in / numpy out) ------
    def forward_host(self, x: np.ndarray, path: str = "full", with_routing: bool = False, out=None):
        """Host f32 in / host f32 out (tq_forward_host): the copies are part of the call.
        ``out`` may be a preallocated (pinned) float32 [B, o] array."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        if x.ndim != 2:
            raise ParamError("x must be a 2-D float array")
        if x.shape[1] != self.in_dim:
            raise ShapeError(f"token width {x.shape[1]} vs in_dim {self.in_dim}")
        B = x.shape[0]
        if out is not None:
            if out.shape != (B, self.out_dim) or out.dtype != np.float32 or not out.flags.c_contiguous:
                raise ParamError("out must be a contiguous float32 [B, out_dim] array")
            y = out
        else:
            y = np.empty((B, self.out_dim), np.float32)
        ids = np.empty((B, self.top_k), np.int64) if with_routing else None
        gates = np.empty((B, self.top_k), np.float32) if with_routing else None
        check(lib().tq_forward_host(self._h, x.ctypes.data, B, y.ctypes.data,
                                    None if ids is None else ids.ctypes.data,
                                    None if gates is None else gates.ctypes.data, _PATHS[path]))
        return (y, ids, gates) if with_routing else y

    # -- instrumentation ------------------------------------------------------
    def launch_count(self) -> int:
        return int(lib().tq_launch_count(self._h))

    def reset_launch_count(self) -> None:
        lib().tq_reset_launch_count(self._h)

    def gemm_timing(self, enable: bool) -> None:
        """Bracket every fused expert-GEMM launch with CUDA events (device time)."""
        check(lib().tq_gemm_timing_enable(self._h, int(enable)))

    def gemm_time(self):
        """(total device ms, launches) of the expert GEMM since gemm_timing(True)."""
        ms = C.c_double()
        n = C.c_int64()
        check(lib().tq_gemm_time_get(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    # -- expert-parallel stages (tq_ep_*; orchestrated by ep.EPLayer) --------
    def ep_row_widths(self):
        """(x row, ext row) widths in fp16 elements of the dispatch buffers."""
        return int(lib().tq_ep_xrow_elems(self._h)), int(lib().tq_ep_extrow_elems(self._h))

    def ep_dispatch_rows(self, x, ids, perm, path: str = "full"):
        """Rows to send, in permuted-slot order: fp16 token rows + fp16 extension rows."""
        torch = _torch()
        self._check_x(x)
        B = x.shape[0]
        xw, ew = self.ep_row_widths()
        xrows = torch.empty((B * self.top_k, xw), dtype=torch.float16, device=x.device)
        erows = torch.empty((B * self.top_k, ew), dtype=torch.float16, device=x.device)
        check(lib().tq_ep_dispatch_rows(self._h, x.data_ptr(), B, ids.data_ptr(), perm.data_ptr(),
                                        xrows.data_ptr(), erows.data_ptr(), _PATHS[path], _stream_ptr(x.device)))
        return xrows, erows

    def ep_expert_rows(self, xrows, erows, segments: np.ndarray, path: str = "full"):
        """Resident-expert outputs (f32 [rows, o]) for received rows; segments int64
        [n, 3] = (local expert, first row, row count) sorted by first row."""
        torch = _torch()
        rows = xrows.shape[0]
        y = torch.empty((rows, self.out_dim), dtype=torch.float32, device=xrows.device)
        seg = np.ascontiguousarray(segments, dtype=np.int64).reshape(-1, 3)
        if rows and len(seg):
            check(lib().tq_ep_expert_rows(self._h, xrows.data_ptr(), erows.data_ptr(), rows, seg.ctypes.data,
                                          len(seg), y.data_ptr(), _PATHS[path], _stream_ptr(xrows.device)))
        return y

    def ep_expert_rows_slab(self, rows, n_src: int, slab: int, counts, path: str = "full"):
        """Resident-expert outputs for rows received in fixed-capacity slabs (no host
        round trip): rows fp16 [n_src * slab, xw + ew] = [x | ext]; counts int32
        [n_src, e_stride] the received count matrix (device).  f32 [n_src * slab, o]."""
        torch = _torch()
        y = torch.empty((n_src * slab, self.out_dim), dtype=torch.float32, device=rows.device)
        cnt = counts.to(device=rows.device, dtype=torch.int32).contiguous()
        check(lib().tq_ep_expert_rows_slab(self._h, rows.data_ptr(), rows.shape[1], n_src, slab, cnt.data_ptr(),
                                           cnt.shape[1], y.data_ptr(), _PATHS[path], _stream_ptr(rows.device)))
        return y

    def ep_combine(self, x, yrows, inv, gates, path: str = "full", out=None):
        """Gate-weighted combine of returned rows (+ shared experts on the home tokens)."""
        torch = _torch()
        B = x.shape[0]
        y = out if out is not None else torch.empty((B, self.out_dim), dtype=torch.float32, device=x.device)
        check(lib().tq_ep_combine(self._h, x.data_ptr(), B, yrows.data_ptr(), inv.data_ptr(), gates.data_ptr(),
                                  y.data_ptr(), _PATHS[path], _stream_ptr(x.device)))
        return y

    def export_codes(self, e: int):
        """Codes of matrix e decoded back from the engine's tile layout (uint32 [o, i] CUDA tensor)."""
        torch = _torch()
        out = torch.empty((self.out_dim, self.in_dim), dtype=torch.int32, device=f"cuda:{self.device}")
        check(lib().tq_layer_export_codes(self._h, int(e), out.data_ptr(), _stream_ptr(self.device)))
        return out


# ---------------------------------------------------------------------------
# reference-shaped free functions (py_module.cpp:56-65, 112-117)
# ---------------------------------------------------------------------------

_layer_cache: dict = {}


def artifact_check(artifact_dir: str, verify_crc: bool = True) -> None:
    """read_artifact's validation alone (io.cpp:186-295,422-485,679-813), on
    the host: raises the same TileqError subclass and message tq_layer_load
    would, without touching a device."""
    check(lib().tq_artifact_check(os.fsencode(artifact_dir), int(verify_crc)))


def route(x, gate_weights, top_k: int):
    """route(x, gate_weights, top_k) -> (int64 ids, float32 gates), computed on the GPU."""
    torch = _torch()
    xa = np.ascontiguousarray(x, dtype=np.float32)
    ga = np.ascontiguousarray(gate_weights, dtype=np.float32)
    if xa.ndim != 2 or ga.ndim != 2:
        raise ParamError("x and gate_weights must be 2-D float arrays")
    K = ga.shape[0]
    if top_k < 1 or top_k > K:
        raise ParamError(f"route: top_k {top_k} outside [1, {K}]")
    if xa.shape[1] != ga.shape[1]:
        raise ShapeError(f"route: token width {xa.shape[1]} vs gate width {ga.shape[1]}")
    dev = torch.device("cuda", torch.cuda.current_device())
    xd = torch.from_numpy(xa).to(dev)
    gd = torch.from_numpy(ga).to(dev)
    B = xa.shape[0]
    ids = torch.empty((B, top_k), dtype=torch.int32, device=dev)
    gates = torch.empty((B, top_k), dtype=torch.float32, device=dev)
    check(lib().tq_route_raw(xd.data_ptr(), B, xa.shape[1], gd.data_ptr(), K, top_k, ids.data_ptr(),
                             gates.data_ptr(), _stream_ptr(dev)))
    return ids.cpu().numpy().astype(np.int64), gates.cpu().numpy()


def forward_from_artifact(artifact_dir: str, x) -> np.ndarray:
    """Load an artifact (cached per directory) and run route + tileq_forward on the GPU."""
    key = os.path.abspath(artifact_dir)
    layer = _layer_cache.get(key)
    if layer is None:
        layer = Layer(artifact_dir)
        _layer_cache[key] = layer
    return layer.forward_host(np.asarray(x, dtype=np.float32))


def unpack_codes_gpu(packed: np.ndarray, bits: int, count: int) -> np.ndarray:
    """unpack_codes (codec.cpp:168-195) on the GPU; raises FormatError on dirty padding."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    pb = torch.from_numpy(np.ascontiguousarray(packed, np.uint8)).to(dev)
    out = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
    check(lib().tq_unpack_codes(pb.data_ptr(), pb.numel(), int(bits), int(count), out.data_ptr(),
                                _stream_ptr(dev)))
    return out[:count].cpu().numpy().astype(np.uint32)


__all__ = ["TileqError", "ShapeError", "ParamError", "SizeError", "FormatError", "IoError",
           "NumericError", "DataError", "CudaError", "NcclError", "Layer", "route",
           "forward_from_artifact", "unpack_codes_gpu", "lib", "PATH_FULL", "PATH_QMOE", "PATH_LOTILE"]
