"""TEST INFRASTRUCTURE ONLY -- the checker, never the product.

Python access to the two CPU checkers:

* ``Oracle``  -- our plain-C restatement (oracle/tileq_oracle.c, built into
  oracle/_build/liboracle.so), each function citing the reference file:line
  it follows.
* ``RefLib``  -- the unmodified reference library compiled from
  /root/reference/proj/src (oracle/_ref/libtileq_ref.so, see oracle/Makefile)
  behind the extern "C" veneer oracle/ref_shim.cpp.

plus ``read_artifact_np``: a numpy reader of the reference's packed artifact
format (io.cpp:679-813) used to feed the oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module.  The product (paper_2605_09281_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtileq_ref.so")

_i64 = C.c_int64
_p = C.c_void_p


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


# --------------------------------------------------------------------------
# artifact reader (numpy)
# --------------------------------------------------------------------------

class ArtifactError(Exception):
    pass


def _packed_len(count: int, bits: int) -> int:
    return (count * bits + 7) // 8


def read_artifact_np(path: str, verify_crc: bool = True) -> dict:
    """Read a 'tileq_artifact' container into numpy arrays (io.cpp:679-813)."""
    with open(os.path.join(path, "manifest.json"), "rb") as f:
        man = json.loads(f.read())
    if man.get("format_version") != 1 or man.get("kind") != "tileq_artifact":
        raise ArtifactError("not a format_version 1 tileq_artifact")
    tens = man["tensors"]

    def blob(name):
        ent = tens[name]
        with open(os.path.join(path, ent["file"]), "rb") as f:
            data = f.read()
        if len(data) != ent["byte_length"]:
            raise ArtifactError(f"tensor '{name}': length mismatch")
        if verify_crc and (zlib.crc32(data) & 0xFFFFFFFF) != ent["crc32"]:
            raise ArtifactError(f"tensor '{name}': checksum mismatch")
        return data, ent

    meta = man["meta"]
    spec = meta["spec"]
    K, top_k, i, o, S = (spec[k] for k in ("num_experts", "top_k", "in_dim", "out_dim", "num_shared"))
    til = meta["tiling"]
    M, N, r = til["grid_rows"], til["grid_cols"], til["rank"]
    out = dict(meta=meta, K=K, top_k=top_k, i=i, o=o, S=S, M=M, N=N, r=r)
    out["gate"] = np.frombuffer(blob("gate_weights")[0], np.float32).reshape(K, i).copy()
    out["scaling"] = np.frombuffer(blob("scaling")[0], np.float32).reshape(K, i).copy()
    out["placement"] = np.frombuffer(blob("placement")[0], np.uint16).reshape(K, 2).copy()
    out["singulars"] = np.frombuffer(blob("tiled.singulars")[0], np.uint16).copy()
    out["u_codes"] = np.frombuffer(blob("tiled.u.codes")[0], np.int8).reshape(M, o, r).copy()
    out["u_absmax"] = np.frombuffer(blob("tiled.u.absmax")[0], np.float32).copy()
    out["v_codes"] = np.frombuffer(blob("tiled.v.codes")[0], np.int8).reshape(N, r, i).copy()
    out["v_absmax"] = np.frombuffer(blob("tiled.v.absmax")[0], np.float32).copy()

    def quant(prefix, qmeta):
        if qmeta["mode"] != "scalar":
            raise ArtifactError("vector mode not handled by the numpy reader")
        bits, g = qmeta["bits"], qmeta["group_size"]
        groups = (i + g - 1) // g
        codes = np.frombuffer(blob(prefix + ".codes")[0], np.uint8).copy()
        scales = np.frombuffer(blob(prefix + ".scales")[0], np.uint16).reshape(o, groups).copy()
        zb = np.frombuffer(blob(prefix + ".zeros")[0], np.uint8).copy()
        zeros = unpack_np(zb, bits, o * groups).reshape(o, groups)
        return dict(packed=codes, scales=scales, zeros=zeros.astype(np.uint32), bits=bits, group_size=g)

    out["experts"] = [quant(f"expert.{e}", meta["quant"]) for e in range(K)]
    out["shared"] = [quant(f"sharedexpert.{s}", meta["shared_quant"]) for s in range(S)]
    return out


def unpack_np(packed: np.ndarray, bits: int, count: int) -> np.ndarray:
    """Vectorised unpack_codes (codec.cpp:168-195) for fixtures; LSB-first."""
    bitsarr = np.unpackbits(np.asarray(packed, np.uint8), bitorder="little")
    need = count * bits
    if bitsarr[need:].any():
        raise ArtifactError("nonzero padding bits")
    b = bitsarr[:need].reshape(count, bits).astype(np.uint32)
    return (b << np.arange(bits, dtype=np.uint32)).sum(axis=1).astype(np.uint32)


def pack_np(codes: np.ndarray, bits: int) -> np.ndarray:
    """Vectorised pack_codes (codec.cpp:150-166)."""
    codes = np.asarray(codes, np.uint32).ravel()
    b = ((codes[:, None] >> np.arange(bits, dtype=np.uint32)) & 1).astype(np.uint8).ravel()
    return np.packbits(b, bitorder="little")


# --------------------------------------------------------------------------
# the C restatement
# --------------------------------------------------------------------------

class _QMat(C.Structure):
    _fields_ = [("packed", _p), ("scales", _p), ("zeros", _p), ("bits", C.c_int),
                ("group_size", _i64)]


class _Tiled(C.Structure):
    _fields_ = [("rank", _i64), ("grid_rows", _i64), ("grid_cols", _i64),
                ("placement", _p), ("u_codes", _p), ("u_absmax", _p), ("v_codes", _p),
                ("v_absmax", _p), ("singulars", _p), ("scaling", _p)]


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        self.lib = C.CDLL(path)
        L = self.lib
        L.tqo_half_to_float.restype = C.c_float
        L.tqo_half_to_float.argtypes = [C.c_uint16]
        L.tqo_float_to_half.restype = C.c_uint16
        L.tqo_float_to_half.argtypes = [C.c_float]
        L.tqo_crc32.restype = C.c_uint32
        L.tqo_crc32.argtypes = [_p, _i64]
        L.tqo_unpack_codes.argtypes = [_p, _i64, C.c_int, _i64, _p]
        L.tqo_pack_codes.argtypes = [_p, _i64, C.c_int, _p]
        L.tqo_route.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p, _p]
        L.tqo_permute.argtypes = [_p, _i64, _i64, _i64, _p, _p, _p]
        L.tqo_qmoe_forward.argtypes = [_p, _i64, _i64, _i64, _i64, _i64, _i64, _p, _p, _p,
                                       _i64, _i64, _p]
        L.tqo_lotile_forward.argtypes = [_p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p,
                                         _i64, _i64, _p]
        L.tqo_dequantize_rows.argtypes = [_p, _i64, _i64, _i64, _i64, _p]
        L.tqo_spd_inverse.argtypes = [_p, _i64, _p, _p, _p]

    def spd_inverse(self, h):
        """quant.cpp:72-112 -> (hinv f64, None) or (None, (column, pivot)) on a bad pivot."""
        h = np.ascontiguousarray(h, np.float32)
        n = h.shape[0]
        out = np.zeros((n, n), np.float64)
        col = C.c_int64(0)
        piv = C.c_double(0.0)
        st = self.lib.tqo_spd_inverse(_ptr(h), n, _ptr(out), C.byref(col), C.byref(piv))
        if st == 6:
            return None, (col.value, piv.value)
        if st:
            raise MemoryError("tqo_spd_inverse")
        return out, None

    def half_to_float(self, bits: int) -> float:
        return self.lib.tqo_half_to_float(bits)

    def float_to_half(self, v: float) -> int:
        return self.lib.tqo_float_to_half(v)

    def crc32(self, data: bytes) -> int:
        a = np.frombuffer(data, np.uint8)
        return self.lib.tqo_crc32(_ptr(a), a.size)

    def unpack(self, packed: np.ndarray, bits: int, count: int) -> tuple[int, np.ndarray]:
        packed = np.ascontiguousarray(packed, np.uint8)
        out = np.zeros(count, np.uint32)
        st = self.lib.tqo_unpack_codes(_ptr(packed), packed.size, bits, count, _ptr(out))
        return st, out

    def pack(self, codes: np.ndarray, bits: int) -> np.ndarray:
        codes = np.ascontiguousarray(codes, np.uint32)
        out = np.zeros(_packed_len(codes.size, bits), np.uint8)
        st = self.lib.tqo_pack_codes(_ptr(codes), codes.size, bits, _ptr(out))
        if st:
            raise ValueError(f"pack status {st}")
        return out

    def route(self, x: np.ndarray, gate: np.ndarray, top_k: int):
        x = np.ascontiguousarray(x, np.float32)
        gate = np.ascontiguousarray(gate, np.float32)
        B, i = x.shape
        K = gate.shape[0]
        ids = np.zeros((B, top_k), np.int64)
        gates = np.zeros((B, top_k), np.float32)
        st = self.lib.tqo_route(_ptr(x), B, i, _ptr(gate), K, top_k, _ptr(ids), _ptr(gates))
        if st:
            raise ValueError(f"route status {st}")
        return ids, gates

    def permute(self, ids: np.ndarray, num_experts: int):
        ids = np.ascontiguousarray(ids, np.int64)
        B, k = ids.shape
        perm = np.zeros(B * k, np.int32)
        inv = np.zeros(B * k, np.int32)
        offs = np.zeros(num_experts + 1, np.int32)
        st = self.lib.tqo_permute(_ptr(ids), B, k, num_experts, _ptr(perm), _ptr(offs), _ptr(inv))
        if st:
            raise ValueError(f"permute status {st}")
        return perm, offs, inv

    @staticmethod
    def _qmats(art):
        mats = art["experts"] + art["shared"]
        arr = (_QMat * len(mats))()
        keep = []
        for k, q in enumerate(mats):
            packed = np.ascontiguousarray(q["packed"], np.uint8)
            scales = np.ascontiguousarray(q["scales"], np.uint16)
            zeros = np.ascontiguousarray(q["zeros"], np.uint32)
            keep += [packed, scales, zeros]
            arr[k] = _QMat(_ptr(packed), _ptr(scales), _ptr(zeros), q["bits"], q["group_size"])
        return arr, keep

    def dequantize(self, art, e: int, r0: int = 0, r1: int | None = None) -> np.ndarray:
        r1 = art["o"] if r1 is None else r1
        arr, keep = self._qmats(art)
        out = np.zeros((r1 - r0, art["i"]), np.float32)
        self.lib.tqo_dequantize_rows(C.byref(arr[e]), art["o"], art["i"], r0, r1, _ptr(out))
        return out

    def qmoe_forward(self, art, x, ids, gates, r0=0, r1=None):
        r1 = art["o"] if r1 is None else r1
        x = np.ascontiguousarray(x, np.float32)
        ids = np.ascontiguousarray(ids, np.int64)
        gates = np.ascontiguousarray(gates, np.float32)
        arr, keep = self._qmats(art)
        y = np.zeros((x.shape[0], r1 - r0), np.float32)
        st = self.lib.tqo_qmoe_forward(_ptr(x), x.shape[0], art["i"], art["o"], art["K"], art["S"],
                                       art["top_k"], arr, _ptr(ids), _ptr(gates), r0, r1, _ptr(y))
        if st:
            raise ValueError(f"qmoe status {st}")
        return y

    def lotile_forward(self, art, x, ids, gates, r0=0, r1=None):
        r1 = art["o"] if r1 is None else r1
        x = np.ascontiguousarray(x, np.float32)
        ids = np.ascontiguousarray(ids, np.int64)
        gates = np.ascontiguousarray(gates, np.float32)
        keep = [np.ascontiguousarray(art[k]) for k in
                ("placement", "u_codes", "u_absmax", "v_codes", "v_absmax", "singulars", "scaling")]
        t = _Tiled(art["r"], art["M"], art["N"], *[_ptr(a) for a in keep])
        y = np.zeros((x.shape[0], r1 - r0), np.float32)
        st = self.lib.tqo_lotile_forward(_ptr(x), x.shape[0], art["i"], art["o"], art["K"],
                                         art["top_k"], C.byref(t), _ptr(ids), _ptr(gates),
                                         r0, r1, _ptr(y))
        if st:
            raise ValueError(f"lotile status {st}")
        return y

    def tileq_forward(self, art, x, r0=0, r1=None):
        """route + qmoe + lotile, summed in f32 (infer.cpp:182-185)."""
        ids, gates = self.route(x, art["gate"], art["top_k"])
        a = self.qmoe_forward(art, x, ids, gates, r0, r1)
        b = self.lotile_forward(art, x, ids, gates, r0, r1)
        return (a + b).astype(np.float32), ids, gates


# --------------------------------------------------------------------------
# the compiled reference
# --------------------------------------------------------------------------

class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class RefLib:
    """ctypes access to the unmodified reference (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)
        L = self.lib
        L.tq_ref_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(_p), C.c_char_p, C.c_int]
        L.tq_ref_free.argtypes = [_p]
        L.tq_ref_spec.argtypes = [_p, _p]
        L.tq_ref_forward.argtypes = [_p, _p, _i64, C.c_int, C.c_int, _p, _p, _p, C.c_char_p, C.c_int]
        L.tq_ref_route.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p, _p, C.c_char_p, C.c_int]
        L.tq_ref_unpack.argtypes = [_p, _i64, C.c_int, _i64, _p, C.c_char_p, C.c_int]
        L.tq_ref_pack.argtypes = [_p, _i64, C.c_int, _p, C.c_char_p, C.c_int]
        L.tq_ref_f16_to_f32.argtypes = [_p, _i64, _p]
        L.tq_ref_f32_to_f16.argtypes = [_p, _i64, _p]
        L.tq_ref_dequantize.argtypes = [_p, _i64, _p, C.c_char_p, C.c_int]
        L.tq_ref_reconstruct.argtypes = [_p, _i64, _p, C.c_char_p, C.c_int]
        L.tq_ref_layout.argtypes = [_p, C.c_int, _p, _i64, _p, _p, _p, _p, C.c_char_p, C.c_int]
        L.tq_ref_bench.argtypes = [_p, C.c_int, _p, _i64, _i64, _i64, C.c_uint64, _p, C.c_char_p, C.c_int]
        L.tq_ref_make_artifact.argtypes = [C.c_char_p] + [_i64] * 8 + [C.c_int, _i64, C.c_int, _i64,
                                           C.c_double, C.c_double, _i64, C.c_uint64, C.c_int,
                                           C.c_int, _i64, C.c_char_p, C.c_int]
        L.tq_ref_estimate_hessian.argtypes = [_p, _i64, _i64, C.c_double, _p, _p, C.c_char_p, C.c_int]
        L.tq_ref_quantize.argtypes = [C.c_int, _p, _i64, _i64, _p, C.c_int, _i64, _p, _p, _p, C.c_char_p, C.c_int]
        L.tq_ref_proxy_loss.argtypes = [_p, _i64, _i64, _p, _p, _p, C.c_int, _i64, _p, _p, C.c_char_p, C.c_int]
        L.tq_ref_sketch_lowrank.argtypes = [_p, _i64, _i64, _i64, C.c_int, C.c_uint64, _p, _p, _p, C.c_char_p,
                                            C.c_int]

    def _check(self, st, buf):
        if st:
            raise RefError(st, buf.value.decode(errors="replace"))

    def load(self, path: str, verify_crc: bool = True) -> "RefLayer":
        h = _p()
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_load(path.encode(), int(verify_crc), C.byref(h), buf, 1024), buf)
        return RefLayer(self, h)

    def route(self, x, gate, top_k):
        x = np.ascontiguousarray(x, np.float32)
        gate = np.ascontiguousarray(gate, np.float32)
        ids = np.zeros((x.shape[0], top_k), np.int64)
        gates = np.zeros((x.shape[0], top_k), np.float32)
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_route(_ptr(x), x.shape[0], x.shape[1], _ptr(gate), gate.shape[0],
                                          top_k, _ptr(ids), _ptr(gates), buf, 1024), buf)
        return ids, gates

    def unpack(self, packed, bits, count):
        packed = np.ascontiguousarray(packed, np.uint8)
        out = np.zeros(count, np.uint32)
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_unpack(_ptr(packed), packed.size, bits, count, _ptr(out), buf, 1024), buf)
        return out

    def pack(self, codes, bits):
        codes = np.ascontiguousarray(codes, np.uint32)
        out = np.zeros(_packed_len(codes.size, bits), np.uint8)
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_pack(_ptr(codes), codes.size, bits, _ptr(out), buf, 1024), buf)
        return out

    # -- artifact producer hot spots (quant.cpp:116-221,325-343) --
    def estimate_hessian(self, calib, damping_fraction):
        calib = np.ascontiguousarray(calib, np.float32)
        h = np.zeros((calib.shape[1], calib.shape[1]), np.float32)
        lam = C.c_double(0.0)
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_estimate_hessian(_ptr(calib), calib.shape[0], calib.shape[1],
                                                     damping_fraction, _ptr(h), C.byref(lam), buf, 1024), buf)
        return h, lam.value

    def quantize(self, method, r, h, bits, group_size):
        """method "rtn" (quantize_rtn) or "gptq" (quantize_gptq): (codes u32, scales f32, zeros i32)."""
        r = np.ascontiguousarray(r, np.float32)
        rows, cols = r.shape
        G = (cols + group_size - 1) // group_size if group_size >= 1 else 0
        codes = np.zeros((rows, cols), np.uint32)
        scales = np.zeros((rows, G), np.float32)
        zeros = np.zeros((rows, G), np.int32)
        hp = None
        if method == "gptq":
            h = np.ascontiguousarray(h, np.float32)
            hp = _ptr(h)
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_quantize(0 if method == "rtn" else 1, _ptr(r), rows, cols, hp, bits, group_size,
                                             _ptr(codes), _ptr(scales), _ptr(zeros), buf, 1024), buf)
        return codes, scales, zeros

    def proxy_loss(self, original, codes, scales, zeros, bits, group_size, h):
        original = np.ascontiguousarray(original, np.float32)
        codes = np.ascontiguousarray(codes, np.uint32)
        scales = np.ascontiguousarray(scales, np.float32)
        zeros = np.ascontiguousarray(zeros, np.int32)
        h = np.ascontiguousarray(h, np.float32)
        out = C.c_double(0.0)
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_proxy_loss(_ptr(original), original.shape[0], original.shape[1], _ptr(codes),
                                               _ptr(scales), _ptr(zeros), bits, group_size, _ptr(h),
                                               C.byref(out), buf, 1024), buf)
        return out.value

    def sketch_lowrank(self, w, rank, power_iters, seed):
        """sketch_lowrank (lowrank.cpp:194-247) -> (left, singulars, right) f32."""
        w = np.ascontiguousarray(w, np.float32)
        rows, cols = w.shape
        left = np.zeros((rows, rank), np.float32)
        right = np.zeros((rank, cols), np.float32)
        sing = np.zeros(rank, np.float32)
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_sketch_lowrank(_ptr(w), rows, cols, rank, power_iters, seed, _ptr(left),
                                                   _ptr(right), _ptr(sing), buf, 1024), buf)
        return left, sing, right

    def f16_to_f32(self, bits):
        bits = np.ascontiguousarray(bits, np.uint16)
        out = np.zeros(bits.size, np.float32)
        self.lib.tq_ref_f16_to_f32(_ptr(bits), bits.size, _ptr(out))
        return out

    def f32_to_f16(self, v):
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros(v.size, np.uint16)
        self.lib.tq_ref_f32_to_f16(_ptr(v), v.size, _ptr(out))
        return out

    def make_artifact(self, path, *, K, top_k, i, o, S=0, M=0, N=0, r=16, bits=3, g=128,
                      calib="signs", calib_tokens=256, noise=0.05, mix_scale=1.0,
                      planted_rank=8, seed=1, full_pipeline=False, quantizer="rtn", sub_dim=2):
        kind = {"signs": 0, "gauss": 1, "none": 2}[calib]
        qz = {"rtn": 0, "gptq": 1, "vq": 2}[quantizer]
        buf = C.create_string_buffer(1024)
        self._check(self.lib.tq_ref_make_artifact(
            path.encode(), K, top_k, i, o, S, M, N, r, bits, g, kind, calib_tokens, noise,
            mix_scale, planted_rank, seed, int(full_pipeline), qz, sub_dim, buf, 1024), buf)
        return path


class RefLayer:
    def __init__(self, ref: RefLib, handle):
        self.ref, self.h = ref, handle
        spec = np.zeros(6, np.int64)
        ref.lib.tq_ref_spec(self.h, _ptr(spec))
        self.K, self.top_k, self.i, self.o, self.S, self.r = (int(v) for v in spec)

    def __del__(self):
        try:
            self.ref.lib.tq_ref_free(self.h)
        except Exception:
            pass

    def forward(self, x, mode: int = 0, threads: int = 1):
        """mode 0 tileq_forward, 1 qmoe_forward, 2 lotile_forward; route() first."""
        x = np.ascontiguousarray(x, np.float32)
        B = x.shape[0]
        y = np.zeros((B, self.o), np.float32)
        ids = np.zeros((B, self.top_k), np.int64)
        gates = np.zeros((B, self.top_k), np.float32)
        buf = C.create_string_buffer(1024)
        self.ref._check(self.ref.lib.tq_ref_forward(self.h, _ptr(x), B, mode, threads, _ptr(y),
                                                    _ptr(ids), _ptr(gates), buf, 1024), buf)
        return y, ids, gates

    LAYOUTS = ("fused_2d", "shared_1d", "element_wise", "dequant_only")

    def layout(self, layout: str, x, ids, gates):
        """The paper's comparison layouts on a given routing (infer.cpp:187-339):
        returns (y, dispatch_count); dequant_only returns (None, count)."""
        x = np.ascontiguousarray(x, np.float32)
        ids = np.ascontiguousarray(ids, np.int64)
        gates = np.ascontiguousarray(gates, np.float32)
        B = x.shape[0]
        y = np.zeros((B, self.o), np.float32)
        disp = np.zeros(1, np.int64)
        buf = C.create_string_buffer(1024)
        self.ref._check(self.ref.lib.tq_ref_layout(self.h, self.LAYOUTS.index(layout), _ptr(x), B, _ptr(ids),
                                                   _ptr(gates), _ptr(y), _ptr(disp), buf, 1024), buf)
        return (None if layout == "dequant_only" else y), int(disp[0])

    def bench(self, layout: str, batches, repeats=5, warmup=1, seed=1):
        """The reference's bench() (infer.cpp:371-426): {batch: (median_ns, p10_ns, p90_ns, dispatches)}."""
        bs = np.ascontiguousarray(batches, np.int64)
        out = np.zeros(4 * len(bs), np.float64)
        buf = C.create_string_buffer(1024)
        self.ref._check(self.ref.lib.tq_ref_bench(self.h, self.LAYOUTS.index(layout), _ptr(bs), len(bs), repeats,
                                                  warmup, C.c_uint64(seed), _ptr(out), buf, 1024), buf)
        return {int(b): tuple(out[4 * t:4 * t + 4]) for t, b in enumerate(bs)}

    def dequantize(self, e):
        out = np.zeros((self.o, self.i), np.float32)
        buf = C.create_string_buffer(1024)
        self.ref._check(self.ref.lib.tq_ref_dequantize(self.h, e, _ptr(out), buf, 1024), buf)
        return out

    def reconstruct(self, e):
        out = np.zeros((self.o, self.i), np.float32)
        buf = C.create_string_buffer(1024)
        self.ref._check(self.ref.lib.tq_ref_reconstruct(self.h, e, _ptr(out), buf, 1024), buf)
        return out


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def gaussian_tokens(batch: int, in_dim: int, seed: int) -> np.ndarray:
    """x = gaussian_matrix(B, i, CounterRng(derive(seed, B))) as the reference
    bench draws it (infer.cpp:389-391, rng.hpp:14-66), restated in numpy."""
    return counter_rng_gaussians(derive(seed, batch), batch * in_dim).reshape(batch, in_dim)


# splitmix64 counter RNG (rng.hpp:14-66), vectorised for fixture generation.
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z):
    z = np.asarray(z, np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def derive(seed: int, stream: int) -> int:
    with np.errstate(over="ignore"):
        return int(_mix(np.uint64(seed) ^ _mix(np.uint64(stream) + _GAMMA)))


def counter_rng_gaussians(seed: int, count: int) -> np.ndarray:
    """CounterRng(seed).next_gaussian() x count, as f32 (Box-Muller pairs: cos first, then sin)."""
    npairs = (count + 1) // 2
    ctr = np.arange(1, 2 * npairs + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        raw = _mix(np.uint64(seed) + ctr * _GAMMA)
    unit = (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    u1 = 1.0 - unit[0::2]
    u2 = unit[1::2]
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 6.283185307179586476925286766559 * u2
    out = np.empty(2 * npairs, np.float64)
    out[0::2] = rad * np.cos(ang)
    out[1::2] = rad * np.sin(ang)
    return out[:count].astype(np.float32)
