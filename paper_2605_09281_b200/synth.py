"""Fast synthetic TileQ artifacts in the reference's packed format.

The reference's CPU quantizer (pipeline.cpp:138-230) takes ~1 h on a
Mixtral-shape layer, so the benchmark uses byte-valid synthetic artifacts of
the named shapes instead: random b-bit codes, positive binary16 scales,
packed zero points, int8 factor blocks with f32 absmax, binary16 singular
values, an injective row-major placement and either neutral scaling (folded
descale tier) or random positive scaling (general tier).  The container is
written exactly like write_artifact (io.cpp:565-677): manifest.json
(format_version 1, kind tileq_artifact, keys sorted, dump(2) + newline) plus
one little-endian blob per tensor with its zlib CRC32; the reference's own
read_artifact accepts these files (checked by
tests/test_cpu_oracle.py::test_synthetic_artifact_readable_by_reference).

Throughput does not depend on the numeric content; parity tests use
artifacts produced by the reference pipeline itself.
"""
from __future__ import annotations

import json
import os
import zlib

import numpy as np

CONFIGS = {
    # name: (K, top_k, i, o, S, bits, r, group)
    "c1": (8, 2, 1024, 2816, 0, 3, 16, 128),
    "c2": (8, 2, 4096, 14336, 0, 3, 32, 128),      # Mixtral-8x7B expert-layer shape
    "c3": (8, 2, 4096, 14336, 0, 3, 32, 128),      # same shape, prefill 4096
    "c4": (60, 4, 2048, 1408, 4, 2, 32, 128),      # Qwen1.5-MoE-A2.7B (4 x 1408 shared = 5632)
    "c4s1": (60, 4, 2048, 1408, 1, 2, 32, 128),    # literal "+ shared expert" reading
    "c5": (64, 6, 2048, 1408, 0, 3, 32, 128),      # DeepSeek-V2-Lite
}


def grid_for(K: int) -> tuple[int, int]:
    """TileQConfig auto grid: M = round(sqrt(K)), N = ceil(K / M) (pipeline.cpp:79-82)."""
    m = int(np.floor(np.sqrt(K) + 0.5)) or 1
    return m, (K + m - 1) // m


def _pack(codes: np.ndarray, bits: int) -> bytes:
    codes = np.asarray(codes, np.uint8).ravel()
    if bits == 8:
        return codes.tobytes()
    b = ((codes[:, None] >> np.arange(bits, dtype=np.uint8)) & 1).astype(np.uint8).ravel()
    return np.packbits(b, bitorder="little").tobytes()


def _f16(a: np.ndarray) -> bytes:
    return np.asarray(a, np.float16).view(np.uint16).tobytes()


class _Writer:
    def __init__(self, path: str):
        self.path = path
        self.tensors = {}
        os.makedirs(path, exist_ok=True)

    def add(self, name: str, shape, dtype: str, data: bytes):
        fname = name + ".bin"
        with open(os.path.join(self.path, fname), "wb") as f:
            f.write(data)
        self.tensors[name] = {"byte_length": len(data), "crc32": zlib.crc32(data) & 0xFFFFFFFF,
                              "dtype": dtype, "file": fname, "shape": list(int(s) for s in shape)}

    def finish(self, meta: dict):
        man = {"format_version": 1, "kind": "tileq_artifact", "meta": meta, "tensors": self.tensors}
        text = json.dumps(man, indent=2, sort_keys=True) + "\n"
        with open(os.path.join(self.path, "manifest.json"), "w") as f:
            f.write(text)


def write_synthetic(path: str, *, K: int, top_k: int, i: int, o: int, S: int = 0, bits: int = 3,
                    r: int = 32, group: int = 128, tier: str = "folded", seed: int = 0,
                    weight_scale: float = 0.02) -> str:
    """Write a synthetic artifact; returns `path`.  tier: 'folded' | 'general'."""
    rng = np.random.default_rng(seed)
    M, N = grid_for(K)
    G = (i + group - 1) // group
    w = _Writer(path)
    w.add("gate_weights", (K, i), "f32", rng.standard_normal((K, i), dtype=np.float32).tobytes())
    if tier == "folded":
        scaling = np.ones((K, i), np.float32)
    else:
        scaling = (0.5 + rng.random((K, i), dtype=np.float32)).astype(np.float32)
    w.add("scaling", (K, i), "f32", scaling.tobytes())
    placement = np.array([[e // N, e % N] for e in range(K)], np.uint16)
    w.add("placement", (K, 2), "u16", placement.tobytes())
    sing = (4.0 * 0.85 ** np.arange(r)).astype(np.float16)
    w.add("tiled.singulars", (r,), "f16-roundtrip", _f16(sing))
    u = rng.integers(-127, 128, size=(M, o, r), dtype=np.int8)
    w.add("tiled.u.codes", (M, o, r), "u8", u.view(np.uint8).tobytes())
    w.add("tiled.u.absmax", (M,), "f32", np.full(M, 0.05, np.float32).tobytes())
    v = rng.integers(-127, 128, size=(N, r, i), dtype=np.int8)
    w.add("tiled.v.codes", (N, r, i), "u8", v.view(np.uint8).tobytes())
    w.add("tiled.v.absmax", (N,), "f32", np.full(N, 0.05, np.float32).tobytes())
    q = 1 << bits

    def qmat(prefix):
        codes = rng.integers(0, q, size=(o, i), dtype=np.uint8)
        w.add(prefix + ".codes", (o, i), f"packed-u{bits}", _pack(codes, bits))
        scales = (weight_scale * (0.5 + rng.random((o, G)))).astype(np.float16)
        w.add(prefix + ".scales", (o, G), "f16-roundtrip", _f16(scales))
        zeros = rng.integers(0, q, size=(o, G), dtype=np.uint8)
        w.add(prefix + ".zeros", (o, G), f"packed-u{bits}", _pack(zeros, bits))

    for e in range(K):
        qmat(f"expert.{e}")
    for s in range(S):
        qmat(f"sharedexpert.{s}")
    qm = {"bits": bits, "group_size": group, "mode": "scalar"}
    meta = {"quant": qm,
            "spec": {"in_dim": i, "num_experts": K, "num_shared": S, "out_dim": o, "top_k": top_k},
            "tiling": {"grid_cols": N, "grid_rows": M, "ideal": placement.astype(int).tolist(), "rank": r,
                       "total_l1_displacement": 0},
            "synthetic": {"seed": seed, "tier": tier}}
    if S > 0:
        meta["shared_quant"] = dict(qm)
    w.finish(meta)
    return path


def config_path(name: str, root: str = "/tmp/tileq_artifacts", tier: str = "folded", seed: int = 0) -> str:
    """Cache path of a config's synthetic artifact, keyed by this writer's source
    (a /tmp cache left by an older writer version is never reused)."""
    import hashlib
    with open(os.path.abspath(__file__), "rb") as f:
        key = hashlib.sha1(f.read()).hexdigest()[:10]
    return os.path.join(root, f"{name}_{tier}_s{seed}_{key}")


def ensure_config(name: str, root: str = "/tmp/tileq_artifacts", tier: str = "folded", seed: int = 0) -> str:
    """Synthetic artifact for a BASELINE config (cached by name and writer version)."""
    K, top_k, i, o, S, bits, r, g = CONFIGS[name]
    path = config_path(name, root, tier, seed)
    if not os.path.exists(os.path.join(path, "manifest.json")):
        # written aside and renamed into place: a killed writer never leaves a
        # half-written artifact under the cache name
        tmp = f"{path}.tmp{os.getpid()}"
        write_synthetic(tmp, K=K, top_k=top_k, i=i, o=o, S=S, bits=bits, r=r, group=g, tier=tier, seed=seed)
        try:
            os.rename(tmp, path)
        except OSError:   # another process won the race
            import shutil
            shutil.rmtree(tmp, ignore_errors=True)
    return path
