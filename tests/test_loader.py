"""Artifact loader fault injection (CPU): the engine's read_artifact checks
against the reference's own, case by case.

Ports the corruption cases of the reference's tests/test_io.cpp:196-218
(manifest-level failures), :268-280 (checksums name the tensor), :282-319
(placement bounds, injectivity, L1 displacement), :336-341 (container kind),
plus the per-tensor checks of io.cpp:222-261,422-485 (dtype, byte_length,
blob size, missing tensor / blob, quant meta, dirty zero-point padding,
non-positive scales).  Each corrupted artifact is fed to

  * the engine's host-side validation, `tq_artifact_check` (the same code
    `tq_layer_load` runs before it touches a device), and
  * the unmodified reference's read_artifact (oracle/_ref),

and both must fail with the same error class (errors.hpp:13-50 <-> tq_status)
and the same message.  No GPU is involved: validation precedes device init.
"""
import json
import os
import shutil

import numpy as np
import pytest

from conftest import REPO

GOLD = os.path.join(REPO, "tests", "golden")

# tq_status / errors.hpp class codes (RefError.code uses the same numbering)
SHAPE, PARAM, SIZE, FORMAT, IO = 1, 2, 3, 4, 5


@pytest.fixture(scope="module")
def tq():
    import paper_2605_09281_b200 as tq
    return tq


def _copy(tmp_path, name, src="scalar_b4_ragged"):
    d = tmp_path / name
    shutil.copytree(os.path.join(GOLD, src), d)
    return d


def _manifest(d):
    with open(d / "manifest.json") as f:
        return json.load(f)


def _write_manifest(d, m):
    with open(d / "manifest.json", "w") as f:
        f.write(json.dumps(m, indent=2, sort_keys=True) + "\n")


def _engine_error(tq, d, verify=True):
    try:
        tq.artifact_check(str(d), verify_crc=verify)
    except tq.TileqError as e:
        return type(e), str(e)
    return None, None


def _ref_error(ref, d, verify=True):
    from oracle.oracle import RefError
    try:
        ref.load(str(d), verify_crc=verify)
    except RefError as e:
        return e.code, str(e).split("] ", 1)[1]
    return None, None


def _expect(tq, ref, d, code, needle, verify=True, same_message=True):
    cls = {SHAPE: tq.ShapeError, PARAM: tq.ParamError, SIZE: tq.SizeError, FORMAT: tq.FormatError, IO: tq.IoError}[code]
    got_cls, got_msg = _engine_error(tq, d, verify)
    assert got_cls is cls, (got_cls, got_msg)
    assert needle in got_msg, got_msg
    if ref is not None:
        rcode, rmsg = _ref_error(ref, d, verify)
        assert rcode == code, (rcode, rmsg)
        assert needle in rmsg, rmsg
        if same_message:
            assert got_msg == rmsg, (got_msg, rmsg)
    return got_msg


@pytest.fixture(scope="module")
def refl():
    from oracle.oracle import RefLib, ref_available
    return RefLib() if ref_available() else None


def test_clean_artifacts_pass(tq, refl):
    for name in ("folded_b3", "general_b8", "general_b2_shared", "scalar_b4_ragged"):
        tq.artifact_check(os.path.join(GOLD, name))
        if refl is not None:
            refl.load(os.path.join(GOLD, name))


# --- test_io.cpp:196-218 ------------------------------------------------------

def test_missing_directory_is_io_error(tq, refl, tmp_path):
    _expect(tq, refl, tmp_path / "nope", IO, "cannot open")


def test_unsupported_format_version(tq, refl, tmp_path):
    d = _copy(tmp_path, "ver")
    m = _manifest(d)
    m["format_version"] += 1
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "format_version")


def test_garbage_manifest(tq, refl, tmp_path):
    d = _copy(tmp_path, "junk")
    (d / "manifest.json").write_bytes(b"junk")
    # the JSON parser's own wording differs between nlohmann builds: class + prefix only
    _expect(tq, refl, d, FORMAT, "manifest is not valid JSON", same_message=False)


# --- test_io.cpp:336-341 ------------------------------------------------------

def test_container_kind_is_checked(tq, refl, tmp_path):
    d = _copy(tmp_path, "kind")
    m = _manifest(d)
    m["kind"] = "tileq_model"
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "tileq_artifact")


# --- test_io.cpp:268-280 ------------------------------------------------------

def test_checksum_names_the_tensor(tq, refl, tmp_path):
    d = _copy(tmp_path, "crc")
    p = d / "expert.2.codes.bin"
    b = bytearray(p.read_bytes())
    b[0] ^= 0xFF
    p.write_bytes(bytes(b))
    _expect(tq, refl, d, FORMAT, "expert.2.codes")
    # 4-bit codes fill bytes exactly: with verification off the flipped byte decodes
    tq.artifact_check(str(d), verify_crc=False)
    if refl is not None:
        refl.load(str(d), verify_crc=False)


@pytest.mark.parametrize("blob", ["gate_weights", "scaling", "placement", "tiled.singulars", "tiled.u.codes",
                                  "tiled.v.absmax", "expert.4.scales", "expert.0.zeros"])
def test_checksum_every_tensor(tq, refl, tmp_path, blob):
    d = _copy(tmp_path, "crc_" + blob)
    p = d / (blob + ".bin")
    b = bytearray(p.read_bytes())
    b[len(b) // 2] ^= 0x01
    p.write_bytes(bytes(b))
    _expect(tq, refl, d, FORMAT, f"tensor '{blob}': checksum mismatch")


# --- test_io.cpp:282-319 ------------------------------------------------------

def test_placement_out_of_grid(tq, refl, tmp_path):
    d = _copy(tmp_path, "pl_bounds")
    p = d / "placement.bin"
    b = bytearray(p.read_bytes())
    b[0] = 9
    p.write_bytes(bytes(b))
    _expect(tq, refl, d, FORMAT, "outside the tile grid", verify=False)


def test_placement_duplicate_cell(tq, refl, tmp_path):
    d = _copy(tmp_path, "pl_dup")
    p = d / "placement.bin"
    b = bytearray(p.read_bytes())
    b[4:8] = b[0:4]
    p.write_bytes(bytes(b))
    _expect(tq, refl, d, FORMAT, "injective", verify=False)


def test_placement_l1_displacement(tq, refl, tmp_path):
    d = _copy(tmp_path, "pl_l1")
    m = _manifest(d)
    m["meta"]["tiling"]["total_l1_displacement"] += 1
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "total_l1_displacement")


# --- per-tensor checks (io.cpp:222-261) -------------------------------------

def test_truncated_blob(tq, refl, tmp_path):
    d = _copy(tmp_path, "trunc")
    p = d / "expert.1.scales.bin"
    p.write_bytes(p.read_bytes()[:-4])
    _expect(tq, refl, d, FORMAT, "tensor 'expert.1.scales': blob is")


def test_missing_blob_file(tq, refl, tmp_path):
    d = _copy(tmp_path, "noblob")
    os.remove(d / "tiled.u.absmax.bin")
    _expect(tq, refl, d, IO, "tensor 'tiled.u.absmax': cannot stat")


def test_missing_tensor_entry(tq, refl, tmp_path):
    d = _copy(tmp_path, "noentry")
    m = _manifest(d)
    del m["tensors"]["expert.3.zeros"]
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "missing tensor 'expert.3.zeros'")


def test_wrong_dtype(tq, refl, tmp_path):
    d = _copy(tmp_path, "dtype")
    m = _manifest(d)
    m["tensors"]["scaling"]["dtype"] = "u16"
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "tensor 'scaling': dtype is 'u16', expected 'f32'")


def test_byte_length_inconsistent_with_shape(tq, refl, tmp_path):
    d = _copy(tmp_path, "blen")
    m = _manifest(d)
    m["tensors"]["tiled.v.codes"]["shape"][2] += 1
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "tensor 'tiled.v.codes': byte_length does not match shape/dtype")


def test_wrong_shape_consistent_length(tq, refl, tmp_path):
    d = _copy(tmp_path, "shape")
    m = _manifest(d)
    t = m["tensors"]["gate_weights"]
    t["shape"] = [t["shape"][1], t["shape"][0]]
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "tensor 'gate_weights': expected shape")


# --- quantized residuals (io.cpp:422-485) ----------------------------------

def test_bad_bits_in_quant_meta(tq, refl, tmp_path):
    d = _copy(tmp_path, "bits")
    m = _manifest(d)
    m["meta"]["quant"]["bits"] = 5
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "bits must be one of 2, 3, 4, 8")


def test_unknown_quant_mode(tq, refl, tmp_path):
    d = _copy(tmp_path, "mode")
    m = _manifest(d)
    m["meta"]["quant"]["mode"] = "lattice"
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "unknown mode 'lattice'")


def test_zero_group_size(tq, refl, tmp_path):
    d = _copy(tmp_path, "gs0")
    m = _manifest(d)
    m["meta"]["quant"]["group_size"] = 0
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "group_size must be >= 1")


def test_non_positive_scale(tq, refl, tmp_path):
    d = _copy(tmp_path, "scale0")
    p = d / "expert.3.scales.bin"
    b = bytearray(p.read_bytes())
    b[6:8] = b"\x00\x80"          # -0.0
    p.write_bytes(bytes(b))
    _expect(tq, refl, d, FORMAT, "tensor 'expert.3.scales': non-positive scale", verify=False)


def test_dirty_zero_point_padding(tq, refl, tmp_path):
    from paper_2605_09281_b200 import synth
    # o = 41 rows x 2 groups of 3-bit zero points = 246 bits: 2 pad bits in the last byte
    d = tmp_path / "pad"
    synth.write_synthetic(str(d), K=3, top_k=2, i=256, o=41, bits=3, r=8, group=128, seed=2)
    tq.artifact_check(str(d))
    p = d / "expert.1.zeros.bin"
    b = bytearray(p.read_bytes())
    assert len(b) == 31
    b[-1] |= 0x80
    p.write_bytes(bytes(b))
    _expect(tq, refl, d, FORMAT, "tensor 'expert.1.zeros': packed stream has nonzero padding past code 82",
            verify=False)


def test_shared_expert_names_itself(tq, refl, tmp_path):
    d = _copy(tmp_path, "shared", src="general_b2_shared")
    p = d / "sharedexpert.0.scales.bin"
    b = bytearray(p.read_bytes())
    b[0] ^= 0x10
    p.write_bytes(bytes(b))
    _expect(tq, refl, d, FORMAT, "sharedexpert.0.scales")


def test_layer_load_reports_host_errors_before_device(tq, tmp_path):
    """tq_layer_load runs the same validation before any CUDA call, so a
    CPU-only process sees the artifact's error, not a device error."""
    d = _copy(tmp_path, "load_crc")
    p = d / "expert.0.codes.bin"
    b = bytearray(p.read_bytes())
    b[3] ^= 0x40
    p.write_bytes(bytes(b))
    with pytest.raises(tq.FormatError, match="expert.0.codes"):
        tq.Layer(str(d))
    with pytest.raises(tq.IoError):
        tq.Layer(str(tmp_path / "missing"))


def test_vector_quantized_artifact_is_read(tq, refl, tmp_path):
    """Codebook residuals (io.cpp:464-480): codes o x ceil(i / sub_dim) and a
    2^bits x sub_dim binary16 codebook per expert; a codebook of the wrong
    shape is a FormatError naming it, like the reference's reader."""
    if refl is None:
        pytest.skip("reference library not built")
    d = tmp_path / "vq"
    refl.make_artifact(str(d), K=4, top_k=2, i=128, o=64, S=1, r=4, bits=2, g=128, calib="gauss", seed=5,
                       quantizer="vq", sub_dim=2)
    tq.artifact_check(str(d))
    refl.load(str(d))
    m = _manifest(d)
    assert m["meta"]["quant"]["mode"] == "vector"
    m["tensors"]["expert.1.codebook"]["shape"] = [8, 1]      # same byte length, wrong shape
    _write_manifest(d, m)
    _expect(tq, refl, d, FORMAT, "expert.1.codebook")
