"""CPU suite: pin the oracle against the reference, check the boundary.

* our C restatement (oracle/tileq_oracle.c) reproduces the reference's
  golden fixtures (tests/golden/, written by the reference itself through
  tests/golden/make_golden.py): routing ids bit-exact, codec bytes and f16
  conversions bit-exact, dequantize exact, forwards within the reference's own
  CPU-vs-CPU verify threshold (rel 1e-5, tileq_main.cpp:277,303);
* the C-ABI library loads without a GPU and exports every symbol
  include/tileq_b200.h declares;
* the synthetic artifacts bench.py times are readable by the reference;
* bench.py's algorithmic byte counts equal SURVEY.md §8's table.
"""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import REPO, rel_frob

GOLD = os.path.join(REPO, "tests", "golden")
ART_NAMES = ["folded_b3", "general_b2_shared", "scalar_b4_ragged", "general_b8"]


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(os.path.join(GOLD, "golden.npz")))


@pytest.mark.parametrize("name", ART_NAMES)
def test_oracle_forward_matches_reference_fixtures(oracle, golden, name):
    from oracle.oracle import read_artifact_np
    art = read_artifact_np(os.path.join(GOLD, name))
    for B in (1, 7, 33):
        x = golden[f"{name}/x{B}"]
        ids, gates = oracle.route(x, art["gate"], art["top_k"])
        np.testing.assert_array_equal(ids, golden[f"{name}/ids{B}"])
        np.testing.assert_array_equal(gates, golden[f"{name}/gates{B}"])
        y, _, _ = oracle.tileq_forward(art, x)
        assert rel_frob(y, golden[f"{name}/tileq{B}"]) <= 1e-5
        yq = oracle.qmoe_forward(art, x, ids, gates)
        np.testing.assert_array_equal(yq, golden[f"{name}/qmoe{B}"])      # same f64 order: bitwise
        yl = oracle.lotile_forward(art, x, ids, gates)
        assert rel_frob(yl, golden[f"{name}/lotile{B}"]) <= 1e-6


@pytest.mark.parametrize("name", ART_NAMES)
def test_oracle_dequantize_exact(oracle, golden, name):
    from oracle.oracle import read_artifact_np
    art = read_artifact_np(os.path.join(GOLD, name))
    for e in range(2):
        np.testing.assert_array_equal(oracle.dequantize(art, e), golden[f"{name}/dequant{e}"])


def test_oracle_route_kats(oracle, golden):
    for t in range(5):
        x, g = golden[f"route{t}/x"], golden[f"route{t}/g"]
        k = golden[f"route{t}/ids"].shape[1]
        ids, gates = oracle.route(x, g, k)
        np.testing.assert_array_equal(ids, golden[f"route{t}/ids"])
        np.testing.assert_array_equal(gates, golden[f"route{t}/gates"])
    # frozen cases of test_moe.cpp:110-130
    x = np.zeros((1, 3), np.float32)
    x[0, 0] = 1.0
    g = np.zeros((4, 3), np.float32)
    g[2, 0] = 50.0
    ids, gates = oracle.route(x, g, 1)
    assert ids[0, 0] == 2 and gates[0, 0] == 1.0
    ids, gates = oracle.route(np.ones((2, 5), np.float32), np.zeros((4, 5), np.float32), 2)
    assert (ids == [[0, 1], [0, 1]]).all() and np.allclose(gates, 0.5)


def test_forced_underflow_case_really_ties(golden):
    """route3 is x*100: softmax underflows to exact zeros; lowest index wins."""
    g = golden["route3/gates"]
    assert (g[:, 1] == 0.0).any()


def test_oracle_codec_kats(oracle, golden):
    for bits in (2, 3, 4, 8):
        for count in (1, 5, 7, 64, 129, 1000):
            codes = golden[f"pack{bits}_{count}/codes"]
            want = golden[f"pack{bits}_{count}/bytes"]
            np.testing.assert_array_equal(oracle.pack(codes, bits), want)
            st, back = oracle.unpack(want, bits, count)
            assert st == 0
            np.testing.assert_array_equal(back, codes)
    # frozen LSB-first layouts (test_codec.cpp:168-178)
    assert oracle.pack(np.array([1, 2, 3], np.uint32), 2).tolist() == [0x39]
    assert oracle.pack(np.array([5, 3], np.uint32), 3).tolist() == [0x1D]
    assert oracle.pack(np.array([0xA, 0x5], np.uint32), 4).tolist() == [0x5A]
    # dirty padding is corruption (test_codec.cpp:195-199)
    b = oracle.pack(np.array([1, 1, 1], np.uint32), 2)
    b[0] |= 0x80
    assert oracle.unpack(b, 2, 3)[0] != 0


def test_oracle_f16_kats(oracle, golden):
    dec = golden["f16/decode"]
    for h in list(range(0, 1 << 16, 97)) + [0x0001, 0x0400, 0x7BFF, 0x8000, 0x7C00, 0xFC00]:
        a, b = oracle.half_to_float(h), float(dec[h])
        assert (np.isnan(a) and np.isnan(b)) or a == b, hex(h)
    for v, want in zip(golden["f16/encode_in"][::13], golden["f16/encode_out"][::13]):
        assert oracle.float_to_half(float(v)) == int(want)
    # frozen patterns (test_codec.cpp:21-33)
    assert oracle.float_to_half(65504.0) == 0x7BFF
    assert oracle.float_to_half(2.0 ** -24) == 0x0001
    assert oracle.float_to_half(65520.0) == 0x7C00


def test_oracle_permutation_is_stable_counting_sort(oracle):
    rng = np.random.default_rng(3)
    for B, k, K in ((1, 1, 1), (17, 2, 8), (300, 6, 64), (0, 2, 4)):
        ids = np.array([rng.permutation(K)[:k] for _ in range(B)], np.int64).reshape(B, k)
        perm, offs, inv = oracle.permute(ids, K)
        flat = ids.reshape(-1)
        want = np.argsort(flat, kind="stable")
        np.testing.assert_array_equal(perm, want)
        np.testing.assert_array_equal(offs, np.concatenate([[0], np.cumsum(np.bincount(flat, minlength=K))]))
        np.testing.assert_array_equal(inv[perm], np.arange(B * k))


def test_artifact_reader_detects_corruption(tmp_path):
    import shutil
    from oracle.oracle import ArtifactError, read_artifact_np
    d = tmp_path / "a"
    shutil.copytree(os.path.join(GOLD, "folded_b3"), d)
    with open(d / "expert.1.codes.bin", "r+b") as f:
        b = f.read(1)
        f.seek(0)
        f.write(bytes([b[0] ^ 1]))
    with pytest.raises(ArtifactError, match="expert.1.codes"):
        read_artifact_np(str(d))


# ---------------------------------------------------------------------------
# the boundary
# ---------------------------------------------------------------------------

def _declared_symbols():
    with open(os.path.join(REPO, "include", "tileq_b200.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\**\s+\**(tq_\w+)\s*\(", txt, re.M)))


def test_abi_library_exports_every_declared_symbol():
    import paper_2605_09281_b200 as tq
    lib = tq.lib()                                   # loads without a GPU
    names = _declared_symbols()
    assert len(names) >= 20, names
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", tq.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tq_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    assert tq.lib().tq_version().decode()


def test_abi_errors_without_gpu(tmp_path):
    """Host-side validation runs before any device work: a missing artifact is
    an IoError, a corrupted one a FormatError naming the tensor."""
    import shutil
    import paper_2605_09281_b200 as tq
    with pytest.raises(tq.IoError):
        tq.Layer(str(tmp_path / "missing"))
    d = tmp_path / "bad"
    shutil.copytree(os.path.join(GOLD, "general_b8"), d)
    with open(d / "expert.0.scales.bin", "r+b") as f:
        f.write(b"\x00\x00")
    with pytest.raises(tq.FormatError, match="tensor 'expert.0.scales': checksum mismatch"):
        tq.Layer(str(d))
    with pytest.raises(tq.FormatError, match="tensor 'expert.0.scales': non-positive scale"):
        tq.Layer(str(d), verify_crc=False)


def test_no_cpu_fallback_in_product():
    """The product package never imports the checker."""
    pkg = os.path.join(REPO, "paper_2605_09281_b200")
    for root, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cpp", ".cu", ".cuh", ".h")):
                with open(os.path.join(root, fn)) as f:
                    src = f.read()
                assert "from oracle" not in src and "import oracle" not in src, fn


# ---------------------------------------------------------------------------
# synthetic workload + measurement bookkeeping
# ---------------------------------------------------------------------------

def test_factory_stage_replay_matches_quantize_moe(ref, tmp_path):
    """The artifact factory replays quantize_moe's stages without proxy_loss
    (oracle/ref_shim.cpp): its blobs must equal quantize_moe's own, byte for byte."""
    kw = dict(K=6, top_k=2, i=128, o=96, S=1, r=8, bits=3, g=64, calib="gauss", seed=9)
    a, b = str(tmp_path / "replay"), str(tmp_path / "full")
    ref.make_artifact(a, **kw)
    ref.make_artifact(b, full_pipeline=True, **kw)
    bins = sorted(f for f in os.listdir(a) if f.endswith(".bin"))
    assert len(bins) > 20
    for f in bins:
        with open(os.path.join(a, f), "rb") as fa, open(os.path.join(b, f), "rb") as fb:
            assert fa.read() == fb.read(), f


def test_synthetic_artifact_readable_by_reference(ref, oracle, tmp_path):
    from oracle.oracle import read_artifact_np
    from paper_2605_09281_b200 import synth
    d = synth.write_synthetic(str(tmp_path / "s"), K=6, top_k=2, i=256, o=160, S=1, bits=3, r=8, group=128,
                              tier="general", seed=5)
    R = ref.load(d)
    x = np.random.default_rng(0).standard_normal((9, 256)).astype(np.float32)
    yr, idr, gr = R.forward(x)
    y, ids, gates = oracle.tileq_forward(read_artifact_np(d), x)
    np.testing.assert_array_equal(ids, idr)
    assert rel_frob(y, yr) <= 1e-5


def test_synthetic_cache_is_versioned_and_atomic(tmp_path, monkeypatch):
    """bench.py's artifact cache: keyed by the writer's source hash (a stale /tmp
    artifact from an older writer is never reused) and renamed into place."""
    import os
    from paper_2605_09281_b200 import synth
    root = str(tmp_path)
    p = synth.config_path("c1", root)
    assert os.path.basename(p).startswith("c1_folded_s0_") and len(os.path.basename(p)) > len("c1_folded_s0_")
    stale = os.path.join(root, "c1_folded_s0")          # the pre-versioning cache name
    os.makedirs(stale)
    open(os.path.join(stale, "manifest.json"), "w").write("{}")
    calls = []
    real = synth.write_synthetic
    monkeypatch.setattr(synth, "write_synthetic", lambda path, **kw: calls.append(path) or real(path, **kw))
    assert synth.ensure_config("c1", root=root) == p
    assert len(calls) == 1 and calls[0] != p and not os.path.exists(calls[0])   # written aside, renamed
    assert os.path.exists(os.path.join(p, "manifest.json"))
    assert synth.ensure_config("c1", root=root) == p and len(calls) == 1       # cached
    assert sorted(os.listdir(root)) == sorted([os.path.basename(p), "c1_folded_s0"])


def test_bench_algorithmic_bytes_match_survey_table():
    import bench
    info = dict(num_experts=8, top_k=2, in_dim=1024, out_dim=2816, num_shared=0, rank=16, bits=3,
                group_size=128, grid_rows=3, grid_cols=3)
    geo = bench.Geometry(info)
    assert geo.residual_bytes() == 1_081_344 + 45_056 + 8_448
    info2 = dict(info, in_dim=4096, out_dim=14336, rank=32)
    geo2 = bench.Geometry(info2)
    assert geo2.residual_bytes() == 22_020_096 + 917_504 + 172_032        # c2 row
    assert abs(geo2.flops(4096) - 971.7e9) / 971.7e9 < 1e-3               # §8(d) c3 flops
    ids = np.array([[0, 1]])
    placement = np.array([[e // 3, e % 3] for e in range(8)])
    b = geo2.layer_bytes(ids, placement, general=False)
    assert abs(b - 47.6e6) / 47.6e6 < 0.01                                # §8(d) c2 B=1


def test_bench_reference_arm_contract(tmp_path):
    """--impl reference prints the contract line (or 'unavailable') and exits 0."""
    env = dict(os.environ, TILEQ_ARTIFACT_ROOT=str(tmp_path), TILEQ_REF_BUDGET_S="1")
    r = subprocess.run(["python", os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    if "unavailable" not in line:
        for k in ("metric", "value", "unit", "cpu_baseline", "e2e", "config"):
            assert k in line
        assert line["e2e"]["h2d_bytes_per_step"] == 0
        assert line["cpu_baseline"]["kind"] == "reference"


# ---------------------------------------------------------------------------
# the paper's bench layouts: reference fixtures
# ---------------------------------------------------------------------------

def test_layout_fixtures_follow_the_dispatch_contract(golden):
    """tests/golden/layouts.npz (reference outputs): dispatch counts are the
    reference's contract -- fused 2, 1D 1 + B*k, element-wise 2*B*k, dequant 0
    (test_infer.cpp:204-231) -- and element-wise equals the fused 2D result
    (same factors, different association; both f64 in the reference)."""
    lay = dict(np.load(os.path.join(GOLD, "layouts.npz")))
    for name in ART_NAMES:
        k = golden[f"{name}/ids7"].shape[1]
        for B in (7, 33):
            assert int(lay[f"{name}/fused_2d{B}_dispatches"]) == 2
            assert int(lay[f"{name}/shared_1d{B}_dispatches"]) == 1 + B * k
            assert int(lay[f"{name}/element_wise{B}_dispatches"]) == 2 * B * k
            assert int(lay[f"{name}/dequant_only{B}_dispatches"]) == 0
            assert rel_frob(lay[f"{name}/element_wise{B}"], lay[f"{name}/fused_2d{B}"]) <= 1e-5
            assert rel_frob(lay[f"{name}/fused_2d{B}"], golden[f"{name}/lotile{B}"]) <= 1e-6


def test_layout_fixtures_reproduce_with_reference(ref, golden):
    """The committed layout fixtures are what the reference computes today."""
    lay = dict(np.load(os.path.join(GOLD, "layouts.npz")))
    R = ref.load(os.path.join(GOLD, "folded_b3"))
    x, ids, gates = golden["folded_b3/x7"], golden["folded_b3/ids7"], golden["folded_b3/gates7"]
    for layout in ("shared_1d", "element_wise"):
        y, d = R.layout(layout, x, ids, gates)
        np.testing.assert_array_equal(y, lay[f"folded_b3/{layout}7"])
        assert d == int(lay[f"folded_b3/{layout}7_dispatches"])
