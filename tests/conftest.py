import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, ORACLE_SO
    if not os.path.exists(ORACLE_SO):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), "oracle"], check=True,
                       capture_output=True)
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libtileq_ref.so not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def artifact_root(tmp_path_factory):
    return str(tmp_path_factory.mktemp("artifacts"))


class ArtifactFactory:
    """Reference-pipeline artifacts (oracle/_ref factory), cached per spec."""

    def __init__(self, ref, root):
        self.ref, self.root, self.cache = ref, root, {}

    def __call__(self, **spec):
        key = tuple(sorted(spec.items()))
        if key not in self.cache:
            name = "art_" + "_".join(f"{k}{v}" for k, v in key)
            path = os.path.join(self.root, name)
            self.ref.make_artifact(path, **spec)
            self.cache[key] = path
        return self.cache[key]


@pytest.fixture(scope="session")
def make_artifact(ref, artifact_root):
    return ArtifactFactory(ref, artifact_root)


def rel_frob(got, want) -> float:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    d = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (d if d > 0 else 1.0))
