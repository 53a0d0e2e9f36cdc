"""Build libtileq_b200.so in-tree (sm_100a) with nvcc.

    python -m paper_2605_09281_b200.build        # or __graft_entry__.build()

The library is the whole product: C++ host runtime + sm_100a kernels behind
the C-ABI in include/tileq_b200.h.  nlohmann/json (the reference artifact's
manifest format, io.hpp:6) is taken from the copy vendored in the venv's
cudnn_frontend headers; zlib provides CRC32 like the reference (io.cpp:71-75).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtileq_b200.so")
SOURCES = ["tq_gemm.cu", "tq_decode.cu", "tq_kernels.cu", "tq_layouts.cu", "tq_producer.cu", "tq_runtime.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def json_include_dir() -> str:
    for d in sys.path:
        if not d:
            continue
        cand = os.path.join(d, "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.exists(os.path.join(cand, "json.hpp")):
            return cand
    raise RuntimeError("nlohmann/json.hpp not found (expected under site-packages/include/cudnn_frontend)")


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "tileq_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB) -> str:
    """Compile the sources (in parallel) and link ``lib``.  ``defines`` builds an
    experiment variant (e.g. TQ_SPIN_WAIT) into a separate library file."""
    if not force and not defines and not needs_rebuild():
        return LIB
    objs = []
    jdir = json_include_dir()
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              f"-I{jdir}", f"-I{os.path.join(HERE, '..', 'include')}", "--expt-relaxed-constexpr",
              *[f"-D{d}" for d in defines]]
    build_dir = os.path.join(HERE, "_build" + "".join("_" + d.lower() for d in defines))
    os.makedirs(build_dir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(build_dir, src + ".o")
        cmd = common + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for src, pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}\n{err}")
        if verbose:
            print(err)
    tmp = lib + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lz", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = LIB if not defs else os.path.join(HERE, "libtileq_b200_" + "_".join(d.lower() for d in defs) + ".so")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, lib=out))
