"""csrc/tq_exp.h (the routers' f64 exp) against the host libm, bit for bit.

route() takes prob_k = std::exp(s_k - mx) (moe.cpp:72) with glibc's exp; the
engine restates that algorithm (tq_exp.h) so routing ties break identically.
This builds the header for the host with FMA contraction off and compares it
with libm's exp on ~70M arguments (softmax-shaped, f32 score differences, the
whole over/underflow range, raw bit patterns, edges).  glibc picks its FMA
variant on FMA-capable CPUs -- the B200 hosts' -- so the check needs one too.
"""
import os
import subprocess
import tempfile

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_2605_09281_b200", "csrc")


def _cpu_has_fma():
    try:
        with open("/proc/cpuinfo") as f:
            return " fma " in f.read().replace("\n", " ")
    except OSError:
        return False


@pytest.mark.skipif(not _cpu_has_fma(), reason="host glibc uses its non-FMA exp variant")
def test_exp_port_matches_libm():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "exp_port_check")
        subprocess.run(["g++", "-O2", "-mfma", "-ffp-contract=off", "-std=c++17", "-I", CSRC,
                        os.path.join(HERE, "exp_port_check.cpp"), "-o", exe, "-lm"], check=True)
        r = subprocess.run([exe, "15000000"], capture_output=True, text=True, timeout=300)
        print(r.stdout)
        assert r.returncode == 0, r.stdout


def test_exp_table_regenerates():
    """csrc/tq_exp.h's 2^(i/128) table is exactly what tools/gen_exp_table.py derives
    from first principles (60-digit decimals)."""
    import re
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tools"))
    import gen_exp_table
    src = open(os.path.join(CSRC, "tq_exp.h")).read()
    body = src[src.index("kTab[256] = {"):src.index("};", src.index("kTab[256] = {"))]
    words = [int(w, 16) for w in re.findall(r"0x([0-9a-f]{16})ull", body)]
    want = [v for pair in gen_exp_table.table() for v in pair]
    assert words == want
