"""The explode kernel's split splitmix64 (csrc/common.cuh draw_key /
mix_draw / mant_lo: + gamma folded into one IMAD.WIDE, final xorshift folded
into the mantissa extraction) is bit-identical to rng.hpp:33-38 — checked on
the host over 1 M random (prefix, coordinate) pairs.  The device form runs in
every GPU parity test (explode / mapping exact against the reference)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


@pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc not available")
def test_split_draw_matches_splitmix64(tmp_path):
    exe = tmp_path / "draw_split_check"
    src = os.path.join(ROOT, "tests", "host", "draw_split_check.cu")
    inc = os.path.join(ROOT, "paper_2501_03944_b200", "csrc")
    r = subprocess.run([NVCC, "-std=c++17", "-O2", "-I", inc, src, "-o", str(exe)], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    out = subprocess.run([str(exe), "1000000"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.startswith("0 mismatches"), out.stdout
