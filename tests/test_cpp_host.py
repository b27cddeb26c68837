"""The header-only C++ face (include/mgfwa_b200.hpp) compiles against the
C-ABI library and behaves like the reference's run(): validation errors as
std::invalid_argument with the reference messages (CPU), a full run (GPU)."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

PKG = os.path.join(ROOT, "paper_2501_03944_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "run_b200")
    cmd = ["/usr/bin/g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "run_b200.cpp"), "-L", PKG, "-lmgfwa_b200", f"-Wl,-rpath,{PKG}", "-o", out]
    subprocess.run(cmd, check=True)
    return out


def test_cpp_validation(exe):
    r = subprocess.run([exe, "validate"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "MgfwaConfig: amp_amplify must be > 1" in r.stdout
    assert "budget too small" in r.stdout


@pytest.mark.gpu
def test_cpp_run(exe):
    r = subprocess.run([exe, "run"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "evaluations 1000" in r.stdout
