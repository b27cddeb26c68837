"""The C-ABI library: loads without a GPU, exports every symbol the header
declares, and runs its host-side validation (config.cpp:42-79,
config.cpp:25-35, engine.cpp:319-323) before touching the device."""
import json
import os
import re

import numpy as np
import pytest

from tests.conftest import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "mgfwa_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mgfwa_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2501_03944_b200 import _capi

    L = _capi.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_capi.SIGNATURES), "ctypes binding out of sync with the header"
    assert b"sm_100a" in L.mgfwa_version()


def test_library_is_not_linked_against_torch_or_python():
    import subprocess

    from paper_2501_03944_b200 import _capi

    out = subprocess.run(["ldd", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in out and "python" not in out


def test_validation_messages_match_reference():
    import paper_2501_03944_b200 as P

    with open(os.path.join(GOLDEN, "validation.json")) as f:
        v = json.load(f)
    space = P.SearchSpace.box(4, -1.0, 1.0)
    for kw, msg in zip(v["cases"], v["messages"]):
        if not msg:
            continue
        base = dict(max_evaluations=1000)
        base.update(kw)
        with pytest.raises(ValueError) as e:
            P.Engine(P.MgfwaConfig(**base), space, P.Sphere(), 0)
        assert str(e.value) == msg


def test_space_and_budget_validation():
    import paper_2501_03944_b200 as P

    cfg = P.MgfwaConfig(max_evaluations=1000)
    with pytest.raises(ValueError, match="lower\\[d\\] < upper\\[d\\]"):
        P.Engine(cfg, P.SearchSpace([0.0, 1.0], [1.0, 1.0]), P.Sphere(), 0)
    with pytest.raises(ValueError, match="non-empty"):
        P.Engine(cfg, P.SearchSpace([], []), P.Sphere(), 0)
    with pytest.raises(ValueError, match="budget too small"):
        P.Engine(P.MgfwaConfig(max_evaluations=39), P.SearchSpace.box(3, -1, 1), P.Sphere(), 0)
    with pytest.raises(ValueError, match="input dimension mismatch"):
        P.Engine(cfg, P.SearchSpace.box(10, -1, 1), P.MlpWeights(), 0)


def test_python_mirror_matches_reference_interface():
    import paper_2501_03944_b200 as P

    c = P.MgfwaConfig()
    assert (c.batches, c.fireworks, c.sparks_per_firework, c.guides_per_firework) == (8, 5, 30, 3)
    assert c.top_spark_count() == 6 and c.evaluations_per_wave() == 8 * 5 * 33
    assert c.resolved_initial_amplitude(20.0) == 10.0
    s = P.SearchSpace.box(3, -2.0, 5.0)
    assert s.dim() == 3 and s.max_range() == 7.0 and s.contains(0, 5.0) and not s.contains(0, 5.0001)
    assert P.MlpWeights().dim() == 25450
