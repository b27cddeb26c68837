import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


def _gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    O.build(with_reference=False)
    return O.Oracle()


@pytest.fixture(scope="session")
def golden():
    def load(name):
        d = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
        return {k: d[k] for k in d.files}

    return load


def golden_cases(g: dict):
    """operators.npz: {case: {field: array}}"""
    out = {}
    for k, v in g.items():
        c, f = k.split("__", 1)
        out.setdefault(c, {})[f] = v
    return out
