"""Time mgfwa_run_once() cold (after mgfwa_release_cached_workspace) and warm,
three times each, for the C2 workload (setup-cost probe)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_03944_b200 as P  # noqa: E402
from paper_2501_03944_b200 import _capi as A  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
steps = 50
cfg = bench.make_config(P, w, w["B"] * w["mu"] + steps * w["B"] * w["mu"] * (w["lam"] + w["M"]))
c, keep = cfg._c()
space = P.SearchSpace.box(w["D"], w["lo"], w["hi"])
obj = bench.make_objective(P, w)
sp, ob = space._c(), obj._c()
B, D = w["B"], w["D"]
bf, bp = np.empty(B), np.empty((B, D))
cap = steps + 2
te, tb, tw = np.zeros((B, cap), np.uint64), np.zeros((B, cap)), np.zeros((B, cap))
cnt = A.mgfwa_counters_t()
pdp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731


def once():
    t = time.perf_counter()
    rc = A.lib().mgfwa_run_once(C.byref(c), C.byref(sp), C.byref(ob), 7, 0, pdp(bf), pdp(bp),
                                te.ctypes.data_as(C.POINTER(C.c_uint64)), pdp(tb), pdp(tw), cap, C.byref(cnt))
    assert rc == 0
    return time.perf_counter() - t


for i in range(3):
    A.lib().mgfwa_release_cached_workspace()
    cold = once()
    warm = once()
    print(f"cold {cold * 1e3:.1f} ms  warm {warm * 1e3:.1f} ms")
