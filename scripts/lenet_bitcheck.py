"""Bit-level fingerprint of LeNet fitness values (A/B check of kernel
variants that must not change results):  python scripts/lenet_bitcheck.py"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_03944_b200 as P  # noqa: E402

rng = np.random.default_rng(7)
for S, n, scale in ((1024, 40, 0.3), (200, 17, 1.0), (77, 3, 0.05)):
    W = rng.uniform(-scale, scale, size=(n, P.LeNet(samples=S).dim())).astype(np.float32)
    fit, nan = P.batched_apply(P.LeNet(samples=S), W)
    print(S, n, nan, hashlib.sha1(np.asarray(fit, dtype=np.float64).tobytes()).hexdigest()[:16], float(np.mean(fit)))
