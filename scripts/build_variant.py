"""Build an experimental variant of the library (extra -D flags on
k_engine.cu / k_mlp_tc.cu) into _variants/lib_<name>.so for A/B timing on
the GPU box (see scripts/kernel_times.py).  Not part of the product build.

    python scripts/build_variant.py NAME [-DKEY=VAL ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_03944_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "_variants")
os.makedirs(out_dir, exist_ok=True)
B.build()
objs = []
for src in B.SOURCES:
    o = os.path.join(B.BUILD, src.replace(".cu", ".o"))
    if src != "engine.cu" and defs:
        o = os.path.join(out_dir, f"{name}_{src[:-3]}.o")
        cmd = [B.nvcc()] + B.ARCH + B.FLAGS + defs + ["-c", os.path.join(B.CSRC, src), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr[-3000:])
        for line in r.stderr.splitlines():
            if "registers" in line or "spill" in line:
                pass
    objs.append(o)
lib = os.path.join(out_dir, f"lib_{name}.so")
subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs, check=True)
print(lib)
