"""Build the CUDA library with extra nvcc flags into _variants/<name>/ (git-
ignored) for A/B experiments; select it at run time with MGFWA_LIB.

    python scripts/build_variant.py probe_nofc -DLENET_PROBE=1
    MGFWA_LIB=_variants/probe_nofc/libmgfwa_b200.so python bench.py ...
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_03944_b200 import build as B  # noqa: E402


def main():
    name, extra = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "_variants", name)
    os.makedirs(out, exist_ok=True)
    objs = []

    def one(src):
        o = os.path.join(out, src.replace(".cu", ".o"))
        cmd = [B.nvcc()] + B.ARCH + B.FLAGS + extra + ["-c", os.path.join(B.CSRC, src), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr[-3000:])
        return o

    with cf.ThreadPoolExecutor(len(B.SOURCES)) as ex:
        objs = list(ex.map(one, B.SOURCES))
    lib = os.path.join(out, "libmgfwa_b200.so")
    subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs, check=True)
    print(lib)


if __name__ == "__main__":
    main()
