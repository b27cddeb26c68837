"""Build the CUDA library of a source tree other than the working copy (e.g.
a `git archive` of another revision) into _variants/<name>/ for A/B runs.

    git archive HEAD paper_2501_03944_b200/csrc include | tar -x -C /tmp/rev
    python scripts/build_rev.py /tmp/rev <name> [extra nvcc flags]
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_03944_b200 import build as B  # noqa: E402


def main():
    tree, name, extra = sys.argv[1], sys.argv[2], sys.argv[3:]
    csrc = os.path.join(tree, "paper_2501_03944_b200", "csrc")
    out = os.path.join(ROOT, "_variants", name)
    os.makedirs(out, exist_ok=True)

    def one(src):
        o = os.path.join(out, src.replace(".cu", ".o"))
        cmd = [B.nvcc()] + B.ARCH + B.FLAGS + extra + ["-c", os.path.join(csrc, src), "-o", o]
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
