"""SASS instruction census of the library's kernels (cuobjdump -sass of the
built objects): tensor-core, TMA, TMEM and FP64 instruction counts per
kernel, the evidence for which unit each kernel runs on.

    python scripts/sass_census.py [out.md]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2501_03944_b200", "_build")
CLASSES = {
    "UTCHMMA / UTCQMMA (tcgen05.mma)": r"^UTC[HQ]MMA",
    "UTMALDG (TMA tile load)": r"^UTMALDG",
    "UBLKCP (bulk copy)": r"^UBLKCP",
    "UTCBAR (tcgen05.commit)": r"^UTCBAR",
    "LDTM (tcgen05.ld)": r"^LDTM",
    "STTM (tcgen05.st)": r"^STTM",
    "HMMA (mma.sync)": r"^HMMA",
    "DFMA/DADD/DMUL (fp64)": r"^D(FMA|ADD|MUL)",
    "IMAD (all)": r"^IMAD",
    "LOP3/SHF (int ALU)": r"^(LOP3|SHF)",
}


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


def census():
    out = {}
    for obj in sorted(os.listdir(BUILD)):
        if not obj.endswith(".o"):
            continue
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(BUILD, obj)], capture_output=True,
                              text=True).stdout
        cur = None
        for line in sass.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                cur = demangle(m.group(1))
                out[cur] = collections.Counter()
                continue
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if cur and m:
                op = m.group(1)
                out[cur]["total"] += 1
                for cls, rx in CLASSES.items():
                    if re.match(rx, op):
                        out[cur][cls] += 1
    return out


def main():
    res = census()
    lines = ["# SASS instruction census (cuobjdump -sass of paper_2501_03944_b200/_build/*.o, sm_100a)", "",
             "Static instruction counts per kernel (not executed counts).", "",
             "| kernel | total | " + " | ".join(CLASSES) + " |", "|---|---|" + "---|" * len(CLASSES)]
    for k in sorted(res):
        c = res[k]
        if not any(c[cls] for cls in list(CLASSES)[:6]) and not k.startswith(("void mgfwa_b200::k_explode",)):
            if "k_explode_map" not in k and "k_net" not in k:
                continue
        short = re.sub(r"\(.*", "", k.replace("(anonymous namespace)::", "").replace("mgfwa_b200::", ""))
        short = short.replace("void ", "")
        lines.append(f"| `{short}` | {c['total']} | " + " | ".join(str(c[cls]) for cls in CLASSES) + " |")
    txt = "\n".join(lines) + "\n"
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
