"""Per-kernel SASS evidence from the built library (runs on the CPU box):
tcgen05 MMA (UTCHMMA / UTCQMMA), TMA loads (UTMALDG), bulk copies (UBLKCP), TMEM loads
(LDTM), legacy tensor-core MMA (HMMA) and the register count ptxas assigned.

    python tools/sass_evidence.py > profiles/r1_sass_evidence.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2510_19470_b200", "libhep.so")
OPS = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMAPF", "UBLKCP", "LDTM", "UTCBAR", "HMMA"]


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        for op in OPS:
            if re.search(r"\b" + op + r"[\s.]", line):
                counts[cur][op] += 1
    print("| kernel | " + " | ".join(OPS) + " |")
    print("|---|" + "---|" * len(OPS))
    for fn, c in counts.items():
        if not any(c.values()):
            continue
        name = demangle(fn)
        name = name.replace("hep::(anonymous namespace)::", "").replace("void ", "", 1)
        name = re.sub(r"\(.*", "", name)
        print(f"| `{name}` | " + " | ".join(str(c[o]) if c[o] else "" for o in OPS) + " |")
    print(f"\n{len(counts)} kernels in {os.path.relpath(LIB, ROOT)}; rows list those using any of the ops above.")


if __name__ == "__main__":
    sys.exit(main())
