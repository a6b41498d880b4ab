"""SASS instruction-class counts per kernel of the built libomniseg.so (static evidence that the
hot kernels use tcgen05 MMAs / TMA / TMEM): cuobjdump -sass, demangled with c++filt.

    python scripts/sass_summary.py [--lib PATH] > profiles/r02_sass_summary.md

Counted mnemonics (B200_PROFILING.md): UTCHMMA (tcgen05.mma kind::f16), UTCQMMA (kind::f8f6f4),
UTCBAR (tcgen05.commit), UTMALDG / UTMASTG (TMA tensor load / store), UBLKCP (bulk copy), LDTM /
STTM (tcgen05.ld / st, TMEM <-> registers), SYNCS (mbarrier ops), FFMA2 / FFMA (packed / scalar
fp32 FMA), ATOMG / RED (global atomics: the stitch)."""
import argparse
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLASSES = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "SYNCS", "FFMA2", "FFMA",
           "REDG", "ATOMG"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2305_14566_b200", "lib", "libomniseg.so"))
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if not m:
            continue
        op, suf = m.group(2), m.group(3) or ""
        funcs[cur]["_total"] += 1
        key = op
        if op in ("UTMALDG", "UTMASTG"):
            key = op
            funcs[cur][op + suf.split(".")[1] if suf.count(".") >= 1 and suf.split(".")[1][0].isdigit() else op] += 0
        for c in CLASSES:
            if key == c:
                funcs[cur][c] += 1
    names = list(funcs)
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    print("# SASS instruction classes per kernel (`python scripts/sass_summary.py`)\n")
    print("Static counts in the built `libomniseg.so` (sm_100a). Kernels without any of the classes are omitted.\n")
    print("| kernel | instrs | " + " | ".join(CLASSES) + " |")
    print("|---|---|" + "---|" * len(CLASSES))
    tot = collections.Counter()
    for n, d in zip(names, dem):
        c = funcs[n]
        if not any(c[k] for k in CLASSES):
            continue
        d = re.sub(r"osg::|\(anonymous namespace\)::", "", d)
        d = re.sub(r"\(.*\)$", "", d)
        print(f"| `{d}` | {c['_total']} | " + " | ".join(str(c[k]) for k in CLASSES) + " |")
        tot.update({k: c[k] for k in CLASSES})
    print("| **all kernels** | | " + " | ".join(str(tot[k]) for k in CLASSES) + " |")


if __name__ == "__main__":
    sys.exit(main())
