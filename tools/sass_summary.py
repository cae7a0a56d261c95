"""SASS instruction counts of the product kernels (cuobjdump -sass of the built libheadinfer.so): the evidence that
the hot loops run on tcgen05 (UTCHMMA, LDTM/STTM), TMA (UTMALDG) and mbarriers (SYNCS), CPU-only.

    python tools/sass_summary.py [out.txt]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2502_12574_b200", "libheadinfer.so")
OPS = ["UTCHMMA", "UTCBAR", "UTMALDG", "LDTM", "STTM", "UTCATOMSWS", "MUFU.EX2", "FFMA2", "FADD2",
       "F2FP.BF16.F32.PACK_AB", "HMMA", "LDSM", "SYNCS", "FMNMX3"]


def main(out=None):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts, forms, fn = collections.OrderedDict(), collections.OrderedDict(), None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            forms[fn] = collections.Counter()
            continue
        if fn is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            if op.startswith(("UTCHMMA", "UTMALDG", "UTCBAR")):
                forms[fn][op] += 1
            for k in OPS:
                if op == k or op.startswith(k + "."):
                    counts[fn][k] += 1
    lines = ["# SASS instruction counts of libheadinfer.so (cuobjdump -sass; tools/sass_summary.py), product build",
             "# UTCHMMA = tcgen05.mma, UTMALDG = TMA tensor load, LDTM/STTM = tcgen05.ld/st (TMEM), HMMA = mma.sync,",
             "# SYNCS = mbarrier ops, MUFU.EX2 = ex2.approx, FFMA2/FADD2 = packed f32x2", ""]
    for f, c in counts.items():
        short = re.sub(r"^_ZN2hi\d+_GLOBAL__N__[0-9a-f]+_\d+", "", f)
        lines.append(short)
        lines.append("   " + "  ".join(f"{k}={c[k]}" for k in OPS if c[k]))
        if forms[f]:
            lines.append("   forms: " + "  ".join(f"{k}={v}" for k, v in forms[f].items()))
    txt = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(txt)
    sys.stdout.write(txt)


if __name__ == "__main__":
    main(*sys.argv[1:])
