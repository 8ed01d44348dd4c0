"""SASS instruction counts of the hot kernels (cuobjdump -sass of the in-tree objects, sm_100a):
FP64 tensor (DMMA.8x8x4), TMA (UTMALDG), mbarrier (SYNCS), DFMA/DMUL/DADD, shared loads, cp.async
(LDGSTS), and predicated DMMAs (a DMMA predicated off still takes its pipe slot, DESIGN.md
section 6) -- the evidence that the kernels run on DMMA + TMA and that tcgen05 has no FP64 kind.

    python tools/sass_summary.py > profiles/sass_r02.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_1701_00285_b200", "build")
KEYS = [("DMMA", r"\bDMMA\.8x8x4\b"), ("pDMMA", r"@!?P\d+\s+DMMA"), ("UTMALDG", r"\bUTMALDG"),
        ("SYNCS", r"\bSYNCS\."), ("DFMA", r"\bDFMA\b"), ("DMUL", r"\bDMUL\b"), ("DADD", r"\bDADD\b"),
        ("LDS", r"\bLDS(\.|\s)"), ("LDGSTS", r"\bLDGSTS\b"), ("tcgen05", r"UTCMMA|UTCHMMA|UTCQMMA|tcgen05")]
KERNELS = {"tile.o": "k_tile_contract", "covsym.o": "k_cov_sym", "nested.o": "k_transfer", "gemm.o": "k_gemm"}


def demangle_args(name):
    m = re.search(r"(k_\w+?)ILi(.*?)EEEv", name)
    if not m:
        return name
    args = re.findall(r"Li(-?\d+)E|Lb([01])E", "Li" + m.group(2) + "E")
    return "%s<%s>" % (m.group(1), ",".join(a or b for a, b in args))


def main():
    tot = collections.Counter()
    print("# cuobjdump -sass of paper_1701_00285_b200/build/*.o (sm_100a); counts per kernel instantiation")
    print("%-34s" % "kernel" + "".join("%9s" % k for k, _ in KEYS))
    for obj, kname in KERNELS.items():
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True,
                              text=True).stdout
        cur, counts = None, collections.OrderedDict()
        for line in sass.splitlines():
            if "Function :" in line:
                cur = line.split("Function :")[1].strip()
                counts[cur] = collections.Counter() if kname in cur else None
                continue
            if cur is None or counts.get(cur) is None:
                continue
            for k, rx in KEYS:
                if re.search(rx, line):
                    counts[cur][k] += 1
        for fn, c in counts.items():
            if c is None:
                continue
            tot.update(c)
            print("%-34s" % demangle_args(fn)[:34] + "".join("%9d" % c[k] for k, _ in KEYS))
    print("%-34s" % "TOTAL" + "".join("%9d" % tot[k] for k, _ in KEYS))


if __name__ == "__main__":
    sys.exit(main())
