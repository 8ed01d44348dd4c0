"""Replay the assembly's work-unit / piece plan (assemble.cu) on a golden pair list, host only:
K5a / K5b flops and the bytes of piece shards per rank, for the orientation rules and row
chunks discussed in DESIGN.md section 6 ("Column-cell reuse").  Balanced trees only (n / leaf a
power of two, as in BASELINE cfg3-5).

    python tools/plan_replay.py cfg5 [--chunk 16384] [--rule small|cheap] [--ranks 8]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PARAMS = {"cfg3": (131072, 256, 21, 20), "cfg4": (262144, 512, 51, 50), "cfg5": (1 << 20, 2048, 1326, 50)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(PARAMS))
    ap.add_argument("--chunk", type=int, default=None)
    ap.add_argument("--rule", choices=["small", "cheap"], default="small")
    ap.add_argument("--ranks", type=int, default=8)
    a = ap.parse_args()
    n, leaf, M, d = PARAMS[a.config]
    t = int(np.log2(n // leaf))
    P = np.load(os.path.join(ROOT, "tests", "golden", "pairs_%s.npz" % a.config))["pairs"]
    ch = a.chunk or (16384 if n >= (1 << 20) else 4096)
    dp = (d + 2 + 3) // 4 * 4

    def depth(q):
        return int(np.floor(np.log2(q + 1)))

    def size(q):
        return n >> depth(q)

    def begin(q):
        return (q - (2 ** depth(q) - 1)) * size(q)

    def p(q):
        return leaf - M if depth(q) == t else M

    def is_anc(anc, q):
        while q > anc:
            q = (q - 1) // 2
        return q == anc

    rows, pairs = {}, []
    for r, c in P:
        r, c = int(r), int(c)
        if r == c or is_anc(c, r):
            x, b = r, c
        elif is_anc(r, c):
            x, b = c, r
        else:
            sr, sc, qr, qc = size(r), size(c), p(r), p(c)
            sw = (2 * sc * sr * qr + 2 * qc * sc * qr) < (2 * sr * sc * qc + 2 * qr * sr * qc)
            if a.rule == "small" and sr != sc:
                sw = sc < sr
            x, b = (c, r) if sw else (r, c)
        pairs.append((x, b))
        rows.setdefault(b, []).append((begin(x), begin(x) + size(x)))
    units, k5a = {}, 0.0
    for b, rg in rows.items():
        rg = sorted(rg + [(begin(b), begin(b) + size(b))])
        merged = []
        for lo, hi in rg:
            if merged and lo <= merged[-1][1]:
                merged[-1] = (merged[-1][0], max(merged[-1][1], hi))
            else:
                merged.append((lo, hi))
        for lo0, hi0 in merged:
            c0 = lo0 // ch
            while c0 * ch < hi0:
                lo, hi = max(lo0, c0 * ch), min(hi0, (c0 + 1) * ch)
                units[(b, c0)] = units.get((b, c0), 0.0) + (hi - lo) * size(b) * (2.0 * dp + 16.0 * 24 + 60.0)
                k5a += (hi - lo) * size(b) * (2.0 * d + 2.0 * p(b))
                c0 += 1
    pieces, k5b = [], 0.0
    for x, b in pairs:
        c0 = begin(x) // ch
        while c0 * ch < begin(x) + size(x):
            lo, hi = max(begin(x), c0 * ch), min(begin(x) + size(x), (c0 + 1) * ch)
            f = 2.0 * p(x) * (hi - lo) * p(b)
            units[(b, c0)] += f
            k5b += f
            pieces.append(((b, c0), p(x) * p(b)))
            c0 += 1
    from paper_1701_00285_b200 import mlk
    keys = list(units)
    own = mlk.partition_lpt(np.array([units[k] for k in keys]), a.ranks)
    owner = {k: own[i] for i, k in enumerate(keys)}
    shard = np.zeros(a.ranks)
    for uk, ln in pieces:
        shard[owner[uk]] += ln
    values = sum(p(x) * p(b) for x, b in pairs)
    print("%s rule=%s chunk=%d: K5a %.3e K5b %.3e flops; pieces %d, %.1f GB (final values %.1f GB); "
          "shard per rank (of %d) max %.1f GB" % (a.config, a.rule, ch, k5a, k5b, len(pieces),
                                                  8e-9 * sum(ln for _, ln in pieces), 8e-9 * values, a.ranks,
                                                  8e-9 * shard.max()))


if __name__ == "__main__":
    main()
