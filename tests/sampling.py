"""Fixed, seeded block samples for the full-size parity tests (SURVEY.md section 8(c) "large
configs") -- shared by tests/test_gpu_parity.py and tools/make_golden_blocks.py so the
goldens and the tests check the same blocks.  Test infrastructure: index selection only, no
arithmetic of the method.

  cfg2: the root-root block, every admitted block with both cells at level <= 2 (the blocks
        summed from several 4096-row pieces), all leaf self blocks, 24 random admitted pairs.
  cfg3, cfg4: all leaf self blocks, 64 random admitted pairs with |a| |b| <= 2^28, the (0,0)
        block, every admitted block with both cells at level <= 1, and 8 random ancestor blocks
        whose row cell spans several 4096-row pieces (row cell at depth 3-4 for cfg3, 5 for cfg4;
        column cell an ancestor at depth >= 1).
Random draws use numpy.random.default_rng([0, 3]).
"""
import numpy as np

# blocks whose oracle evaluation costs more than this many covariance entries are read from
# tests/golden/blocks_<cfg>.npz (written by tools/make_golden_blocks.py, oracle only)
GOLDEN_MIN_ENTRIES = 1 << 26


def size(tree, q):
    return int(tree.end[q] - tree.begin[q])


def select_blocks(name, pairs, tree):
    """Sorted indices into `pairs` (the admitted (row, col) list in BSR order)."""
    rng = np.random.default_rng([0, 3])
    depth = tree.depth
    idx = set()
    leaf_self = [k for k, (a, b) in enumerate(pairs) if a == b and tree.is_leaf[a]]
    idx |= set(leaf_self)
    idx |= {k for k, (a, b) in enumerate(pairs) if a == 0 and b == 0}
    if name == "cfg2":
        idx |= {k for k, (a, b) in enumerate(pairs) if depth[a] <= 2 and depth[b] <= 2}
        rest = [k for k in range(len(pairs)) if k not in idx]
        idx |= set(rng.choice(rest, 24, replace=False).tolist())
    else:
        cand = [k for k, (a, b) in enumerate(pairs)
                if not (a == b and tree.is_leaf[a]) and size(tree, a) * size(tree, b) <= (1 << 28)
                and not (a == 0 and b == 0)]
        idx |= set(rng.choice(cand, 64, replace=False).tolist())
        idx |= {k for k, (a, b) in enumerate(pairs) if depth[a] <= 1 and depth[b] <= 1}
        rdep = (3, 4) if name == "cfg3" else (5,)

        def is_anc(b, a):
            while a > 0:
                a = (a - 1) // 2
                if a == b:
                    return True
            return False
        multi = [k for k, (a, b) in enumerate(pairs)
                 if depth[a] in rdep and depth[b] >= 1 and is_anc(b, a) and k not in idx]
        idx |= set(rng.choice(multi, 8, replace=False).tolist())
    return sorted(int(k) for k in idx)


def golden_needed(pairs, tree, idx):
    return [k for k in idx if size(tree, pairs[k][0]) * size(tree, pairs[k][1]) > GOLDEN_MIN_ENTRIES]


def matvec_rows(n, count=512):
    """Seeded sample of point-space rows for the sampled C a checks."""
    return np.sort(np.random.default_rng([0, 3]).choice(n, count, replace=False))
