"""Host-side checks of libmlk.so that need no GPU: every symbol of include/mlk.h is exported,
and the host logic of the multi-GPU path (LPT partition, shard plan, gather protocol)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_1701_00285_b200 import mlk
    return mlk


def test_header_symbols_exported():
    mlk = _lib()
    hdr = open(os.path.join(ROOT, "include", "mlk.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(mlk_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 30
    for nm in names:
        assert hasattr(mlk._lib, nm), nm
    assert set(mlk.SYMBOLS) == names


def test_lpt_partition_properties():
    mlk = _lib()
    rng = np.random.default_rng(0)
    cost = rng.pareto(1.5, 5000) + 0.01
    for R in (1, 2, 3, 8):
        own = mlk.partition_lpt(cost, R)
        assert own.min() >= 0 and own.max() < R
        loads = np.bincount(own, weights=cost, minlength=R)
        # LPT bound: max load <= mean + max cost
        assert loads.max() <= cost.sum() / R + cost.max() + 1e-9
        # deterministic
        assert np.array_equal(own, mlk.partition_lpt(cost, R))
    with pytest.raises(mlk.MlkError):
        mlk.partition_lpt(np.array([1.0, -1.0]), 2)


def test_shard_plan_is_a_disjoint_cover():
    mlk = _lib()
    rng = np.random.default_rng(1)
    sizes = rng.integers(1, 50, 300)
    val_off = np.concatenate([[0], np.cumsum(sizes)])
    owner = mlk.partition_lpt(sizes.astype(float), 4)
    so, sl = mlk.shard_plan(val_off, owner, 4)
    assert sl.sum() == val_off[-1]
    for r in range(4):
        ks = np.nonzero(owner == r)[0]
        spans = sorted((so[k], so[k] + sizes[k]) for k in ks)
        pos = 0
        for a, b in spans:
            assert a == pos
            pos = b
        assert pos == sl[r]
