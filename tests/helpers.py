"""Shared input builders for the tests; the parity rule itself lives in oracle/parity.py."""
from __future__ import annotations

import math

import numpy as np

from oracle.pyoracle import BlockSet

from oracle.parity import OUT_TOL, SCORE_TIE, TAU, check_parity, max_abs  # noqa: F401

FIG4_MASSES = [400, 330, 250, 55, 40, 30, 20, 14.08, 12, 10, 9, 5.848, 5, 4, 3, 2]


def fig4_blockset():
    """Reference test_engine.cpp:27-45: 16 single-token d=2 blocks whose mass at
    scale 1 and q=(2,0) is the chosen mass (up to float key rounding)."""
    keys, vals, realized = [], [], []
    for i, m in enumerate(FIG4_MASSES):
        k0 = np.float32(math.log(m) / 2.0)
        keys.append(np.array([[k0, 0.0]], np.float32))
        vals.append(np.array([[i + 1, 2 * i + 1]], np.float32))
        realized.append(math.exp(2.0 * float(k0)))
    return BlockSet(keys, vals), np.array([2.0, 0.0], np.float32), realized


def random_blockset(rng, n, d, tok_lo=1, tok_hi=16, planted_frac=0.0, skew=3.0, ids=None, full=None):
    """N(0,1) keys/values (reference testutil::make_block) with optional planted bias."""
    bias = rng.standard_normal(d).astype(np.float32) * skew
    keys, vals = [], []
    for i in range(n):
        t = full if full else int(rng.integers(tok_lo, tok_hi + 1))
        k = rng.standard_normal((t, d)).astype(np.float32)
        if planted_frac and rng.random() < planted_frac:
            k = k + bias
        keys.append(k)
        vals.append(rng.standard_normal((t, d)).astype(np.float32))
    return BlockSet(keys, vals, ids)


