"""Shared input builders and the parity rule used by the tests.

Parity rule (BASELINE.json north_star, SURVEY.md §7 hard part 2):
  * ranked/processed block sets identical, except where estimated scores tie
    within SCORE_TIE (1e-6) or the stop decision sits within TAU (1e-5) of eps;
  * outputs within OUT_TOL (1e-3) max-abs (fp32 accumulate); when the block
    set legitimately differs, the output is checked against the fp64 exact
    attention over the GPU's own block set.
"""
from __future__ import annotations

import math

import numpy as np

from oracle.pyoracle import BlockSet

SCORE_TIE = 1e-6
TAU = 1e-5
OUT_TOL = 1e-3

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


def max_abs(a, b) -> float:
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)))) if np.size(a) else 0.0


def check_parity(oracle, q, bs: BlockSet, cfg, topk, gpu_ids, gpu_bp, gpu_out, gpu_est, orc=None, ranked_gpu=None):
    """Asserts the GPU result equals the oracle's under the parity rule. Returns a tag:
    'exact' (same block set) or 'tie' (difference explained by a score tie or a
    stop decision within TAU of eps)."""
    orc = orc or oracle.psa(q, bs, cfg, topk)
    assert orc.status == 0
    if gpu_bp == orc.blocks_processed and np.array_equal(np.asarray(gpu_ids), orc.processed_ids):
        assert max_abs(gpu_out, orc.output) <= OUT_TOL, (max_abs(gpu_out, orc.output), gpu_bp)
        if gpu_est is not None:
            assert abs(gpu_est - orc.estimated_coverage) <= 1e-4, (gpu_est, orc.estimated_coverage)
        return "exact"
    # Different block set: must be explained by ties.
    _, scores = oracle.plan(q, bs, cfg)
    id2score = {int(i): s for i, s in zip(bs.ids, scores)}
    n_common = min(gpu_bp, orc.blocks_processed)
    g_set = set(map(int, gpu_ids[:n_common]))
    o_set = set(map(int, orc.processed_ids[:n_common]))
    diff = g_set ^ o_set
    if diff:
        # every swapped block must tie (within SCORE_TIE) with the boundary score
        bscore = sorted(id2score[i] for i in o_set)[0] if o_set else 0.0
        for i in diff:
            assert abs(id2score[i] - bscore) <= SCORE_TIE * max(1.0, abs(bscore)), ("ranking differs", i)
    if gpu_bp != orc.blocks_processed:
        eps = 1.0 if topk else cfg.epsilon
        m = cfg.microbatch_size
        # oracle estimate at the boundary where the GPU stopped / the oracle stopped
        k_gpu = (gpu_bp + m - 1) // m - 1
        k_orc = (orc.blocks_processed + m - 1) // m - 1
        k = min(k_gpu, k_orc)
        est_k = orc.iteration_estimates[k]
        assert abs(est_k - eps) <= TAU, ("stop point differs beyond tau", gpu_bp, orc.blocks_processed, est_k, eps)
    # output vs the fp64 exact attention over the GPU's own block set
    pos = {int(i): j for j, i in enumerate(bs.ids)}
    sel = np.array([pos[int(i)] for i in gpu_ids[:gpu_bp]], np.int64)
    scale = cfg.scale_override if cfg.scale_override > 0 else 1.0 / math.sqrt(bs.d)
    exact = oracle.exact_attention_blocks(q, bs, sel, scale)
    assert max_abs(gpu_out, exact) <= OUT_TOL
    return "tie"
