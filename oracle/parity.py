"""The parity rule — TEST INFRASTRUCTURE (the checker, never the thing measured).

Used by tests/ (through tests/helpers.py) and by bench.py's post-timing `--check` leg.

Parity rule (BASELINE.json north_star, SURVEY.md §7 hard part 2):
  * ranked/processed block sets identical, except where estimated scores tie
    within SCORE_TIE (1e-6) or the stop decision sits within TAU (1e-5) of eps;
  * outputs within OUT_TOL (1e-3) max-abs (fp32 accumulate); when the block
    set legitimately differs, the output is checked against the fp64 exact
    attention over the GPU's own block set.
"""
from __future__ import annotations

import math
import os
import threading

import numpy as np

from oracle.pyoracle import BlockSet

SCORE_TIE = 1e-6
TAU = 1e-5
OUT_TOL = 1e-3


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


def check_sampled_units(p, units, n_tokens, eps, microbatch=1, threads=8):
    """Checks GPU results of whole GQA units against the reference on the SAME synthetic data.

    p: workload.synth params (the generator the benchmark's pool was filled with).
    units: list of dicts {uid, q [g, d], out [g, d], bp [g], ids: list of g arrays of the processed
    list positions (rank order)} taken from the device run.
    Each unit is regenerated on the host (bf16-rounded values upcast to fp32, as the pool holds
    them) and run through the COMPILED REFERENCE's psa_attention_multi_head (reference
    engine.cpp:240-260) when oracle/_ref exists, else the C oracle port head by head. The parity
    rule above decides each query ('exact' or 'tie'); a violation raises AssertionError.
    Returns {units, queries, exact, tie, max_abs_err, oracle}."""
    from oracle.pyoracle import COracle, RefDriver, make_config, ref_available
    from workload import synth

    cfg = make_config(epsilon=eps, microbatch_size=microbatch)
    orc = COracle()
    drv = RefDriver() if ref_available() else None
    tags, errs, lock = [], [], threading.Lock()
    failures = []

    def one(unit):
        try:
            k, v = synth.unit_host(p, int(unit["uid"]), n_tokens)
            n = k.shape[0]
            T = p.block_tokens
            nt = [min(T, n_tokens - b * T) for b in range(n)]
            bs = BlockSet([k[b, : nt[b]] for b in range(n)], [v[b, : nt[b]] for b in range(n)])
            qs = np.asarray(unit["q"], np.float32)
            g = qs.shape[0]
            if drv is not None:
                st = drv.store(capacity=0)
                if all(x == T for x in nt):
                    st.put_many(0, k, v)
                else:
                    st.put_blockset(bs)
                res, _ = st.multi_head(qs, np.arange(n, dtype=np.int64)[None, :], cfg)
                del st
            else:
                res = [orc.psa(qs[h], bs, cfg) for h in range(g)]
            loc_tags, loc_err = [], 0.0
            for h in range(g):
                ids = np.asarray(unit["ids"][h], np.int64)
                bp = int(unit["bp"][h])
                out = np.asarray(unit["out"][h], np.float32)
                r = res[h]
                if bp == r.blocks_processed and np.array_equal(ids[:bp], r.processed_ids):
                    err = max_abs(out, r.output)
                    assert err <= OUT_TOL, ("output", int(unit["uid"]), h, err)
                    loc_tags.append("exact")
                    loc_err = max(loc_err, err)
                else:  # the C oracle (bit-identical to the reference) judges ties / stop points
                    loc_tags.append(check_parity(orc, qs[h], bs, cfg, 0, ids, bp, out, None))
            with lock:
                tags.extend(loc_tags)
                errs.append(loc_err)
        except AssertionError as e:  # noqa: PERF203
            with lock:
                failures.append((int(unit["uid"]), repr(e)))

    pending = list(units)
    while pending:
        batch, pending = pending[:threads], pending[threads:]
        ths = [threading.Thread(target=one, args=(u,)) for u in batch]
        [t.start() for t in ths]
        [t.join() for t in ths]
    if failures:
        raise AssertionError(f"parity violated on {len(failures)} unit(s): {failures[:3]}")
    return dict(units=len(units), queries=len(tags), exact=tags.count("exact"), tie=tags.count("tie"),
                max_abs_err=float(max(errs) if errs else 0.0),
                oracle="compiled reference psa_attention_multi_head" if drv is not None else "C oracle port")

