"""Pins the C oracle (oracle/psa_oracle.c) before it is trusted as the checker:
against the reference's own known-answer tests (test_engine.cpp, test_core.cpp,
SPEC.md examples), against the committed golden fixtures (tests/golden/, made by
tests/golden/make_golden.py from the compiled reference), and bit-for-bit against
the compiled reference itself (oracle/_ref) when it is present. CPU only."""
import json
import math
import os

import numpy as np
import pytest

from helpers import fig4_blockset, random_blockset
from oracle.pyoracle import BlockSet, make_config

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_fig4_walkthrough(oracle):
    """test_engine.cpp:130-211: m=4, eps=0.98, Oracle ranking + audit, scale 1."""
    bs, q, realized = fig4_blockset()
    cfg = make_config(epsilon=0.98, microbatch_size=4, block_size=1, ranking_mode=1, audit_coverage=1,
                      scale_override=1.0)
    r = oracle.psa(q, bs, cfg)
    assert r.blocks_processed == 12 and r.total_blocks == 16 and r.terminated_early
    assert list(r.processed_ids) == list(range(12))
    exp_cov = []
    acc, mn = 0.0, math.inf
    for i, m in enumerate(realized):
        acc += m
        mn = min(mn, m)
        if (i + 1) % 4 == 0:
            exp_cov.append(acc / (acc + mn * (16 - i - 1)))
            if exp_cov[-1] > 0.98:
                break
    assert len(exp_cov) == 3
    np.testing.assert_allclose(exp_cov, [0.6106, 0.9100, 0.9805], rtol=1e-3)
    np.testing.assert_allclose(r.iteration_estimates, exp_cov, rtol=1e-9)
    assert r.estimated_coverage == pytest.approx(exp_cov[2], rel=1e-9)
    tc = sum(realized[:12]) / sum(realized)
    assert r.true_coverage == pytest.approx(tc, rel=1e-9)
    assert r.estimated_coverage <= r.true_coverage + 1e-12
    assert oracle.psa(q, bs, make_config(epsilon=0.6, microbatch_size=4, ranking_mode=1, audit_coverage=1,
                                         scale_override=1.0)).blocks_processed == 4
    assert oracle.psa(q, bs, make_config(epsilon=0.99, microbatch_size=4, ranking_mode=1, audit_coverage=1,
                                         scale_override=1.0)).blocks_processed > 12


def test_two_token_softmax(oracle):
    """test_core.cpp:104-125: keys {0, ln 3}, values {1, 5} -> output 4."""
    k = np.array([[0.0], [np.log(np.float32(3.0))]], np.float32)
    v = np.array([[1.0], [5.0]], np.float32)
    p = oracle.block_partial(np.array([1.0], np.float32), k, v, 1.0)
    assert p["max_score"] == pytest.approx(math.log(3.0), rel=1e-6)
    assert p["exp_sum"] == pytest.approx(4.0 / 3.0, rel=1e-6)
    assert p["log_as"] == pytest.approx(math.log(4.0), rel=1e-6)
    bs = BlockSet([k], [v])
    r = oracle.psa(np.array([1.0], np.float32), bs, make_config(epsilon=1.0, scale_override=1.0))
    assert r.output[0] == pytest.approx(4.0, rel=1e-6)


def test_merge_stable_at_300(oracle):
    """test_core.cpp:250-284: scores near +-300 stay finite; all values 1 -> output 1."""
    d = 4
    big = np.zeros((2, d), np.float32)
    small = np.zeros((2, d), np.float32)
    big[0, 0], big[1, 0], small[0, 0], small[1, 0] = 300, 299, -300, -299
    ones = np.ones((2, d), np.float32)
    q = np.array([1, 0, 0, 0], np.float32)
    for order in ([small, big], [big, small]):
        bs = BlockSet(order, [ones, ones])
        r = oracle.psa(q, bs, make_config(epsilon=1.0, scale_override=1.0))
        assert np.all(np.isfinite(r.output)) and np.allclose(r.output, 1.0)


def test_metadata_examples(oracle):
    """rows [1,-2],[3,4] -> lo [1,-2], hi [3,4], mean [2,1]; single row -> all equal."""
    mean, lo, hi = oracle.build_metadata(np.array([[1, -2], [3, 4]], np.float32))
    assert list(lo) == [1, -2] and list(hi) == [3, 4] and list(mean) == [2, 1]
    k = np.array([[0.5, -7.25, 3.0]], np.float32)
    mean, lo, hi = oracle.build_metadata(k)
    assert np.array_equal(mean, k[0]) and np.array_equal(lo, k[0]) and np.array_equal(hi, k[0])


def test_cuboid_examples(oracle):
    """SPEC.md:128-129."""
    z = np.zeros(2, np.float32)
    lo, hi = np.array([0, 0], np.float32), np.array([2, 3], np.float32)
    assert oracle.criticality(np.array([1, 1], np.float32), z, lo, hi, 1, 1.0) == 5.0
    assert oracle.criticality(np.array([-1, 0], np.float32), z, lo, hi, 1, 1.0) == 0.0


def test_cuboid_is_upper_bound(oracle):
    """SPEC.md:130 / test_acceptance crit 3: bound >= every token score."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        d = int(rng.integers(1, 40))
        k = rng.standard_normal((int(rng.integers(1, 20)), d)).astype(np.float32)
        q = rng.standard_normal(d).astype(np.float32)
        mean, lo, hi = oracle.build_metadata(k)
        ub = oracle.criticality(q, mean, lo, hi, 1, 0.25)
        assert ub >= max(float(np.dot(q.astype(np.float64), r.astype(np.float64))) * 0.25 for r in k) - 1e-12


def test_rank_tie_break(oracle):
    """test_core.cpp:396-433 (ids 7,3,5 identical -> 3,5,7) and rank_by_scores example."""
    order = oracle.rank_by_scores([1.0, 3.0, 3.0, -2.0, 0.5], [10, 9, 4, 2, 3])
    assert [[10, 9, 4, 2, 3][i] for i in order] == [4, 9, 10, 3, 2]
    proto = np.array([[1, 0], [0, 1]], np.float32)
    bs = BlockSet([proto] * 3, [np.zeros((2, 2), np.float32)] * 3, ids=[7, 3, 5])
    ranked, _ = oracle.plan(np.array([1, 1], np.float32), bs, make_config(scale_override=1.0))
    assert list(ranked) == [3, 5, 7]


def test_coverage_arithmetic(oracle):
    """test_engine.cpp:75-114."""
    assert oracle.estimate_coverage(math.log(9.0), 0.0, 1) == pytest.approx(0.9, rel=1e-12)
    assert oracle.estimate_coverage(1.0, 0.5, 0) == 1.0
    assert oracle.estimate_coverage(0.0, 800.0, 3) == 0.0
    rng = np.random.default_rng(42)
    for _ in range(200):
        a = math.exp(rng.uniform(-3, 6))
        m = a * rng.uniform() + 1e-9
        nl = int(rng.integers(0, 41))
        assert oracle.estimate_coverage(math.log(a), math.log(m), nl) == pytest.approx(a / (a + m * nl), rel=1e-12)


def test_eps1_exact(oracle):
    """test_engine.cpp:213-234 / acceptance crit 1: eps=1 equals fp64 exact attention."""
    rng = np.random.default_rng(909)
    bs = random_blockset(rng, 24, 32, full=8)
    q = rng.standard_normal(32).astype(np.float32)
    r = oracle.psa(q, bs, make_config(epsilon=1.0, microbatch_size=5))
    assert r.blocks_processed == 24 and not r.terminated_early and r.estimated_coverage == 1.0
    ex = oracle.exact_attention_blocks(q, bs, np.arange(24), 1 / math.sqrt(32))
    assert np.linalg.norm(r.output - ex) / np.linalg.norm(ex) < 1e-5


def test_oracle_ranking_guarantee(oracle):
    """test_engine.cpp:236-256 / crit 2: estimate <= true coverage, true >= eps."""
    rng = np.random.default_rng(1234)
    for _ in range(10):
        bs = random_blockset(rng, 32, 16, full=4)
        for eps in (0.8, 0.9, 0.95, 0.99):
            q = rng.standard_normal(16).astype(np.float32)
            r = oracle.psa(q, bs, make_config(epsilon=eps, microbatch_size=3, ranking_mode=1, audit_coverage=1))
            assert r.estimated_coverage <= r.true_coverage + 1e-12
            assert r.true_coverage >= eps - 1e-12


def test_topk_counts(oracle):
    """test_engine.cpp:329-367."""
    rng = np.random.default_rng(555)
    bs = random_blockset(rng, 20, 16, full=4)
    q = rng.standard_normal(16).astype(np.float32)
    cfg = make_config(microbatch_size=4)
    ranked, _ = oracle.plan(q, bs, cfg)
    for k in (1, 7, 20, 50):
        r = oracle.psa(q, bs, cfg, topk=k)
        take = min(k, 20)
        assert r.blocks_processed == take and r.terminated_early == (take < 20)
        assert list(r.processed_ids) == list(ranked[:take])


def test_golden_fixtures(oracle):
    """Frozen outputs of the compiled reference (tests/golden/make_golden.py)."""
    path = os.path.join(GOLDEN, "ref_cases.json")
    cases = json.load(open(path))
    assert len(cases) >= 20
    for c in cases:
        rng = np.random.default_rng(c["seed"])
        bs = random_blockset(rng, c["n"], c["d"], 1, c["tok_hi"], planted_frac=c["planted"])
        q = (rng.standard_normal(c["d"]) * c["qscale"]).astype(np.float32)
        cfg = make_config(**c["cfg"])
        r = oracle.psa(q, bs, cfg, c["topk"])
        assert r.blocks_processed == c["blocks_processed"]
        assert list(map(int, r.processed_ids)) == c["processed_ids"]
        assert r.output.astype(np.float32).tobytes().hex() == c["output_hex"], "oracle drifted from the reference"
        assert r.estimated_coverage == c["estimated_coverage"]
        assert (r.true_coverage if r.true_coverage is not None else -1.0) == c["true_coverage"]


def test_bit_identical_to_reference(oracle, ref):
    """Random configurations: the C oracle equals the compiled reference bit for bit."""
    rng = np.random.default_rng(2024)
    for trial in range(60):
        d = int(rng.choice([2, 8, 16, 32, 64, 128]))
        n = int(rng.integers(1, 60))
        bs = random_blockset(rng, n, d, 1, 20, planted_frac=0.2, ids=rng.permutation(1000)[:n])
        st = ref.store(capacity=int(rng.integers(0, 40)))
        st.put_blockset(bs)
        q = (rng.standard_normal(d) * 2).astype(np.float32)
        cfg = make_config(epsilon=float(rng.choice([0.5, 0.8, 0.95, 0.99, 1.0])),
                          microbatch_size=int(rng.integers(1, 5)), estimator=int(rng.integers(0, 3)),
                          ranking_mode=int(rng.integers(0, 2)), audit_coverage=int(rng.integers(0, 2)))
        topk = int(rng.integers(0, 3)) * int(rng.integers(1, n + 3))
        a, b = oracle.psa(q, bs, cfg, topk), st.query(q, bs.ids, cfg, topk)
        assert a.output.tobytes() == b.output.tobytes()
        assert a.blocks_processed == b.blocks_processed
        assert np.array_equal(a.processed_ids, b.processed_ids)
        assert a.estimated_coverage == b.estimated_coverage and a.true_coverage == b.true_coverage
        assert a.terminated_early == b.terminated_early
        assert np.array_equal(a.iteration_estimates, b.iteration_estimates)


def test_cache_model_matches_reference(oracle, ref):
    """Fast-tier accounting model (store.cpp:80-124) vs the reference store."""
    import ctypes as C
    rng = np.random.default_rng(5)
    for policy in (0, 1):
        for fifo in (0, 1):
            st = ref.store(capacity=6, n_layers=2, partitioned=policy, fifo=fifo)
            cm = oracle.L.orc_cache_create(6, 2, policy, fifo)
            k = np.ones((2, 4), np.float32)
            ev = C.c_int64()
            for i in range(10):
                st.put(i, k, k, layer=i % 2)
                oracle.L.orc_cache_put(cm, i, i % 2, C.byref(ev))
            for _ in range(200):
                i = int(rng.integers(0, 10))
                q = np.ones(4, np.float32)
                st.query(q, [i], make_config(epsilon=1.0))
                oracle.L.orc_cache_load(cm, i, i % 2, 64, C.byref(ev))
            out = np.zeros(4, np.uint64)
            oracle.L.orc_cache_stats(cm, out.ctypes.data)
            s = st.stats()
            assert [s["hits"], s["misses"], s["evictions"], s["bytes_transferred"]] == list(map(int, out))
            oracle.L.orc_cache_destroy(cm)
