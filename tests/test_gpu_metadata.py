"""Per-call scoring and ranking over host metadata records on the device
(psattn_criticality_scores / psattn_rank_by_scores; the reference's criticality_score,
rank_blocks, rank_by_scores, src/metadata.cpp:41-96). Bit-exact against the C oracle and
the compiled reference; the reference's own known answers (tests/test_core.cpp:396-434)."""
import numpy as np
import pytest

from paper_2503_00392_b200 import capi


def _metas(rng, n, d):
    keys = rng.standard_normal((n, 16, d)).astype(np.float32)
    return keys.mean(1).astype(np.float32), keys.min(1), keys.max(1)


def test_entry_points_refuse_without_gpu():
    """No CPU fallback: without a CUDA device both calls fail with PSATTN_ERR_RUNTIME."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    q = np.ones(4, np.float32)
    m = np.zeros((2, 4), np.float32)
    with pytest.raises(capi.PsattnError, match="no CPU fallback"):
        capi.criticality_scores(q, m, m, m)
    with pytest.raises(capi.PsattnError, match="no CPU fallback"):
        capi.rank_by_scores([1.0, 2.0], [0, 1])


@pytest.mark.gpu
@pytest.mark.parametrize("d", [128, 64, 7])
@pytest.mark.parametrize("est", [0, 1, 2])
def test_scores_bit_exact(oracle, d, est):
    rng = np.random.default_rng(100 + d + est)
    q = rng.standard_normal(d).astype(np.float32)
    mean, lo, hi = _metas(rng, 300, d)
    got = capi.criticality_scores(q, mean, lo, hi, est)
    want = np.array([oracle.criticality(q, mean[i], lo[i], hi[i], est) for i in range(300)])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.gpu
def test_scores_match_compiled_reference(ref):
    rng = np.random.default_rng(7)
    q = rng.standard_normal(128).astype(np.float32)
    mean, lo, hi = _metas(rng, 200, 128)
    for est in (0, 1, 2):
        got = capi.criticality_scores(q, mean, lo, hi, est, scale=0.125)
        want = np.array([ref.criticality(q, mean[i], lo[i], hi[i], est, 0.125) for i in range(200)])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), est


@pytest.mark.gpu
def test_reference_known_answers():
    """The reference's known answers: SPEC.md:128-129 (cuboid examples), test_core.cpp:396-420
    (identical blocks rank by ascending id; empty list throws) and :422-434 (rank_by_scores)."""
    z = np.zeros((1, 2), np.float32)
    lo = np.array([[0.0, 0.0]], np.float32)
    hi = np.array([[2.0, 3.0]], np.float32)
    assert capi.criticality_scores(np.array([1, 1], np.float32), z, lo, hi, 1, 1.0)[0] == 5.0
    assert capi.criticality_scores(np.array([-1, 0], np.float32), z, lo, hi, 1, 1.0)[0] == 0.0
    # three identical 2-token blocks, keys (1,0),(0,1): mean (.5,.5), lo (0,0), hi (1,1)
    m3 = np.full((3, 2), 0.5, np.float32)
    order = capi.rank_blocks(np.array([1, 1], np.float32), m3, np.zeros((3, 2), np.float32),
                             np.ones((3, 2), np.float32), [7, 3, 5], 2, 1.0)
    assert [[7, 3, 5][i] for i in order] == [3, 5, 7]
    ids = [10, 9, 4, 2, 3]
    order = capi.rank_by_scores([1.0, 3.0, 3.0, -2.0, 0.5], ids)
    assert [ids[i] for i in order] == [4, 9, 10, 3, 2]


@pytest.mark.gpu
def test_upper_bound_dominates_token_scores():
    rng = np.random.default_rng(3)
    keys = rng.standard_normal((50, 16, 32)).astype(np.float32)
    q = rng.standard_normal(32).astype(np.float32)
    ub = capi.criticality_scores(q, keys.mean(1), keys.min(1), keys.max(1), 1, 0.25)
    tok = (keys.astype(np.float64) @ q.astype(np.float64)).max(1) * 0.25
    assert np.all(ub >= tok - 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 1000, 70000])
def test_rank_by_scores_ties(oracle, n):
    rng = np.random.default_rng(n)
    scores = rng.integers(0, max(2, n // 10), n).astype(np.float64) * 0.5  # many ties
    ids = rng.permutation(n * 3)[:n].astype(np.int64)
    got = capi.rank_by_scores(scores, ids)
    want = np.lexsort((ids, -scores))
    assert np.array_equal(got, want)
    if n <= 1000:
        assert np.array_equal(got, oracle.rank_by_scores(scores, ids))


@pytest.mark.gpu
def test_rank_blocks_and_edges(oracle):
    rng = np.random.default_rng(11)
    q = rng.standard_normal(128).astype(np.float32)
    mean, lo, hi = _metas(rng, 500, 128)
    ids = rng.permutation(500).astype(np.int64) + 1000
    got = capi.rank_blocks(q, mean, lo, hi, ids)
    s = np.array([oracle.criticality(q, mean[i], lo[i], hi[i], 2) for i in range(500)])
    assert np.array_equal(got, oracle.rank_by_scores(s, ids))
    assert capi.rank_by_scores(np.zeros(0), np.zeros(0, np.int64)).size == 0
    with pytest.raises(ValueError):
        capi.rank_blocks(q, mean[:0], lo[:0], hi[:0], [])
    with pytest.raises(capi.PsattnError, match="unknown estimator"):
        capi.criticality_scores(q, mean, lo, hi, 3)
