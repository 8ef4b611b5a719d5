"""C ABI on the GPU: the reference's test_capi.cpp cases re-stated against
libpsattn_b200.so, plus parity of psattn_run_query / psattn_run_topk with the
oracle (and the compiled reference's store accounting when present)."""
import numpy as np
import pytest

from helpers import OUT_TOL, check_parity, fig4_blockset, max_abs, random_blockset
from oracle.pyoracle import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_2503_00392_b200 import capi as c
    return c


def test_store_create_validation(capi):
    import ctypes as C
    o = capi.store_options_default()
    h = C.c_void_p()
    assert capi.lib.psattn_store_create(None, C.byref(h)) == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert capi.lib.psattn_store_create(C.byref(o), None) == capi.PSATTN_ERR_INVALID_ARGUMENT
    o.fast_capacity_slots = -1
    assert capi.lib.psattn_store_create(C.byref(o), C.byref(h)) == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert len(capi.last_error()) > 0
    o = capi.store_options_default()
    o.pool_policy = 42
    assert capi.lib.psattn_store_create(C.byref(o), C.byref(h)) == capi.PSATTN_ERR_INVALID_ARGUMENT
    o = capi.store_options_default()
    o.eviction_policy = -3
    assert capi.lib.psattn_store_create(C.byref(o), C.byref(h)) == capi.PSATTN_ERR_INVALID_ARGUMENT
    o = capi.store_options_default()
    o.n_layers = 0
    assert capi.lib.psattn_store_create(C.byref(o), C.byref(h)) != capi.PSATTN_OK
    o = capi.store_options_default()
    assert capi.lib.psattn_store_create(C.byref(o), C.byref(h)) == capi.PSATTN_OK
    capi.lib.psattn_store_destroy(h)
    capi.lib.psattn_store_destroy(None)


def test_put_contains_stats_release(capi):
    """test_capi.cpp:131-189."""
    s = capi.Store(capacity=2)
    k = np.full((3, 16), 0.25, np.float32)
    import ctypes as C
    assert capi.lib.psattn_store_put_block(None, 0, 0, 7, 3, 16, k.ctypes.data, k.ctypes.data) == 1
    assert capi.lib.psattn_store_put_block(s.h, 0, 0, 7, 3, 16, None, k.ctypes.data) == 1
    assert capi.lib.psattn_store_put_block(s.h, 0, 0, 7, 0, 16, k.ctypes.data, k.ctypes.data) == 1
    for i in range(4):
        assert s.put(i, k, k, owner=7) == capi.PSATTN_OK
    assert s.put(2, k, k, owner=7) == capi.PSATTN_ERR_RUNTIME  # duplicate id
    assert s.contains(3) == (0, True)
    assert s.contains(0) == (0, False)
    assert s.contains(99)[0] == capi.PSATTN_ERR_NOT_FOUND
    st = s.stats()
    assert st == dict(hits=0, misses=0, evictions=2, bytes_transferred=0)
    cfg = capi.config_default(epsilon=1.0, microbatch_size=4)
    rc, r = s.run_query(np.full(16, 0.1, np.float32), [0, 1, 2, 3], cfg)
    assert rc == 0
    st = s.stats()
    assert st["hits"] + st["misses"] == 4
    assert st["bytes_transferred"] == st["misses"] * 384
    assert (r.blocks_processed, r.total_blocks, r.terminated_early) == (4, 4, False)
    assert np.allclose(r.output, 0.25)
    assert s.release(7) == 0
    assert s.contains(3)[0] == capi.PSATTN_ERR_NOT_FOUND
    assert s.release(7) == capi.PSATTN_ERR_NOT_FOUND
    assert capi.lib.psattn_store_stats(s.h, None) == capi.PSATTN_ERR_INVALID_ARGUMENT


def test_config_validation_codes(capi):
    """test_capi.cpp:191-236."""
    rng = np.random.default_rng(11)
    s = capi.Store()
    bs = random_blockset(rng, 4, 16, full=3)
    s.put_blockset(bs)
    q = rng.standard_normal(16).astype(np.float32)
    for kw in (dict(epsilon=0.0), dict(epsilon=1.5), dict(microbatch_size=0), dict(estimator=9),
               dict(ranking_mode=9)):
        assert s.run_query(q, bs.ids, capi.config_default(**kw))[0] == capi.PSATTN_ERR_INVALID_ARGUMENT
    cfg = capi.config_default()
    import ctypes as C
    out = np.zeros(16, np.float32)
    assert capi.lib.psattn_run_query(s.h, q.ctypes.data, 16, bs.ids.ctypes.data, 0, C.byref(cfg), out.ctypes.data,
                                     None) == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert capi.lib.psattn_run_query(s.h, None, 16, bs.ids.ctypes.data, 4, C.byref(cfg), out.ctypes.data,
                                     None) == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert s.run_topk(q, bs.ids, 0, cfg)[0] == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert s.run_query(q, [0, 99], cfg)[0] == capi.PSATTN_ERR_NOT_FOUND
    assert s.run_query(q[:8], bs.ids, cfg)[0] == capi.PSATTN_ERR_RUNTIME  # dim mismatch
    # NULL cfg selects the defaults
    assert capi.lib.psattn_run_query(s.h, q.ctypes.data, 16, bs.ids.ctypes.data, 4, None, out.ctypes.data,
                                     None) == capi.PSATTN_OK


def test_fig4_on_device(capi):
    """Reference KAT test_engine.cpp:130-211 through psattn_run_query (Oracle ranking + audit)."""
    bs, q, realized = fig4_blockset()
    s = capi.Store(capacity=16)
    s.put_blockset(bs)
    cfg = capi.config_default(epsilon=0.98, microbatch_size=4, block_size=1, ranking_mode=1, audit_coverage=1,
                              scale_override=1.0)
    rc, r = s.run_query(q, bs.ids, cfg)
    assert rc == 0, capi.last_error()
    assert (r.blocks_processed, r.total_blocks, r.terminated_early) == (12, 16, True)
    assert r.estimated_coverage == pytest.approx(0.9805, rel=1e-3)
    assert r.true_coverage == pytest.approx(sum(realized[:12]) / sum(realized), rel=1e-9)
    assert r.estimated_coverage <= r.true_coverage + 1e-12
    # outputs reveal which blocks were processed: weighted mean of values of ids 0..11
    w = np.array(realized[:12])
    vals = np.array([[i + 1, 2 * i + 1] for i in range(12)], np.float64)
    assert max_abs(r.output, (w[:, None] * vals).sum(0) / w.sum()) <= OUT_TOL
    cfg.epsilon = 0.6
    assert s.run_query(q, bs.ids, cfg)[1].blocks_processed == 4
    cfg.epsilon = 0.99
    assert s.run_query(q, bs.ids, cfg)[1].blocks_processed > 12


@pytest.mark.parametrize("seed", range(12))
def test_run_query_parity(capi, oracle, seed):
    rng = np.random.default_rng(100 + seed)
    d = int(rng.choice([8, 16, 32, 64, 128]))
    n = int(rng.integers(1, 200))
    ids = rng.permutation(10_000)[:n]
    bs = random_blockset(rng, n, d, 1, 16, planted_frac=float(rng.choice([0.0, 0.1])), ids=ids)
    s = capi.Store(capacity=64)
    s.put_blockset(bs)
    q = (rng.standard_normal(d) * 2).astype(np.float32)
    kw = dict(epsilon=float(rng.choice([0.5, 0.8, 0.9, 0.95, 0.99, 1.0])), microbatch_size=int(rng.integers(1, 6)),
              estimator=int(rng.integers(0, 3)), ranking_mode=int(rng.integers(0, 2)),
              audit_coverage=int(rng.integers(0, 2)))
    topk = int(rng.integers(0, 2)) * int(rng.integers(1, n + 5))
    ccfg, ocfg = capi.config_default(**kw), make_config(**kw)
    rc, r = s.run_topk(q, ids, topk, ccfg) if topk else s.run_query(q, ids, ccfg)
    assert rc == 0, capi.last_error()
    o = oracle.psa(q, bs, ocfg, topk)
    assert r.total_blocks == o.total_blocks
    if r.blocks_processed == o.blocks_processed:
        assert max_abs(r.output, o.output) <= OUT_TOL
        assert r.estimated_coverage == pytest.approx(o.estimated_coverage, abs=1e-4)
        assert r.terminated_early == o.terminated_early
        if o.true_coverage is not None:
            assert r.true_coverage == pytest.approx(o.true_coverage, abs=1e-9)
    else:
        # only a stop decision within tau of eps may differ
        m = ocfg.microbatch_size
        k = min(r.blocks_processed, o.blocks_processed)
        est_k = o.iteration_estimates[(k + m - 1) // m - 1]
        assert abs(est_k - (1.0 if topk else ocfg.epsilon)) <= 1e-5


def test_store_accounting_matches_reference(capi, ref):
    """Hit/miss/eviction/bytes after a query stream equal the reference store's."""
    rng = np.random.default_rng(9)
    d = 16
    bs = random_blockset(rng, 40, d, 1, 8)
    for policy, evict in ((0, 0), (0, 1), (1, 0)):
        mine = capi.Store(capacity=12, n_layers=2, policy=policy, eviction=evict)
        theirs = ref.store(capacity=12, n_layers=2, partitioned=policy, fifo=evict)
        for i in range(bs.n):
            k, v = bs.block(i)
            assert mine.put(int(bs.ids[i]), k, v, layer=i % 2, owner=i % 3) == 0
            theirs.put(int(bs.ids[i]), k, v, layer=i % 2, owner=i % 3)
        for t in range(15):
            sel = rng.choice(bs.n, size=int(rng.integers(3, 20)), replace=False)
            q = rng.standard_normal(d).astype(np.float32) * 3
            kw = dict(epsilon=float(rng.choice([0.5, 0.9, 1.0])), microbatch_size=int(rng.integers(1, 4)))
            rc, r = mine.run_query(q, bs.ids[sel], capi.config_default(**kw))
            o = theirs.query(q, bs.ids[sel], make_config(**kw))
            assert rc == 0
            if r.blocks_processed != o.blocks_processed:
                continue  # a tie at the stop boundary would make the streams diverge; rare
            assert mine.stats() == theirs.stats(), (policy, evict, t)
        for i in range(bs.n):
            assert mine.contains(int(bs.ids[i]))[1] == theirs.contains(int(bs.ids[i]))
        assert mine.release(1) == 0 and theirs.release(1) == 0


@pytest.mark.parametrize("seed", range(6))
def test_long_blocks_parity(capi, oracle, seed):
    """Blocks of 33..128 tokens (the reference accepts any n_tokens, types.hpp:29-48): the chunked
    per-head kernel scores them in 32-token chunks folded online; parity with the oracle."""
    rng = np.random.default_rng(500 + seed)
    d = int(rng.choice([16, 64, 128, 256]))
    n = int(rng.integers(2, 80))
    ids = rng.permutation(5_000)[:n]
    bs = random_blockset(rng, n, d, 1, 128, planted_frac=0.1, ids=ids)
    s = capi.Store(capacity=64)
    s.put_blockset(bs)
    q = (rng.standard_normal(d) * 2).astype(np.float32)
    kw = dict(epsilon=float(rng.choice([0.8, 0.95, 1.0])), microbatch_size=int(rng.integers(1, 4)),
              audit_coverage=int(seed % 2))
    rc, r = s.run_query(q, ids, capi.config_default(**kw))
    assert rc == 0, capi.last_error()
    o = oracle.psa(q, bs, make_config(**kw))
    if r.blocks_processed == o.blocks_processed:
        assert max_abs(r.output, o.output) <= OUT_TOL
        assert r.estimated_coverage == pytest.approx(o.estimated_coverage, abs=1e-4)
    else:
        m = kw["microbatch_size"]
        k = min(r.blocks_processed, o.blocks_processed)
        assert abs(o.iteration_estimates[(k + m - 1) // m - 1] - kw["epsilon"]) <= 1e-5
    # > 128 tokens is refused with a clear error (not silently truncated)
    big = rng.standard_normal((129, d)).astype(np.float32)
    assert s.put(99_999, big, big) == capi.PSATTN_ERR_RUNTIME


@pytest.mark.parametrize("case", ["disjoint", "shared", "wide_group"])
def test_run_multi_head_matches_reference(capi, ref, case):
    """psattn_run_multi_head (reference psa_attention_multi_head, engine.cpp:240-260) against the
    compiled reference on the same store contents: per-head outputs / blocks processed, the
    fetched-union size (sorted distinct ids over every head, engine.cpp:255-258) and the store's
    accounting afterwards. Ids mix the direct-indexed range, negatives and values beyond 2^24
    (the store's id table, csrc/block_table.h); `shared` gives kv-head lists common ids; a group
    wider than 8 runs one list per q-head."""
    rng = np.random.default_rng({"disjoint": 1, "shared": 2, "wide_group": 3}[case])
    d, n, hkv = 32, 60, 2
    g = 12 if case == "wide_group" else 3
    pool = np.concatenate([rng.permutation(1000)[:70], -5 - rng.permutation(1000)[:70],
                           (1 << 40) + rng.permutation(1000)[:70]])
    rng.shuffle(pool)
    bs = random_blockset(rng, pool.size, d, 1, 16, planted_frac=0.1, ids=pool)
    mine = capi.Store(capacity=150, n_layers=1)
    theirs = ref.store(capacity=150, n_layers=1)
    for i in range(bs.n):
        k, v = bs.block(i)
        assert mine.put(int(bs.ids[i]), k, v, owner=i % 2) == 0
        theirs.put(int(bs.ids[i]), k, v, owner=i % 2)
    if case == "shared":
        a = rng.permutation(bs.n)[:n]
        b = np.concatenate([a[: n // 2], rng.permutation(np.setdiff1d(np.arange(bs.n), a))[: n - n // 2]])
        kv = np.stack([bs.ids[a], bs.ids[b]])
    else:
        sel = rng.permutation(bs.n)[: hkv * n]
        kv = bs.ids[sel].reshape(hkv, n)
    qs = (rng.standard_normal((hkv * g, d)) * 2).astype(np.float32)
    for eps, m in ((0.9, 1), (0.97, 3)):
        cfg = capi.config_default(epsilon=eps, microbatch_size=m)
        rc, out, res, un = mine.run_multi_head(qs, list(kv), cfg)
        assert rc == 0, capi.last_error()
        want, wuni = theirs.multi_head(qs, kv, make_config(epsilon=eps, microbatch_size=m))
        same = all(r.blocks_processed == w.blocks_processed for r, w in zip(res, want))
        if not same:
            continue  # a tie at a stop boundary (rare): covered by the per-query parity tests
        for h in range(hkv * g):
            assert max_abs(out[h], want[h].output) <= OUT_TOL
        assert un == wuni.size
        assert mine.stats() == theirs.stats()
    assert mine.release(1) == 0 and theirs.release(1) == 0
    for i in range(bs.n):
        rc, res = mine.contains(int(bs.ids[i]))
        t = theirs.contains(int(bs.ids[i]))  # None: not in the store
        assert (rc == capi.PSATTN_ERR_NOT_FOUND) == (t is None) and (t is None or res == t)
    # a released id can be put again (its handle is reused) and is then resident
    k, v = bs.block(1)
    assert mine.put(int(bs.ids[1]), k, v, owner=1) == 0
    theirs.put(int(bs.ids[1]), k, v, owner=1)
    assert mine.contains(int(bs.ids[1])) == (0, True) and theirs.contains(int(bs.ids[1]))
    assert mine.stats() == theirs.stats()


def _to_bf16_exact(x):
    b = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).view(np.float32)


@pytest.mark.parametrize("d,g", [(128, 4), (64, 2), (32, 3)])
def test_lossless_bf16_store_and_migration(capi, ref, d, g):
    """Blocks whose values are all exact bf16 (an upcast bf16 KV cache) are stored losslessly in a
    bf16 pool (the production kernels); the first block that is not moves every stored block to an
    fp32 pool. Query results before and after the move match the compiled reference on the same
    fp32 values, and match a store that held fp32 from the start."""
    from oracle.pyoracle import BlockSet
    rng = np.random.default_rng(d + g)
    n, hkv = 300, 2
    raw = random_blockset(rng, n, d, 16, 16, planted_frac=0.05, skew=4.0, ids=np.arange(n) * 3 + 1)
    blocks = [raw.block(i) for i in range(n)]
    bs = BlockSet([_to_bf16_exact(k) for k, _ in blocks], [_to_bf16_exact(v) for _, v in blocks], raw.ids)
    odd = rng.standard_normal((16, d)).astype(np.float32)  # not bf16-exact
    mine = capi.Store(capacity=2 * n, n_layers=1)
    f32 = capi.Store(capacity=2 * n, n_layers=1)
    theirs = ref.store(capacity=2 * n, n_layers=1)
    assert f32.put(10**6, odd, odd) == 0  # fp32 pool from the first block
    for s in (mine, f32, theirs):
        s.put_blockset(bs)
    kv = bs.ids[rng.permutation(n)[: hkv * (n // hkv)]].reshape(hkv, -1)
    qs = (rng.standard_normal((hkv * g, d)) * 2).astype(np.float32)
    cfg = dict(epsilon=0.9, microbatch_size=2)

    def check(tag):
        rc, out, res, un = mine.run_multi_head(qs, list(kv), capi.config_default(**cfg))
        assert rc == 0, capi.last_error()
        rc2, out2, res2, _ = f32.run_multi_head(qs, list(kv), capi.config_default(**cfg))
        assert rc2 == 0, capi.last_error()
        want, wuni = theirs.multi_head(qs, kv, make_config(**cfg))
        if all(r.blocks_processed == w.blocks_processed for r, w in zip(res, want)):
            for h in range(hkv * g):
                assert max_abs(out[h], want[h].output) <= OUT_TOL, tag
            assert un == wuni.size
            assert mine.stats() == theirs.stats()
        if all(r.blocks_processed == w.blocks_processed for r, w in zip(res2, res)):
            assert max_abs(out, out2) <= OUT_TOL, tag

    check("bf16 pool")
    assert mine.put(10**6, odd, odd) == 0  # moves the 300 stored blocks to an fp32 pool
    theirs.put(10**6, odd, odd)
    check("after the move")


def test_repeated_queries_across_pool_growth_and_knobs(capi, ref):
    """The store replays a captured launch sequence for a repeated query shape: it
    must see blocks put since (contents), a pool that grew (new device buffers), and launch knobs
    changed in between (psattn_set_*), each time matching the compiled reference."""
    import ctypes as C
    rng = np.random.default_rng(77)
    from oracle.pyoracle import BlockSet
    d, g = 128, 4  # bf16-exact values: the bf16 pool, stream kernel and dense hand-over

    def exact(b):
        blocks = [b.block(i) for i in range(b.ids.size)]
        return BlockSet([_to_bf16_exact(k) for k, _ in blocks], [_to_bf16_exact(v) for _, v in blocks], b.ids)
    mine = capi.Store(capacity=4096, n_layers=1)
    theirs = ref.store(capacity=4096, n_layers=1)
    ids = np.arange(200, dtype=np.int64)
    bs = exact(random_blockset(rng, ids.size, d, 16, 16, planted_frac=0.1, ids=ids))
    for s in (mine, theirs):
        s.put_blockset(bs)
    qs = (rng.standard_normal((g, d)) * 2).astype(np.float32)
    cfg = dict(epsilon=0.9, microbatch_size=1)

    def run(lst):
        rc, out, res, un = mine.run_multi_head(qs, [lst], capi.config_default(**cfg))
        assert rc == 0, capi.last_error()
        want, wuni = theirs.multi_head(qs, lst[None, :], make_config(**cfg))
        if all(r.blocks_processed == w.blocks_processed for r, w in zip(res, want)):
            assert max_abs(out, np.stack([w.output for w in want])) <= OUT_TOL
            assert un == wuni.size
            assert mine.stats() == theirs.stats()

    for _ in range(3):
        run(ids)
    # overwrite nothing, but put 600 more blocks: the pool doubles (new device buffers)
    more = np.arange(1000, 1600, dtype=np.int64)
    bs2 = exact(random_blockset(rng, more.size, d, 16, 16, planted_frac=0.2, ids=more))
    for s in (mine, theirs):
        s.put_blockset(bs2)
    for _ in range(2):
        run(ids)
    both = np.concatenate([ids, more[:56]])  # a new shape
    run(both)
    try:
        assert capi.lib.psattn_set_dense_partial(C.c_int32(0)) == 0
        run(ids)
        run(both)
    finally:
        capi.lib.psattn_set_dense_partial(C.c_int32(1024))
