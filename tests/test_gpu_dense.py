"""Dense hand-over of the GQA path (kernels_dense.cu): units whose heads need more than the first
384 ranks (weakly skewed / isotropic keys) are redone by one K pass, a per-head stop rule
over the masses in rank order and one V pass. Parity with the C oracle for every head, and
equivalence with the round kernel run to the end (psattn_set_dense(1))."""
import numpy as np
import pytest

from helpers import check_parity
from oracle.pyoracle import BlockSet, make_config
from workload import synth  # fixture: the seekable synthetic generator

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def mods():
    from paper_2503_00392_b200 import batch, capi
    return capi, batch


def synth_batch(mods, tokens, g, planted, cfg, seed=5):
    capi, batch = mods
    d, T = 128, 16
    p = synth.params(seed=seed, dim=d, block_tokens=T, skew=8.0, planted_prob=planted, round_bf16=1)
    nb = [(t + T - 1) // T for t in tokens]
    off = np.zeros(len(tokens) + 1, np.int64)
    off[1:] = np.cumsum(nb)
    uids = [40 + i for i in range(len(tokens))]
    pool = batch.DevicePool(d, T, capi.PSATTN_KV_BF16, int(off[-1]))
    synth.fill(pool, p, uids, off[:-1], tokens)
    dev = torch.device("cuda")
    qs = np.array([[synth.query(p, uid, h) for h in range(g)] for uid in uids], np.float32)
    run = batch.BatchRun(pool, torch.tensor(qs, device=dev), torch.arange(int(off[-1]), dtype=torch.int32, device=dev),
                         torch.tensor(off, device=dev), max(nb), batch.BatchConfig(**cfg), want_ranked=True)
    return p, uids, nb, off, qs, run


def results(run, off, nb, g):
    torch.cuda.synchronize()
    out = []
    for u in range(len(nb)):
        for h in range(g):
            qi = u * g + h
            bp = int(run.bp[qi])
            hb = int(off[u]) * g + h * nb[u]
            out.append(dict(bp=bp, ids=run.ranked[hb: hb + bp].cpu().numpy(), out=run.out[u, h].cpu().numpy(),
                            est=float(run.est[qi]), term=int(run.term[qi])))
    return out


@pytest.mark.parametrize("g", [4, 3, 2])
@pytest.mark.parametrize("cfg", [dict(epsilon=0.95), dict(epsilon=0.9, microbatch_size=4), dict(topk=1200),
                                 dict(epsilon=0.99, estimator=0)])
def test_dense_handover_parity(mods, oracle, g, cfg):
    capi, _ = mods
    tokens = [16 * 3000 + 7, 16 * 1500]  # isotropic: every head needs most of its list
    p, uids, nb, off, qs, run = synth_batch(mods, tokens, g, 0.0, cfg)
    assert capi.lib.psattn_set_dense(0) == 0
    run.run()
    dense = results(run, off, nb, g)
    assert capi.lib.psattn_set_dense(1) == 0
    try:
        run.run()
        rounds = results(run, off, nb, g)
    finally:
        capi.lib.psattn_set_dense(0)
    assert max(r["bp"] for r in dense) > 384  # the hand-over was exercised
    oc = make_config(epsilon=cfg.get("epsilon", 1.0) if not cfg.get("topk") else 1.0,
                     microbatch_size=cfg.get("microbatch_size", 1), estimator=cfg.get("estimator", 2))
    for u, uid in enumerate(uids):
        k, v = synth.unit_host(p, uid, tokens[u])
        nt = [min(16, tokens[u] - i * 16) for i in range(nb[u])]
        bs = BlockSet([k[i, :nt[i]] for i in range(nb[u])], [v[i, :nt[i]] for i in range(nb[u])])
        for h in range(g):
            a, b = dense[u * g + h], rounds[u * g + h]
            check_parity(oracle, qs[u, h], bs, oc, cfg.get("topk", 0), a["ids"], a["bp"], a["out"], a["est"])
            # identical masses and decide arithmetic: same processed sets and stop points as the round kernel
            assert a["bp"] == b["bp"] and np.array_equal(a["ids"], b["ids"]) and a["term"] == b["term"]
            assert abs(a["est"] - b["est"]) <= 1e-6
            assert np.max(np.abs(a["out"] - b["out"])) <= 1e-4


def test_planted_units_stay_on_round_kernel(mods):
    """Sparse (planted) units finish inside their first tranche, never handed over: dense on (64-rank
    rounds) and off (32-rank rounds) process the same blocks; outputs agree up to summation order."""
    capi, _ = mods
    tokens = [16 * 4096, 16 * 2048 + 3]
    p, uids, nb, off, qs, run = synth_batch(mods, tokens, 4, 1 / 32, dict(epsilon=0.95))
    run.run()
    a = results(run, off, nb, 4)
    assert capi.lib.psattn_set_dense(1) == 0
    try:
        run.run()
        b = results(run, off, nb, 4)
    finally:
        capi.lib.psattn_set_dense(0)
    assert max(r["bp"] for r in a) < 384
    for x, y in zip(a, b):
        assert x["bp"] == y["bp"] and np.array_equal(x["ids"], y["ids"]) and abs(x["est"] - y["est"]) <= 1e-6
        assert np.max(np.abs(x["out"] - y["out"])) <= 1e-5


@pytest.mark.parametrize("g", [4, 3, 2])
@pytest.mark.parametrize("cfg", [dict(epsilon=0.95), dict(epsilon=0.9, microbatch_size=3), dict(topk=100)])
def test_wide_rounds_parity(mods, oracle, g, cfg):
    """64-rank rounds of the tensor-core path on planted (sparse) units, every head vs the oracle."""
    capi, _ = mods
    tokens = [16 * 2500 + 9, 16 * 800]
    p, uids, nb, off, qs, run = synth_batch(mods, tokens, g, 1 / 32, cfg, seed=9)
    run.run()
    res = results(run, off, nb, g)
    oc = make_config(epsilon=cfg.get("epsilon", 1.0) if not cfg.get("topk") else 1.0,
                     microbatch_size=cfg.get("microbatch_size", 1))
    for u, uid in enumerate(uids):
        k, v = synth.unit_host(p, uid, tokens[u])
        nt = [min(16, tokens[u] - i * 16) for i in range(nb[u])]
        bs = BlockSet([k[i, :nt[i]] for i in range(nb[u])], [v[i, :nt[i]] for i in range(nb[u])])
        for h in range(g):
            a = res[u * g + h]
            check_parity(oracle, qs[u, h], bs, oc, cfg.get("topk", 0), a["ids"], a["bp"], a["out"], a["est"])


@pytest.mark.parametrize("cfg", [dict(topk=1200), dict(epsilon=0.999)])
def test_dense_decide_crowded_bins(mods, oracle, cfg):
    """Hand-over units whose keys crowd one score bin (1500 identical blocks: equal scores, ties by
    position): dense_decide_kernel's bucket sort declines and the bitonic fallback orders them. Same
    processed sets as the round kernel, and the oracle's parity rule."""
    capi, batch = mods
    d, T, g, n = 128, 16, 4, 2000
    rng = np.random.default_rng(21)
    K = rng.standard_normal((n, T, d)).astype(np.float32)
    K[:1500] = K[0]
    V = rng.standard_normal((n, T, d)).astype(np.float32)
    pool = batch.DevicePool(d, T, capi.PSATTN_KV_BF16, n)
    pool.put_blocks(np.arange(n), np.full(n, T), K, V)
    dev = torch.device("cuda")
    qs = (0.3 * rng.standard_normal((1, g, d))).astype(np.float32)
    off = np.array([0, n], np.int64)
    run = batch.BatchRun(pool, torch.tensor(qs, device=dev), torch.arange(n, dtype=torch.int32, device=dev),
                         torch.tensor(off, device=dev), n, batch.BatchConfig(**cfg), want_ranked=True)
    assert capi.lib.psattn_set_dense(0) == 0
    run.run()
    dense = results(run, off, [n], g)
    assert capi.lib.psattn_set_dense(1) == 0
    try:
        run.run()
        rounds = results(run, off, [n], g)
    finally:
        capi.lib.psattn_set_dense(0)
    assert max(r["bp"] for r in dense) > 384
    # the pool holds bf16 K/V: the oracle sees the same rounded blocks
    kb = torch.tensor(K).to(torch.bfloat16).float().numpy()
    vb = torch.tensor(V).to(torch.bfloat16).float().numpy()
    bs = BlockSet([kb[i] for i in range(n)], [vb[i] for i in range(n)])
    oc = make_config(epsilon=cfg.get("epsilon", 1.0), microbatch_size=1, estimator=2)
    for h in range(g):
        a, b = dense[h], rounds[h]
        assert a["bp"] == b["bp"] and np.array_equal(a["ids"], b["ids"]) and a["term"] == b["term"]
        assert np.max(np.abs(a["out"] - b["out"])) <= 1e-4
        check_parity(oracle, qs[0, h], bs, oc, cfg.get("topk", 0), a["ids"], a["bp"], a["out"], a["est"])


@pytest.mark.parametrize("cfg", [dict(epsilon=0.99), dict(epsilon=0.99, microbatch_size=4), dict(topk=1500)])
def test_dense_partial_prefix(mods, oracle, cfg):
    """Partial dense mode: round 0 computes only each head's candidate prefix (~ranks keys) and
    decides on it, heads that do not stop inside it send their unit to round 1 (rest of the K
    pass, full decide). Every prefix size gives the same processed sets, stop points and
    outputs (bit for bit) as the whole-list pass, and parity with the oracle."""
    capi, _ = mods
    g = 4
    tokens = [16 * 6000 + 5, 16 * 9000, 16 * 5000 + 11]  # planted 1/32 at eps 0.99: heads need 400+ ranks
    p, uids, nb, off, qs, run = synth_batch(mods, tokens, g, 1 / 32, cfg, seed=9)
    got = {}
    try:
        for ranks in (0, 64, 700, 1024, 2048):
            assert capi.lib.psattn_set_dense_partial(ranks) == 0
            run.run()
            got[ranks] = results(run, off, nb, g)
    finally:
        capi.lib.psattn_set_dense_partial(1024)
    assert max(r["bp"] for r in got[0]) > 384  # the hand-over was exercised
    for ranks in (64, 700, 1024, 2048):
        for a, b in zip(got[ranks], got[0]):
            assert a["bp"] == b["bp"] and np.array_equal(a["ids"], b["ids"]) and a["term"] == b["term"]
            assert np.array_equal(a["out"], b["out"]) and a["est"] == b["est"]
    oc = make_config(epsilon=cfg.get("epsilon", 1.0), microbatch_size=cfg.get("microbatch_size", 1))
    for u, uid in enumerate(uids):
        k, v = synth.unit_host(p, uid, tokens[u])
        nt = [min(16, tokens[u] - i * 16) for i in range(nb[u])]
        bs = BlockSet([k[i, :nt[i]] for i in range(nb[u])], [v[i, :nt[i]] for i in range(nb[u])])
        for h in range(g):
            a = got[1024][u * g + h]
            check_parity(oracle, qs[u, h], bs, oc, cfg.get("topk", 0), a["ids"], a["bp"], a["out"], a["est"])


def test_dense_partial_setter(mods):
    capi, _ = mods
    assert capi.lib.psattn_set_dense_partial(-1) != 0
    assert capi.lib.psattn_set_dense_partial(1024) == 0
