"""Device-batched path (psattn_run_batch) against the oracle: random GQA batches,
ragged blocks, every estimator / ranking mode / top-k / microbatch size, bf16
pools filled by the device generator, metadata bit-exactness, the GQA union
counter, and GQA == per-head equivalence."""
import math

import numpy as np
import pytest

from helpers import check_parity, random_blockset
from oracle.pyoracle import BlockSet, make_config
from workload import synth  # fixture: the seekable synthetic generator

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def mods():
    from paper_2503_00392_b200 import batch, capi
    return capi, batch


def run_units(mods, units, queries, T, kv_dtype=0, want_iter=True, **cfg):
    """units: list of BlockSet (ids ascending 0..n-1); queries: [U][g][d]."""
    capi, batch = mods
    d = units[0].d
    total = sum(u.n for u in units)
    pool = batch.DevicePool(d, T, kv_dtype, total)
    slots, ntok, ks, vs = [], [], [], []
    s = 0
    for u in units:
        for i in range(u.n):
            k, v = u.block(i)
            kk = np.zeros((T, d), np.float32)
            vv = np.zeros((T, d), np.float32)
            kk[: k.shape[0]] = k
            vv[: v.shape[0]] = v
            ks.append(kk)
            vs.append(vv)
            ntok.append(k.shape[0])
            slots.append(s)
            s += 1
    pool.put_blocks(slots, ntok, np.stack(ks), np.stack(vs))
    off = np.zeros(len(units) + 1, np.int64)
    off[1:] = np.cumsum([u.n for u in units])
    dev = torch.device("cuda")
    q = torch.tensor(np.asarray(queries, np.float32), device=dev)
    run = batch.BatchRun(pool, q, torch.tensor(np.array(slots, np.int32), device=dev),
                         torch.tensor(off, device=dev), max(u.n for u in units), batch.BatchConfig(**cfg),
                         want_ranked=True, want_iter=want_iter)
    run.run()
    torch.cuda.synchronize()
    return pool, run, off


def unpack(run, off, u, h, n):
    g = run.group
    qi = u * g + h
    hb = int(off[u]) * g + h * n
    ranked = run.ranked[hb: hb + n].cpu().numpy()
    bp = int(run.bp[qi])
    return dict(out=run.out[u, h].cpu().numpy(), bp=bp, est=float(run.est[qi]), term=int(run.term[qi]),
                tcov=float(run.tcov[qi]), ids=ranked[:bp], ranked=ranked)


CFGS = [dict(epsilon=0.95), dict(epsilon=0.8, microbatch_size=4), dict(epsilon=0.99, estimator=0),
        dict(epsilon=0.9, estimator=1, microbatch_size=3), dict(epsilon=1.0), dict(topk=7),
        dict(topk=64, microbatch_size=5), dict(epsilon=0.9, ranking_mode=1),
        dict(epsilon=0.95, audit_coverage=1, microbatch_size=2), dict(epsilon=0.5)]


@pytest.mark.parametrize("ci", range(len(CFGS)))
@pytest.mark.parametrize("d,T,g", [(128, 16, 4), (64, 16, 2), (32, 8, 1), (128, 32, 8), (20, 5, 3)])
def test_batch_parity(mods, oracle, ci, d, T, g):
    cfgd = CFGS[ci]
    rng = np.random.default_rng(ci * 1000 + d * 7 + T + g)
    U = 3
    units, queries = [], []
    for u in range(U):
        n = int(rng.integers(1, 150))
        units.append(random_blockset(rng, n, d, 1, T, planted_frac=0.1 if u % 2 else 0.0))
        base = rng.standard_normal(d)
        queries.append([(base + 0.3 * rng.standard_normal(d)).astype(np.float32) * 2 for _ in range(g)])
    pool, run, off = run_units(mods, units, queries, T, **cfgd)
    topk = cfgd.get("topk", 0)
    ocfg = make_config(**{k: v for k, v in cfgd.items() if k != "topk"})
    tags = []
    for u in range(U):
        for h in range(g):
            r = unpack(run, off, u, h, units[u].n)
            tags.append(check_parity(oracle, np.asarray(queries[u][h]), units[u], ocfg, topk, r["ids"], r["bp"],
                                     r["out"], r["est"]))
            o = oracle.psa(np.asarray(queries[u][h]), units[u], ocfg, topk)
            if tags[-1] == "exact":
                assert r["term"] == int(o.terminated_early)
                if ocfg.audit_coverage:
                    assert r["tcov"] == pytest.approx(o.true_coverage, abs=1e-9)
                # iteration estimates at every microbatch boundary
                m = ocfg.microbatch_size
                it = run.iest[int(off[u]) * g + h * units[u].n:].cpu().numpy()
                bounds, cur = [], 0
                while cur < r["bp"]:
                    c = min(units[u].n - cur, m)
                    if topk:
                        c = min(c, min(topk, units[u].n) - cur)
                    cur += c
                    bounds.append(cur - 1)
                np.testing.assert_allclose(it[bounds], o.iteration_estimates, rtol=0, atol=1e-4)
    assert tags.count("exact") >= len(tags) - 1


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("d,g", [(128, 4), (64, 2), (128, 3)])
def test_gqa_equals_per_head(mods, d, g, mode):
    """psa_attention_multi_head semantics (engine.cpp:240-260): a GQA launch (per-head or
    GQA-group kernel) equals g independent g=1 runs: same ranks, same stop points (identical
    fp32 block masses), outputs equal up to summation order."""
    capi, _ = mods
    rng = np.random.default_rng(31337 + d + g)
    T = 16
    unit = random_blockset(rng, 300, d, 1, 16, planted_frac=0.05)
    base = rng.standard_normal(d)
    qs = [((base + 0.5 * rng.standard_normal(d)) * 2).astype(np.float32) for _ in range(g)]
    assert capi.lib.psattn_set_progressive_kernel(mode) == 0
    try:
        _, rg, offg = run_units(mods, [unit], [qs], T, epsilon=0.9)
        _, r1, off1 = run_units(mods, [unit] * g, [[q] for q in qs], T, epsilon=0.9)
    finally:
        capi.lib.psattn_set_progressive_kernel(0)
    for h in range(g):
        a = unpack(rg, offg, 0, h, unit.n)
        b = unpack(r1, off1, h, 0, unit.n)
        assert a["bp"] == b["bp"]
        assert np.array_equal(a["ids"], b["ids"])
        assert a["est"] == b["est"]
        assert np.max(np.abs(a["out"] - b["out"])) <= 1e-5


@pytest.mark.parametrize("ci", [0, 1, 5, 6, 7, 8])
def test_per_head_kernel_parity(mods, oracle, ci):
    """The per-q-head progressive kernel (forced) on the GQA shapes, against the oracle."""
    capi, _ = mods
    capi.lib.psattn_set_progressive_kernel(1)
    try:
        test_batch_parity(mods, oracle, ci, 128, 16, 4)
    finally:
        capi.lib.psattn_set_progressive_kernel(0)


def test_union_counter(mods):
    rng = np.random.default_rng(5)
    d, T = 64, 16
    units = [random_blockset(rng, int(rng.integers(50, 300)), d, 16, 16, planted_frac=0.05) for _ in range(3)]
    qs = [[rng.standard_normal(d).astype(np.float32) * 2 for _ in range(4)] for _ in units]
    _, run, off = run_units(mods, units, qs, T, epsilon=0.9)
    un = run.union_blocks().cpu().numpy()
    torch.cuda.synchronize()
    for u, unit in enumerate(units):
        s = set()
        for h in range(4):
            s |= set(map(int, unpack(run, off, u, h, unit.n)["ids"]))
        assert un[u] == len(s)


def test_metadata_bit_exact(mods, oracle):
    """K1: device metadata == reference build_metadata (metadata.cpp:8-34), bit for bit."""
    rng = np.random.default_rng(8)
    for d, T in ((128, 16), (20, 7), (64, 32)):
        bs = random_blockset(rng, 50, d, 1, T)
        pool, _, _ = run_units(mods, [bs], [[np.ones(d, np.float32)]], T, epsilon=1.0)
        for i in range(bs.n):
            k, _ = bs.block(i)
            m, lo, hi = pool.read_metadata(i)
            om, olo, ohi = oracle.build_metadata(k)
            assert m.tobytes() == om.tobytes() and lo.tobytes() == olo.tobytes() and hi.tobytes() == ohi.tobytes()


def test_bf16_pool_synthetic_parity(mods, oracle):
    """bf16 pool filled on device by the seekable generator; the oracle gets the same
    values regenerated on the host (bf16-rounded, upcast to fp32)."""
    capi, batch = mods
    d, T, g = 128, 16, 4
    for planted in (0.0, 64 / 2048):
        p = synth.params(seed=1, dim=d, block_tokens=T, skew=8.0, planted_prob=planted, round_bf16=1)
        tokens = [16 * 700 + 5, 16 * 300]
        nb = [(t + T - 1) // T for t in tokens]
        slot_off = [0, nb[0]]
        pool = batch.DevicePool(d, T, capi.PSATTN_KV_BF16, sum(nb))
        synth.fill(pool, p, [11, 12], slot_off, tokens)
        torch.cuda.synchronize()
        dev = torch.device("cuda")
        qs = [[synth.query(p, uid, h) for h in range(g)] for uid in (11, 12)]
        slots = np.arange(sum(nb), dtype=np.int32)
        off = np.array([0, nb[0], nb[0] + nb[1]], np.int64)
        run = batch.BatchRun(pool, torch.tensor(np.array(qs), device=dev), torch.tensor(slots, device=dev),
                             torch.tensor(off, device=dev), max(nb), batch.BatchConfig(epsilon=0.95),
                             want_ranked=True)
        run.run()
        torch.cuda.synchronize()
        for u, uid in enumerate((11, 12)):
            k, v = synth.unit_host(p, uid, tokens[u])
            ntok = [min(T, tokens[u] - b * T) for b in range(nb[u])]
            bs = BlockSet([k[b, :ntok[b]] for b in range(nb[u])], [v[b, :ntok[b]] for b in range(nb[u])])
            # metadata of the device pool equals the oracle's on the same values
            mm, lo, hi = pool.read_metadata(slot_off[u] + 3)
            om, olo, ohi = oracle.build_metadata(k[3, :ntok[3]])
            assert mm.tobytes() == om.tobytes() and lo.tobytes() == olo.tobytes()
            for h in range(g):
                r = unpack(run, off, u, h, nb[u])
                check_parity(oracle, qs[u][h], bs, make_config(epsilon=0.95), 0, r["ids"], r["bp"], r["out"],
                             r["est"])


def test_synthetic_device_equals_host(mods):
    """The device fill kernel and the host generator produce identical bits."""
    capi, batch = mods
    d, T = 128, 16
    for prob, rb, dt in ((0.1, 1, capi.PSATTN_KV_BF16), (0.05, 0, capi.PSATTN_KV_F32)):
        p = synth.params(seed=7, dim=d, block_tokens=T, skew=8.0, planted_prob=prob, round_bf16=rb)
        tokens = [16 * 40 + 3]
        pool = batch.DevicePool(d, T, dt, 41)
        synth.fill(pool, p, [5], [0], tokens)
        torch.cuda.synchronize()
        lay = pool.layout()
        raw_np = read_device(lay.kv, 41 * lay.slot_bytes)
        k, v = synth.unit_host(p, 5, tokens[0])
        per = T * d
        if dt == capi.PSATTN_KV_BF16:
            words = np.frombuffer(raw_np, np.uint16).reshape(41, 2, per)
            dk = (words[:, 0].astype(np.uint32) << 16).view(np.float32)
            dv = (words[:, 1].astype(np.uint32) << 16).view(np.float32)
        else:
            f = np.frombuffer(raw_np, np.float32).reshape(41, 2, per)
            dk, dv = f[:, 0], f[:, 1]
        assert dk.reshape(-1).tobytes() == k.reshape(-1).tobytes()
        assert dv.reshape(-1).tobytes() == v.reshape(-1).tobytes()


class _DevBytes:
    """Wraps a raw device pointer for torch.as_tensor (CUDA array interface)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = dict(shape=(nbytes,), typestr="|u1", data=(int(ptr), False), version=3)


def read_device(ptr, nbytes) -> bytes:
    t = torch.as_tensor(_DevBytes(ptr, nbytes), device="cuda")
    return t.cpu().numpy().tobytes()


def test_c1_shape_full_parity(mods, oracle, ref):
    """BASELINE config 1 (fp32 KV, 32K ctx, 32 q / 8 kv heads, B=16, eps=0.95): every head vs
    the COMPILED REFERENCE's psa_attention_multi_head on the same synthetic inputs (2 kv heads)."""
    capi, batch = mods
    d, T, g, n = 128, 16, 4, 2048
    for planted in (0.0, 64 / 2048):
        p = synth.params(seed=1, dim=d, block_tokens=T, skew=8.0, planted_prob=planted, round_bf16=0)
        units = [0, 5]
        pool = batch.DevicePool(d, T, capi.PSATTN_KV_F32, n * len(units))
        synth.fill(pool, p, units, [0, n], [n * T] * len(units))
        torch.cuda.synchronize()
        qs = [[synth.query(p, uid, h) for h in range(g)] for uid in units]
        dev = torch.device("cuda")
        off = np.array([0, n, 2 * n], np.int64)
        run = batch.BatchRun(pool, torch.tensor(np.array(qs), device=dev),
                             torch.tensor(np.arange(2 * n, dtype=np.int32), device=dev),
                             torch.tensor(off, device=dev), n, batch.BatchConfig(epsilon=0.95), want_ranked=True)
        run.run()
        torch.cuda.synchronize()
        st = ref.store(capacity=0)
        kv_ids = []
        for u, uid in enumerate(units):
            k, v = synth.unit_host(p, uid, n * T)
            for b in range(n):
                st.put(u * n + b, k[b], v[b])
            kv_ids.append(np.arange(u * n, (u + 1) * n))
        allq = np.array([q for qq in qs for q in qq], np.float32)
        res, union = st.multi_head(allq, np.array(kv_ids), make_config(epsilon=0.95))
        exact = 0
        for u in range(len(units)):
            k, v = synth.unit_host(p, units[u], n * T)
            bs = BlockSet(list(k), list(v))
            for h in range(g):
                r = unpack(run, off, u, h, n)
                o = res[u * g + h]
                gpu_ids = r["ids"]
                if r["bp"] == o.blocks_processed and np.array_equal(gpu_ids + u * n, o.processed_ids):
                    exact += 1
                    assert np.max(np.abs(r["out"] - o.output)) <= 1e-3
                else:
                    check_parity(oracle, qs[u][h], bs, make_config(epsilon=0.95), 0, gpu_ids, r["bp"], r["out"],
                                 r["est"])
        assert exact >= len(units) * g - 1


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("subs", [2, 5])
def test_pipelined_launch_identical(mods, subs, kernel):
    """Score/progressive overlap over sub-batches (psattn_set_pipeline) gives bit-identical
    results, for both progressive kernels (the GQA kernel numbers its union deterministically)."""
    capi, _ = mods
    capi.lib.psattn_set_progressive_kernel(kernel)
    rng = np.random.default_rng(77 + subs)
    d, T, g = 128, 16, 4
    units = [random_blockset(rng, int(rng.integers(20, 200)), d, 1, 16, planted_frac=0.05) for _ in range(11)]
    qs = [[rng.standard_normal(d).astype(np.float32) * 2 for _ in range(g)] for _ in units]
    res = {}
    for mode in (1, subs):
        assert capi.lib.psattn_set_pipeline(mode) == 0
        try:
            _, run, off = run_units(mods, units, qs, T, epsilon=0.9)
        finally:
            capi.lib.psattn_set_pipeline(0)
        res[mode] = (run.out.cpu().numpy(), run.bp.cpu().numpy(), run.est.cpu().numpy())
    capi.lib.psattn_set_progressive_kernel(0)
    for a, b in zip(res[1], res[subs]):
        assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("kv_dtype", [0, 1])
def test_long_lists_multi_tranche(mods, oracle, kernel, kv_dtype):
    """Lists longer than one ordering tranche (GQA: 512, per-head: 1024 ranks) with eps near 1,
    so heads consume several tranches (bucket-select refinement + histogram paths)."""
    capi, _ = mods
    rng = np.random.default_rng(99 + kernel + 10 * kv_dtype)
    d, T, g, n = 128, 16, 4, 2600
    units = [random_blockset(rng, n, d, 16, 16) for _ in range(2)]
    if kv_dtype == 1:
        for u in units:
            u.keys[:] = torch.tensor(u.keys).bfloat16().float().numpy()
            u.values[:] = torch.tensor(u.values).bfloat16().float().numpy()
    qs = [[(rng.standard_normal(d) * 0.3).astype(np.float32) for _ in range(g)] for _ in units]
    capi.lib.psattn_set_progressive_kernel(kernel)
    try:
        _, run, off = run_units(mods, units, qs, T, kv_dtype=kv_dtype, epsilon=0.99)
    finally:
        capi.lib.psattn_set_progressive_kernel(0)
    for u in range(2):
        for h in range(g):
            r = unpack(run, off, u, h, n)
            assert r["bp"] > 1100  # several tranches consumed
            check_parity(oracle, qs[u][h], units[u], make_config(epsilon=0.99), 0, r["ids"], r["bp"], r["out"], r["est"])


@pytest.mark.parametrize("planted", [1 / 32, 0.0])
def test_graph_replay_identical(mods, planted):
    """A decode step captured as a CUDA graph (psattn_graph_*) replays bit-identically to the
    direct launch, including after the queries are refreshed in place (the serving pattern);
    planted = 0 exercises the dense hand-over inside the graph."""
    capi, batch = mods
    d, T, g = 128, 16, 4
    p = synth.params(seed=3, dim=d, block_tokens=T, skew=8.0, planted_prob=planted, round_bf16=1)
    units, n = [21, 22, 23], 1200
    pool = batch.DevicePool(d, T, capi.PSATTN_KV_BF16, n * len(units))
    synth.fill(pool, p, units, np.arange(len(units)) * n, [n * T] * len(units))
    dev = torch.device("cuda")
    q0 = torch.tensor(np.array([[synth.query(p, u, h) for h in range(g)] for u in units], np.float32), device=dev)
    q1 = torch.tensor(np.array([[synth.query(p, u + 100, h) for h in range(g)] for u in units], np.float32),
                      device=dev)
    slots = torch.arange(n * len(units), dtype=torch.int32, device=dev)
    off = torch.arange(len(units) + 1, dtype=torch.int64, device=dev) * n
    run = batch.BatchRun(pool, q0.clone(), slots, off, n, batch.BatchConfig(epsilon=0.95), want_ranked=True)
    stream = torch.cuda.Stream()
    run.capture(stream)
    for q in (q0, q1, q0):
        run.q.copy_(q)
        run.run()
        torch.cuda.synchronize()
        ref = (run.out.clone(), run.bp.clone(), run.est.clone())
        run.out.zero_()
        run.bp.zero_()
        assert run.run_graph() == run.run()
        torch.cuda.synchronize()
        run.out.zero_()
        run.run_graph()
        torch.cuda.synchronize()
        assert torch.equal(run.out, ref[0]) and torch.equal(run.bp, ref[1]) and torch.equal(run.est, ref[2])


@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("T", [8, 12, 16])
@pytest.mark.parametrize("g", [4, 2])
@pytest.mark.parametrize("planted", [0.08, 0.0])
def test_bf16_short_blocks_tensor_core_path(mods, oracle, d, T, g, planted):
    """bf16 pools with blocks of fewer than 16 tokens and ragged blocks on the GQA paths: d = 128
    is the tensor-core path (rows past T clamp to the last row and are masked) through 64-rank
    rounds and — with isotropic keys — the dense hand-over; d = 64 the FFMA GQA path with
    32-rank rounds and later tranches. Every head against the oracle."""
    rng = np.random.default_rng(int(T * 10 + g + planted * 100 + d))
    n = 900
    units = [random_blockset(rng, n, d, 1, T, planted_frac=planted, skew=2.5) for _ in range(2)]
    for u in units:
        u.keys[:] = torch.tensor(u.keys).bfloat16().float().numpy()
        u.values[:] = torch.tensor(u.values).bfloat16().float().numpy()
    qs = [[(rng.standard_normal(d) * 0.5 + 0.5).astype(np.float32) for _ in range(g)] for _ in units]
    _, run, off = run_units(mods, units, qs, T, kv_dtype=1, epsilon=0.95)
    for u in range(2):
        for h in range(g):
            r = unpack(run, off, u, h, n)
            check_parity(oracle, qs[u][h], units[u], make_config(epsilon=0.95), 0, r["ids"], r["bp"], r["out"], r["est"])


@pytest.mark.parametrize("kv_dtype", [0, 1])
@pytest.mark.parametrize("cfg", [dict(epsilon=0.95), dict(epsilon=1.0), dict(topk=5), dict(epsilon=0.9, microbatch_size=7)])
def test_tiny_and_ragged_lists(mods, oracle, kv_dtype, cfg):
    """Edge shapes on every path: lists of 1, 2 and 3 blocks, single-token blocks, top-k larger than
    the list, microbatch larger than the list, GQA 4 at d = 128 (tensor-core path for bf16)."""
    rng = np.random.default_rng(17 + kv_dtype)
    d, T, g = 128, 16, 4
    units = [random_blockset(rng, n, d, 1, T) for n in (1, 2, 3, 40)]
    units.append(random_blockset(rng, 5, d, 1, 1))  # single-token blocks
    if kv_dtype == 1:
        for u in units:
            u.keys[:] = torch.tensor(u.keys).bfloat16().float().numpy()
            u.values[:] = torch.tensor(u.values).bfloat16().float().numpy()
    qs = [[rng.standard_normal(d).astype(np.float32) for _ in range(g)] for _ in units]
    _, run, off = run_units(mods, units, qs, T, kv_dtype=kv_dtype, **cfg)
    oc = make_config(epsilon=cfg.get("epsilon", 1.0) if not cfg.get("topk") else 1.0,
                     microbatch_size=cfg.get("microbatch_size", 1))
    for u, bs in enumerate(units):
        for h in range(g):
            r = unpack(run, off, u, h, bs.n)
            check_parity(oracle, qs[u][h], bs, oc, cfg.get("topk", 0), r["ids"], r["bp"], r["out"], r["est"])
            if cfg.get("topk"):
                assert r["bp"] == min(cfg["topk"], bs.n)
