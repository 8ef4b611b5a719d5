"""GPU oracle/audit tooling and BASELINE config 3:

* psattn_tradeoff reproduces the reference's own tradeoff reports
  (proj/out/tradeoff_*.tradeoff.json, frozen in tests/golden/tradeoff_cases.json) on the
  reference's own workload (generate_workload through the compiled reference);
* psattn_exact_attention (fp64 exact attention, reference attention.cpp:36-63) equals the oracle;
* config 3: threshold sweep eps in {0.8, 0.9, 0.95, 0.99} vs fixed top-k in {64, 128} at 64K
  context (Llama GQA shape, bf16 pool), blocks read and output error against fp64 exact attention,
  with per-head parity against the C oracle.
"""
import json
import math
import os

import numpy as np
import pytest

from helpers import check_parity
from oracle.pyoracle import BlockSet, make_config
from workload import synth  # fixture: the seekable synthetic generator

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
HERE = os.path.dirname(os.path.abspath(__file__))
EST = {"mean": 0, "cuboid_upper": 1, "cuboid_mean": 2}


@pytest.fixture(scope="module")
def mods():
    from paper_2503_00392_b200 import batch, capi
    return capi, batch


def workload_batch(mods, wl, cfg):
    """Every (request, step, layer) query of a reference workload as a group-1 unit over its
    layer's block list; all blocks in one fp32 device pool."""
    capi, batch = mods
    d, B = wl.spec["dim"], wl.spec["block_size"]
    total = sum(len(r["ids"]) for r in wl.requests)
    pool = batch.DevicePool(d, B, capi.PSATTN_KV_F32, total)
    slot_of, s = {}, 0
    for r in wl.requests:
        n = len(r["ids"])
        pool.put_blocks(np.arange(s, s + n, dtype=np.int32), r["ntok"], r["keys"], r["values"])
        for i, bid in enumerate(r["ids"]):
            slot_of[int(bid)] = s + i
        s += n
    qs, lists = [], []
    for r in wl.requests:
        for t in range(r["steps"]):
            for l, lst in enumerate(r["lists"]):
                qs.append(r["queries"][t, l][None, :])
                lists.append(np.array([slot_of[int(b)] for b in lst], np.int32))
    off = np.zeros(len(lists) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in lists])
    dev = torch.device("cuda")
    run = batch.BatchRun(pool, torch.tensor(np.array(qs, np.float32), device=dev),
                         torch.tensor(np.concatenate(lists), device=dev), torch.tensor(off, device=dev),
                         max(len(x) for x in lists), batch.BatchConfig(**cfg))
    return pool, run


@pytest.mark.parametrize("name", ["tradeoff_bimodal", "tradeoff_uniform"])
def test_tradeoff_reproduces_reference_report(mods, ref, name):
    case = json.load(open(os.path.join(HERE, "golden", "tradeoff_cases.json")))[name]
    wl = ref.workload(**case["workload"])
    eng = case["engine"]
    cfg = dict(microbatch_size=eng["microbatch"], estimator=EST[eng["estimator"]],
               ranking_mode=1 if eng["ranking"] == "oracle" else 0, audit_coverage=1)
    _, run = workload_batch(mods, wl, cfg)
    got = run.tradeoff(case["target"])
    want = case["report"]
    for k in ("n_queries", "max_blocks", "k_min"):
        assert got[k] == want[k], (k, got[k], want[k])
    for k in ("psa_mean_blocks", "psa_p99_blocks", "block_access_ratio"):
        assert got[k] == pytest.approx(want[k], rel=1e-12), k
    for k in ("worst_coverage_at_kmin", "worst_coverage_below_kmin", "psa_mean_coverage"):
        assert got[k] == pytest.approx(want[k], rel=1e-9, abs=1e-12), (k, got[k], want[k])


def test_exact_attention_matches_oracle(mods, oracle):
    capi, batch = mods
    rng = np.random.default_rng(3)
    for d, T, dt in ((64, 16, capi.PSATTN_KV_F32), (128, 16, capi.PSATTN_KV_BF16), (20, 5, capi.PSATTN_KV_F32)):
        n = 37
        ntok = rng.integers(1, T + 1, n).astype(np.int32)
        k = np.zeros((n, T, d), np.float32)
        v = np.zeros((n, T, d), np.float32)
        for i in range(n):
            k[i, :ntok[i]] = rng.standard_normal((ntok[i], d))
            v[i, :ntok[i]] = rng.standard_normal((ntok[i], d))
        if dt == capi.PSATTN_KV_BF16:  # the oracle sees the values the bf16 pool stores
            k = torch.tensor(k).bfloat16().float().numpy()
            v = torch.tensor(v).bfloat16().float().numpy()
        pool = batch.DevicePool(d, T, dt, n)
        pool.put_blocks(np.arange(n, dtype=np.int32), ntok, k, v)
        q = rng.standard_normal((1, 2, d)).astype(np.float32)
        dev = torch.device("cuda")
        run = batch.BatchRun(pool, torch.tensor(q, device=dev), torch.arange(n, dtype=torch.int32, device=dev),
                             torch.tensor([0, n], dtype=torch.int64, device=dev), n, batch.BatchConfig())
        out = run.exact_attention().cpu().numpy()
        bs = BlockSet([k[i, :ntok[i]] for i in range(n)], [v[i, :ntok[i]] for i in range(n)])
        for h in range(2):
            want = oracle.exact_attention_blocks(q[0, h], bs, np.arange(n), 1.0 / math.sqrt(d))
            assert np.max(np.abs(out[0, h] - want)) <= 1e-12


def config3_sweep(mods, n_kv_units=2, ctx=65536, seed=1, planted=1 / 32):
    """BASELINE config 3: 64K context, Llama GQA group 4, d=128, B=16, bf16 pool, planted keys.
    Returns {setting: dict(blocks_read, kv_fraction, max_err, mean_err)} and the raw runs."""
    capi, batch = mods
    d, T, g = 128, 16, 4
    n = ctx // T
    p = synth.params(seed=seed, dim=d, block_tokens=T, skew=8.0, planted_prob=planted, round_bf16=1)
    units = list(range(100, 100 + n_kv_units))
    pool = batch.DevicePool(d, T, capi.PSATTN_KV_BF16, n * len(units))
    synth.fill(pool, p, units, np.arange(len(units)) * n, [ctx] * len(units))
    dev = torch.device("cuda")
    qs = torch.tensor(np.array([[synth.query(p, u, h) for h in range(g)] for u in units], np.float32),
                      device=dev)
    slots = torch.arange(n * len(units), dtype=torch.int32, device=dev)
    off = torch.arange(len(units) + 1, dtype=torch.int64, device=dev) * n
    exact = batch.BatchRun(pool, qs, slots, off, n, batch.BatchConfig()).exact_attention().cpu().numpy()
    settings = [("eps", e) for e in (0.8, 0.9, 0.95, 0.99)] + [("topk", k) for k in (64, 128)]
    rows, runs = {}, {}
    for kind, val in settings:
        cfg = batch.BatchConfig(epsilon=val) if kind == "eps" else batch.BatchConfig(topk=val)
        run = batch.BatchRun(pool, qs, slots, off, n, cfg, want_ranked=True)
        run.run()
        torch.cuda.synchronize()
        out = run.out.cpu().numpy()
        bp = run.bp.cpu().numpy()
        union = run.union_blocks().cpu().numpy()
        err = np.max(np.abs(out - exact), axis=2)
        rows[f"{kind}={val}"] = dict(mean_blocks_per_head=float(bp.mean()), max_blocks_per_head=int(bp.max()),
                                    kv_fraction_read=float(union.sum() / (n * len(units))),
                                    max_abs_err=float(err.max()), mean_abs_err=float(err.mean()))
        runs[(kind, val)] = (run, cfg)
    return rows, runs, (p, units, n, qs.cpu().numpy())


def test_config3_threshold_vs_topk(mods, oracle):
    rows, runs, (p, units, n, qs) = config3_sweep(mods)
    capi, _ = mods
    eps_rows = [rows[f"eps={e}"] for e in (0.8, 0.9, 0.95, 0.99)]
    # more coverage -> more blocks read, smaller error
    assert all(a["mean_blocks_per_head"] <= b["mean_blocks_per_head"] for a, b in zip(eps_rows, eps_rows[1:]))
    assert eps_rows[-1]["max_abs_err"] <= eps_rows[0]["max_abs_err"]
    assert rows["topk=64"]["max_blocks_per_head"] == 64 and rows["topk=128"]["max_blocks_per_head"] == 128
    # PSA reads a fraction of the KV
    assert eps_rows[2]["kv_fraction_read"] < 0.5
    # parity of every head of the first kv-head unit against the C oracle, for every setting
    k, v = synth.unit_host(p, units[0], n * 16)
    bs = BlockSet(list(k), list(v))
    for (kind, val), (run, cfg) in runs.items():
        oc = make_config(epsilon=val if kind == "eps" else 1.0)
        topk = val if kind == "topk" else 0
        for h in range(4):
            bp = int(run.bp[h])
            ids = run.ranked[h * n: h * n + bp].cpu().numpy()
            check_parity(oracle, qs[0, h], bs, oc, topk, ids, bp, run.out[0, h].cpu().numpy(), None)
