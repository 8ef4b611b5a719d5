"""Batched serving loop on the GPU path (psattn_serving) against the reference's
own serving reports (proj/out/{smoke,serving_rho0,serving_rho95}.csv, frozen in
tests/golden/serving_cases.json), on the reference's own workload (generate_workload through the
compiled reference): every report row — blocks per call, KV fraction, coverage, store hit ratio,
simulated TBT percentiles and overlap efficiency — for exact, PSA and top-k methods."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
HERE = os.path.dirname(os.path.abspath(__file__))
EST = {"mean": 0, "cuboid_upper": 1, "cuboid_mean": 2}


def build(capi, ref, case):
    wl = ref.workload(**case["workload"])
    sp = wl.spec
    st, eng, srv = case["store"], case["engine"], case["serving"]
    store = capi.TierDesc(sp["dim"], sp["block_size"], capi.PSATTN_KV_F32, sp["n_layers"], 0, st["capacity"],
                          0 if st["policy"] == "unified" else 1, 0 if st["eviction"] == "lru" else 1)
    cfg = capi.config_default(epsilon=eng["epsilon"], microbatch_size=eng["microbatch"],
                              estimator=EST[eng["estimator"]], ranking_mode=1 if eng["ranking"] == "oracle" else 0,
                              audit_coverage=1 if eng["audit"] else 0)
    cost = capi.ServingCost(srv["miss_cost_ms"], srv["hit_cost_ms"], srv["compute_cost_ms"], 1 if srv["overlap"] else 0, 0)
    s = capi.Serving(store, cfg, cost)
    for r in wl.requests:
        s.add_request(r["request_id"], 0.0, r["steps"], np.array(r["lists"]), r["ids"], r["layers"], r["ntok"],
                      r["keys"], r["values"], r["queries"])
    return s


@pytest.mark.parametrize("name", ["smoke", "serving_rho0", "serving_rho95"])
def test_serving_reproduces_reference_report(ref, name):
    from paper_2503_00392_b200 import capi
    case = json.load(open(os.path.join(HERE, "golden", "serving_cases.json")))[name]
    s = build(capi, ref, case)
    for row in case["rows"]:
        method = {"psa": capi.PSATTN_METHOD_PSA, "topk": capi.PSATTN_METHOD_TOPK,
                  "exact": capi.PSATTN_METHOD_EXACT}[row["method"]]
        got = s.run(method, epsilon=row["param"], k=int(row["param"]))
        tag = (name, row["method"], row["param"])
        for k in ("mean_blocks", "p99_blocks", "kv_fraction", "hit_ratio", "tbt_p50_ms", "tbt_p99_ms", "overlap_eff"):
            assert got[k] == pytest.approx(row[k], rel=1e-12, abs=1e-12), (tag, k, got[k], row[k])
        # coverage: fp64 oracle masses under audit (smoke), fp32 block masses otherwise (summation order)
        for k in ("mean_coverage", "min_coverage"):
            assert got[k] == pytest.approx(row[k], rel=1e-5), (tag, k, got[k], row[k])
        assert got["gpu_ms"] > 0 and got["device_batches"] > 0
