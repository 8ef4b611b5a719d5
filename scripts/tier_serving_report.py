#!/usr/bin/env python3
"""Device-time report of the two-tier store and the serving loop.

1. Two-tier store at config-4 scale: a mixed-length batch (8 requests, 8K..128K context, ragged last
   blocks) over 4 layers with uneven attention budgets (planted blocks per 2048: 2 / 16 / 128 / isotropic),
   GQA 4, bf16, through `psattn_tier` with a fast tier holding 1/4 of the blocks (unified and
   layer-partitioned LRU), several decode steps; per step: device time (CUDA events around the batch,
   the installs of newly cached blocks included), bytes moved host->HBM, hits / misses — next to the
   same batch on the all-HBM pool.
2. Serving loop: the reference's serving scenarios (tests/golden/serving_cases.json, the reference's
   own workload through the compiled reference) — per method: device time of the per-layer batches
   per decode step and per batch, with the simulated TBT the reference reports.

usage: python scripts/tier_serving_report.py out.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2503_00392_b200 import batch, capi  # noqa: E402
from workload import synth  # noqa: E402


def tier_section(steps=4):
    d, T, g = 128, 16, 4
    ctxs = [8192 + 5, 24576 + 7, 40960 + 3, 57344 + 11, 73728 + 1, 90112 + 9, 106496 + 13, 131072]
    planted = [2 / 2048, 16 / 2048, 128 / 2048, 0.0]
    L = len(planted)
    blocks, layers, ntok, lists, K, V, qs = [], [], [], [], [], [], []
    base = 0
    for r, c in enumerate(ctxs):
        for l in range(L):
            uid = 5000 + 10 * r + l
            p = synth.params(seed=4, dim=d, block_tokens=T, skew=8.0, planted_prob=planted[l], round_bf16=1)
            k, v = synth.unit_host(p, uid, c)
            n = k.shape[0]
            blocks.extend(range(base, base + n))
            layers.extend([l] * n)
            ntok.extend(min(T, c - i * T) for i in range(n))
            K.append(k)
            V.append(v)
            lists.append(np.arange(base, base + n, dtype=np.int32))
            qs.append([synth.query(p, uid, h) for h in range(g)])
            base += n
    K, V = np.concatenate(K), np.concatenate(V)
    nb = base
    dev = torch.device("cuda")
    off = np.zeros(len(lists) + 1, np.int64)
    off[1:] = np.cumsum([x.size for x in lists])
    q = torch.tensor(np.asarray(qs, np.float32), device=dev)
    slots = torch.tensor(np.concatenate(lists), device=dev)
    offs = torch.tensor(off, device=dev)
    cfg = batch.BatchConfig(epsilon=0.95)

    def timed(run):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        run.run()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    out = dict(workload=dict(requests=len(ctxs), ctx=ctxs, layers=L, planted_per_2048=[x * 2048 for x in planted],
                             group=g, dim=d, block=T, kv_dtype="bf16", blocks=nb, kv_gib=nb * 2 * T * d * 2 / 2**30,
                             queries_per_step=len(lists) * g, eps=0.95))
    pool = batch.DevicePool(d, T, capi.PSATTN_KV_BF16, nb)
    pool.put_blocks(np.arange(nb, dtype=np.int32), ntok, K, V)
    run = batch.BatchRun(pool, q, slots, offs, int(max(x.size for x in lists)), cfg)
    timed(run)
    out["hbm_pool_ms_per_step"] = float(np.median([timed(run) for _ in range(steps)]))
    for policy, name in ((capi.PSATTN_POOL_UNIFIED, "unified"), (capi.PSATTN_POOL_LAYER_PARTITIONED, "partitioned")):
        tier = batch.DeviceTier(d, T, capi.PSATTN_KV_BF16, L, nb, nb // 4, policy, capi.PSATTN_EVICT_LRU)
        tier.put_blocks(np.array(blocks), np.array(layers), np.array(ntok), K, V)
        tr = batch.BatchRun(tier, q, slots, offs, int(max(x.size for x in lists)), cfg)
        rows = []
        for s in range(steps):
            h0, st0 = tier.h2d_bytes(), tier.stats()
            ms = timed(tr)
            st1 = tier.stats()
            rows.append(dict(step=s, device_ms=ms, h2d_bytes=tier.h2d_bytes() - h0, hits=st1["hits"] - st0["hits"],
                             misses=st1["misses"] - st0["misses"]))
        out[f"tier_{name}"] = dict(fast_slots=nb // 4, steps=rows)
        tier.close()
    return out


def serving_section():
    from oracle.pyoracle import RefDriver
    from test_gpu_serving import build
    ref = RefDriver()
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "serving_cases.json")))
    out = {}
    for name, case in cases.items():
        s = build(capi, ref, case)
        rows = []
        for row in case["rows"]:
            method = {"psa": capi.PSATTN_METHOD_PSA, "topk": capi.PSATTN_METHOD_TOPK,
                      "exact": capi.PSATTN_METHOD_EXACT}[row["method"]]
            t0 = time.perf_counter()
            got = s.run(method, epsilon=row["param"], k=int(row["param"]))
            wall = time.perf_counter() - t0
            rows.append(dict(method=row["method"], param=row["param"], gpu_ms=got["gpu_ms"],
                             device_batches=got["device_batches"], n_steps=got["n_steps"],
                             gpu_ms_per_step=got["gpu_ms"] / max(1, got["n_steps"]),
                             gpu_ms_per_batch=got["gpu_ms"] / max(1, got["device_batches"]),
                             wall_s=wall, sim_tbt_p50_ms=got["tbt_p50_ms"], hit_ratio=got["hit_ratio"],
                             kv_fraction=got["kv_fraction"], reference_tbt_p50_ms=row["tbt_p50_ms"]))
        out[name] = rows
    return out


def main():
    res = dict(device=torch.cuda.get_device_name(0), tier=tier_section(), serving=serving_section())
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    t = res["tier"]
    print("hbm pool ms/step", round(t["hbm_pool_ms_per_step"], 3))
    for k in ("tier_unified", "tier_partitioned"):
        print(k, [(round(r["device_ms"], 2), r["h2d_bytes"] >> 20, r["hits"], r["misses"]) for r in t[k]["steps"]])
    for name, rows in res["serving"].items():
        print(name, [(r["method"], r["param"], round(r["gpu_ms_per_step"], 3)) for r in rows])


if __name__ == "__main__":
    main()
