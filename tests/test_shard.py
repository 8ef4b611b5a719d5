"""N>1 host logic on CPU: world_size-2 gloo processes shard requests with no overlap,
agree on max-over-ranks timing and gather outputs in rank order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_00392_b200 import shard
    reqs = shard.shard_requests(9, world, rank)
    units = shard.unit_ids(reqs, layers=3, kv_heads=2)
    t = shard.max_over_ranks(1.0 + rank)
    out = torch.full((len(units), 2, 4), float(rank))
    allout = shard.gather_outputs(out)
    q.put((rank, reqs.tolist(), units.tolist(), t, allout.shape[0], allout[:, 0, 0].tolist()))
    dist.destroy_process_group()


def test_gloo_world2_sharding():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    res = sorted(q.get(timeout=120) for _ in range(world))
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    reqs = [r[1] for r in res]
    assert reqs[0] == [0, 1, 2, 3, 4] and reqs[1] == [5, 6, 7, 8]
    units = res[0][2] + res[1][2]
    assert sorted(units) == list(range(9 * 3 * 2))  # every unit exactly once
    assert all(r[3] == 2.0 for r in res)            # max over ranks
    for r in res:
        assert r[4] == len(units)
        assert r[5] == [0.0] * len(res[0][2]) + [1.0] * len(res[1][2])


def test_shard_balance():
    from paper_2503_00392_b200 import shard
    for n in range(1, 70):
        for w in (1, 2, 4, 8):
            parts = [shard.shard_requests(n, w, r) for r in range(w)]
            assert np.array_equal(np.concatenate(parts), np.arange(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1


def test_plan_units_kv_head_split():
    """requests < ranks: (request, kv head) pairs split across ranks, all layers of a pair on one rank."""
    from paper_2503_00392_b200 import shard
    for reqs, world in ((1, 8), (1, 2), (3, 8), (2, 4), (8, 8), (64, 8), (64, 2)):
        parts = [shard.plan_units(reqs, 4, 8, world, r) for r in range(world)]
        allu = np.concatenate(parts)
        assert np.array_equal(np.sort(allu), np.arange(reqs * 4 * 8))  # every unit exactly once
        for p in parts:
            kvh = set(((p // 8) // 4 * 8 + p % 8).tolist())  # (request, kv head) pairs of the rank
            assert len(p) == len(kvh) * 4                     # each owned pair with all 4 layers
    one = [shard.plan_units(1, 32, 8, 8, r) for r in range(8)]
    assert all(set((p % 8).tolist()) == {r} for r, p in enumerate(one))  # config 1 on 8 GPUs: one kv head each


def test_resident_layers():
    from paper_2503_00392_b200 import shard
    blk = 8192 + 1024
    assert shard.resident_layers(8, 32, 8, 8192, blk, 150 << 30) == 32
    l2 = shard.resident_layers(32, 32, 8, 8192, blk, 150 << 30)  # 64 requests on 2 GPUs
    assert 1 <= l2 < 32 and 32 * 8 * 8192 * blk * l2 <= 150 << 30
