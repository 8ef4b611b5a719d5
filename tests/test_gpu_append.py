"""Decode-step KV append + metadata maintenance: tokens appended one
at a time into tail slots on the device; after every append the slot's metadata equals
the reference's build_metadata over the rows so far (bit for bit), full slots are
refused, and a progressive query over a list ending in the growing tail block matches
the oracle."""
import numpy as np
import pytest

from helpers import check_parity
from oracle.pyoracle import BlockSet, make_config

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("kv_dtype", [0, 1])
def test_append_tokens_metadata_and_query(oracle, kv_dtype):
    from paper_2503_00392_b200 import batch, capi
    rng = np.random.default_rng(21 + kv_dtype)
    d, T, nseq, prefix = 128, 16, 3, 40
    pool = batch.DevicePool(d, T, kv_dtype, nseq * (prefix + 1))
    dev = torch.device("cuda")
    rnd = (lambda a: a) if kv_dtype == 0 else (lambda a: np.asarray(torch.tensor(a).bfloat16().float()))
    # full prefix blocks via put_blocks, tail slots start empty
    keys = rnd(rng.standard_normal((nseq, prefix, T, d)).astype(np.float32))
    vals = rnd(rng.standard_normal((nseq, prefix, T, d)).astype(np.float32))
    slots = np.arange(nseq * (prefix + 1), dtype=np.int32).reshape(nseq, prefix + 1)
    pool.put_blocks(slots[:, :prefix].reshape(-1), np.full(nseq * prefix, T, np.int32),
                    keys.reshape(-1, T, d), vals.reshape(-1, T, d))
    tail = torch.tensor(slots[:, prefix].copy(), device=dev)
    tk = np.zeros((nseq, T, d), np.float32)
    tv = np.zeros((nseq, T, d), np.float32)
    for t in range(T):
        k = rnd(rng.standard_normal((nseq, d)).astype(np.float32))
        v = rnd(rng.standard_normal((nseq, d)).astype(np.float32))
        tk[:, t], tv[:, t] = k, v
        assert pool.append_tokens(tail, torch.tensor(k, device=dev), torch.tensor(v, device=dev)) == 0
        for s in range(nseq):
            m, lo, hi = pool.read_metadata(int(slots[s, prefix]))
            om, olo, ohi = oracle.build_metadata(tk[s, : t + 1])
            assert m.tobytes() == om.tobytes() and lo.tobytes() == olo.tobytes() and hi.tobytes() == ohi.tobytes()
        if t in (0, 6, T - 1):
            q = (rng.standard_normal((nseq, 1, d)) * 2).astype(np.float32)
            off = np.arange(nseq + 1, dtype=np.int64) * (prefix + 1)
            run = batch.BatchRun(pool, torch.tensor(q, device=dev), torch.tensor(slots.reshape(-1), device=dev),
                                 torch.tensor(off, device=dev), prefix + 1, batch.BatchConfig(epsilon=0.95),
                                 want_ranked=True)
            run.run()
            torch.cuda.synchronize()
            for s in range(nseq):
                blocks_k = [keys[s, b] for b in range(prefix)] + [tk[s, : t + 1]]
                blocks_v = [vals[s, b] for b in range(prefix)] + [tv[s, : t + 1]]
                bs = BlockSet(blocks_k, blocks_v)
                bp = int(run.bp[s])
                ids = run.ranked[s * (prefix + 1): s * (prefix + 1) + bp].cpu().numpy()
                check_parity(oracle, q[s, 0], bs, make_config(epsilon=0.95), 0, ids, bp, run.out[s, 0].cpu().numpy(),
                             float(run.est[s]))
    # a full tail slot refuses the next token
    k = torch.zeros((nseq, d), device=dev)
    assert pool.append_tokens(tail, k, k) == 1
