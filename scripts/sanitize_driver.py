"""Small end-to-end launches of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): score (TMA), first tranche, GQA round kernel, dense hand-over, per-head kernel, metadata
build, append, tier install, tradeoff/exact, per-call scoring/ranking. Sizes are tiny: the tools replay every access."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_00392_b200 import batch, capi  # noqa: E402
from workload import synth  # fixture: the seekable synthetic generator

dev = torch.device("cuda")
d, T, g = 128, 16, 4


def synth_run(tokens, planted, cfg, kv=capi.PSATTN_KV_BF16, kernel=0):
    p = synth.params(seed=2, dim=d, block_tokens=T, skew=8.0, planted_prob=planted, round_bf16=1)
    nb = [(t + T - 1) // T for t in tokens]
    off = np.zeros(len(tokens) + 1, np.int64)
    off[1:] = np.cumsum(nb)
    pool = batch.DevicePool(d, T, kv, int(off[-1]))
    uids = list(range(7, 7 + len(tokens)))
    synth.fill(pool, p, uids, off[:-1], tokens)
    qs = np.array([[synth.query(p, u, h) for h in range(g)] for u in uids], np.float32)
    run = batch.BatchRun(pool, torch.tensor(qs, device=dev), torch.arange(int(off[-1]), dtype=torch.int32, device=dev),
                         torch.tensor(off, device=dev), max(nb), batch.BatchConfig(**cfg), want_ranked=True)
    capi.check(capi.lib.psattn_set_progressive_kernel(kernel))
    run.run()
    torch.cuda.synchronize()
    capi.check(capi.lib.psattn_set_progressive_kernel(0))
    return pool, run


synth_run([16 * 900 + 3, 16 * 300], 1 / 32, dict(epsilon=0.95))            # score + first tranche + GQA
synth_run([16 * 700 + 5], 0.0, dict(epsilon=0.95))                          # dense hand-over
for ranks in (256, 32):  # partial dense: candidate prefix select, windowed K / V walks (32: escalations)
    capi.check(capi.lib.psattn_set_dense_partial(ranks))
    synth_run([16 * 3000 + 9, 16 * 1200], 1 / 32, dict(epsilon=0.99))
capi.check(capi.lib.psattn_set_dense_partial(1024))
synth_run([16 * 500], 0.0, dict(epsilon=0.9), kernel=1)                     # per-head kernel
synth_run([16 * 600 + 7, 16 * 90], 1 / 32, dict(epsilon=0.95), kernel=2)     # GQA round kernel
synth_run([16 * 400], 1 / 32, dict(epsilon=0.95, scale_override=4.0))        # stream kernel -> dense redo (extreme logits)
synth_run([16 * 300, 16 * 77 + 2], 1 / 32, dict(epsilon=0.8, microbatch_size=3, topk=40))  # stream kernel, top-k
synth_run([16 * 400 + 1], 0.05, dict(topk=64, microbatch_size=3), kv=capi.PSATTN_KV_F32)
pool, run = synth_run([16 * 300], 0.05, dict(epsilon=0.9, audit_coverage=1, microbatch_size=2))
run.exact_attention()
torch.cuda.synchronize()
# append + metadata rebuild
tail = torch.tensor([5, 9], dtype=torch.int32, device=dev)
pool.append_tokens(tail, torch.randn(2, d, device=dev), torch.randn(2, d, device=dev))
torch.cuda.synchronize()
# two-tier store: put, batch with host-resident blocks, install
tier = batch.DeviceTier(d, T, capi.PSATTN_KV_BF16, 2, 200, 60)
rng = np.random.default_rng(0)
K = rng.standard_normal((200, T, d)).astype(np.float32)
V = rng.standard_normal((200, T, d)).astype(np.float32)
tier.put_blocks(np.arange(200), np.arange(200) % 2, np.full(200, T), K, V)
lists = [np.arange(0, 200, 2), np.arange(1, 200, 2)]
off = torch.tensor([0, 100, 200], dtype=torch.int64, device=dev)
tr = batch.BatchRun(tier, torch.randn(2, g, d, device=dev), torch.tensor(np.concatenate(lists).astype(np.int32), device=dev),
                    off, 100, batch.BatchConfig(epsilon=0.9))
tr.run()
tr.run()
torch.cuda.synchronize()
# per-call scoring / ranking over host records (metadata_api.cu)
mk = rng.standard_normal((50, T, 40)).astype(np.float32)
sc = capi.criticality_scores(rng.standard_normal(40).astype(np.float32), mk.mean(1), mk.min(1), mk.max(1), 2)
capi.rank_by_scores(np.round(sc, 1), np.arange(50))
torch.cuda.synchronize()
# drop-in store with long blocks (33..128 tokens: chunked per-head kernel)
st = capi.Store(capacity=32)
rng2 = np.random.default_rng(3)
for i in range(24):
    nt = int(rng2.integers(1, 129))
    kk = rng2.standard_normal((nt, 64)).astype(np.float32)
    capi.check(st.put(i, kk, kk))
capi.check(st.run_query(rng2.standard_normal(64).astype(np.float32), np.arange(24), capi.config_default(epsilon=0.9))[0])
torch.cuda.synchronize()
# drop-in store, bf16-exact values: lossless bf16 pool (stream kernel), run_multi_head over two
# kv-head lists twice (the second replays the captured graph; compact read-back), then a block
# that is not bf16-exact moves the pool to fp32 and the query runs again
st2 = capi.Store(capacity=1024)
n2 = 600
kb = rng2.standard_normal((n2, 16, 128)).astype(np.float32)
kb = (kb.view(np.uint32) & 0xFFFF0000).view(np.float32)
st2.put_many(0, kb, kb)
q2 = rng2.standard_normal((8, 128)).astype(np.float32)
lists2 = [np.arange(0, 300, dtype=np.int64), np.arange(300, 600, dtype=np.int64)]
for _ in range(2):
    capi.check(st2.run_multi_head(q2, lists2, capi.config_default(epsilon=0.95))[0])
odd = rng2.standard_normal((16, 128)).astype(np.float32)
capi.check(st2.put(10_000, odd, odd))
capi.check(st2.run_multi_head(q2, lists2, capi.config_default(epsilon=0.95))[0])
torch.cuda.synchronize()
print("sanitize driver ok")
