import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2503_00392_b200 import batch, capi, shard
from workload import synth  # fixture: the seekable synthetic generator
args = bench.parse()
p = bench.synth(args)
g = args.hq // args.hkv; n = args.ctx // args.block
U = args.requests * args.layers * args.hkv
pool = batch.DevicePool(args.dim, args.block, capi.PSATTN_KV_BF16, U * n)
uids = shard.unit_ids(shard.shard_requests(args.requests, 1, 0), args.layers, args.hkv)
synth.fill(pool, p, uids, np.arange(U) * n, np.full(U, args.ctx))
q = np.array([[synth.query(p, int(u), h) for h in range(g)] for u in uids], np.float32)
dev = torch.device('cuda')
run = batch.BatchRun(pool, torch.tensor(q, device=dev), torch.arange(U * n, dtype=torch.int32, device=dev),
                     torch.arange(U + 1, dtype=torch.int64, device=dev) * n, n, batch.BatchConfig(epsilon=args.eps))
run.run(); torch.cuda.synchronize()
bp = run.bp.cpu().numpy().reshape(U, g)
print("max bp", bp.max(), "p99", np.percentile(bp, 99), "units with a head > 384:", int((bp.max(1) > 384).sum()), "of", U)
