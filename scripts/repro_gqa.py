"""Small GQA-kernel reproducer (lists longer than one tranche) for compute-sanitizer runs."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from helpers import random_blockset, check_parity  # noqa: E402
from oracle.pyoracle import COracle, make_config  # noqa: E402
from paper_2503_00392_b200 import batch, capi  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dt = int(sys.argv[2]) if len(sys.argv) > 2 else 1
capi.check(capi.lib.psattn_set_progressive_kernel(mode))
rng = np.random.default_rng(3)
d, T, g, n = 128, 16, 4, 1300
units = [random_blockset(rng, n, d, 16, 16, planted_frac=0.0) for _ in range(2)]
if dt == 1:
    for u in units:
        u.keys[:] = torch.tensor(u.keys).bfloat16().float().numpy()
        u.values[:] = torch.tensor(u.values).bfloat16().float().numpy()
qs = np.array([[rng.standard_normal(d) * 0.3 for _ in range(g)] for _ in units], np.float32)
pool = batch.DevicePool(d, T, dt, n * len(units))
ks = np.concatenate([u.keys.reshape(n, T, d) for u in units])
vs = np.concatenate([u.values.reshape(n, T, d) for u in units])
pool.put_blocks(np.arange(n * len(units), dtype=np.int32), np.full(n * len(units), T, np.int32), ks, vs)
dev = torch.device("cuda")
off = np.array([0, n, 2 * n], np.int64)
run = batch.BatchRun(pool, torch.tensor(qs, device=dev), torch.arange(2 * n, dtype=torch.int32, device=dev),
                     torch.tensor(off, device=dev), n, batch.BatchConfig(epsilon=0.99), want_ranked=True)
run.run()
torch.cuda.synchronize()
orc = COracle()
for u in range(2):
    for h in range(g):
        bp = int(run.bp[u * g + h])
        ids = run.ranked[u * n * g + h * n: u * n * g + h * n + bp].cpu().numpy()
        tag = check_parity(orc, qs[u, h], units[u], make_config(epsilon=0.99), 0, ids, bp, run.out[u, h].cpu().numpy(),
                           float(run.est[u * g + h]))
        print(u, h, bp, tag)
print("ok")
