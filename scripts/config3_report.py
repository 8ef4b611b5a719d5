"""BASELINE config 3 report: threshold sweep eps 0.8-0.99 vs fixed top-k 64/128 at 64K context
(one request, one layer: 8 kv heads x GQA group 4 = 32 q-heads, d=128, B=16, bf16 pool, planted keys),
blocks read and output error against fp64 exact attention (psattn_exact_attention).
usage: python scripts/config3_report.py [out.json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_gpu_tradeoff import config3_sweep  # noqa: E402
from paper_2503_00392_b200 import batch, capi  # noqa: E402

rows = {}
for dist, planted in (("planted", 1 / 32), ("iso", 0.0)):
    r, _, _ = config3_sweep((capi, batch), n_kv_units=8, planted=planted)
    rows[dist] = r
rep = dict(config="config3: 64K ctx, 1 request x 1 layer, 32 q / 8 kv heads, d=128, B=16, bf16 KV, microbatch 1, "
                  "CuboidMean; error = max-abs vs fp64 exact attention over all blocks", rows=rows)
txt = json.dumps(rep, indent=1)
print(txt)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(txt)
