"""Generates tests/golden/ref_cases.json from the COMPILED REFERENCE (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py

Each case stores its generator seed and config plus the reference's outputs
(blocks processed, processed ids, fp32 output bytes, coverage estimates), so the
C oracle can be pinned on machines where the reference cannot be compiled.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import random_blockset  # noqa: E402
from oracle.pyoracle import RefDriver, make_config  # noqa: E402


def main():
    drv = RefDriver()
    rng = np.random.default_rng(77)
    cases = []
    for i in range(40):
        c = dict(seed=1000 + i, n=int(rng.integers(1, 80)), d=int(rng.choice([2, 8, 16, 32, 64, 128])),
                 tok_hi=int(rng.integers(1, 21)), planted=float(rng.choice([0.0, 0.1, 0.3])),
                 qscale=float(rng.choice([1.0, 2.0, 4.0])),
                 cfg=dict(epsilon=float(rng.choice([0.5, 0.8, 0.9, 0.95, 0.99, 1.0])),
                          microbatch_size=int(rng.integers(1, 6)), estimator=int(rng.integers(0, 3)),
                          ranking_mode=int(rng.integers(0, 2)), audit_coverage=int(rng.integers(0, 2))),
                 topk=int(rng.integers(0, 2)) * int(rng.integers(1, 30)))
        g = np.random.default_rng(c["seed"])
        bs = random_blockset(g, c["n"], c["d"], 1, c["tok_hi"], planted_frac=c["planted"])
        q = (g.standard_normal(c["d"]) * c["qscale"]).astype(np.float32)
        st = drv.store(capacity=64)
        st.put_blockset(bs)
        r = st.query(q, bs.ids, make_config(**c["cfg"]), c["topk"])
        assert r.status == 0
        c.update(blocks_processed=r.blocks_processed, processed_ids=list(map(int, r.processed_ids)),
                 output_hex=r.output.astype(np.float32).tobytes().hex(), estimated_coverage=r.estimated_coverage,
                 true_coverage=r.true_coverage if r.true_coverage is not None else -1.0,
                 terminated_early=r.terminated_early)
        cases.append(c)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_cases.json")
    json.dump(cases, open(out, "w"), indent=1)
    print(f"wrote {len(cases)} cases to {out}")


if __name__ == "__main__":
    main()
