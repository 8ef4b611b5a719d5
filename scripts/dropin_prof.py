"""Per-call cost of the drop-in C ABI (psattn_run_multi_head) on bench-shaped units.

usage (GPU box): PSA_RUN_PROF=1 python scripts/dropin_prof.py [units] [calls] 2> gpurun_out/dropin_prof.log
Prints the mean wall time per call and, with PSA_RUN_PROF set, run_device's phase times go to stderr.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_00392_b200 import capi  # noqa: E402
from workload import synth  # noqa: E402

units = int(sys.argv[1]) if len(sys.argv) > 1 else 4
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ctx, block, g = 131072, 16, 4
n = ctx // block
p = synth.params(seed=1, dim=128, block_tokens=block, skew=8.0, planted_prob=1.0 / 32.0, round_bf16=1)
st = capi.Store(capacity=n * units, n_layers=1)
lists, qs = [], []
for i in range(units):
    uid = i * 137
    k, v = synth.unit_host(p, uid, ctx)
    st.put_many(i * n, k, v)
    lists.append(np.arange(i * n, (i + 1) * n, dtype=np.int64))
    qs.append(np.stack([synth.query(p, uid, h) for h in range(g)]).astype(np.float32))
cfg = capi.config_default(epsilon=0.95, microbatch_size=1)
for i in range(units):
    capi.check(st.run_multi_head(qs[i], [lists[i]], cfg)[0])


def timed(tag):
    t = []
    for c in range(calls):
        i = c % units
        t0 = time.perf_counter()
        capi.check(st.run_multi_head(qs[i], [lists[i]], cfg)[0])
        t.append(time.perf_counter() - t0)
    t = np.array(t) * 1e6
    print(f"{tag}: dropin per call: mean {t.mean():.1f} us, median {np.median(t):.1f} us, min {t.min():.1f} us "
          f"({g / t.mean() * 1e6:.0f} queries/s)", flush=True)
    print(f"=== {tag} done", file=sys.stderr, flush=True)


ref_out = [st.run_multi_head(qs[i], [lists[i]], cfg) for i in range(units)]
timed("default")
if os.environ.get("LAYER_CALL"):  # one call over every unit (all kv-head lists, g q-heads each)
    qa = np.concatenate(qs)
    t0 = time.perf_counter()
    for c in range(calls):
        capi.check(st.run_multi_head(qa, lists, cfg)[0])
    el = (time.perf_counter() - t0) / calls
    print(f"layer call ({units} lists): {el * 1e6:.1f} us per call ({qa.shape[0] / el:.0f} queries/s)", flush=True)
    print("=== layer done", file=sys.stderr, flush=True)
# the raw C call with prebuilt arguments (no Python wrapper work)
import ctypes as C  # noqa: E402
ids = lists[0]
off = np.array([0, n], np.int64)
out = np.zeros((g, 128), np.float32)
stt = (capi.RunStats * g)()
un = C.c_int64(0)
t0 = time.perf_counter()
for c in range(calls):
    capi.check(capi.lib.psattn_run_multi_head(st.h, capi._p(qs[0]), g, 128, capi._p(ids), capi._p(off), 1,
                                              C.byref(cfg), capi._p(out), stt, C.byref(un)))
print(f"raw ctypes: {(time.perf_counter() - t0) / calls * 1e6:.1f} us per call", flush=True)
for m in sys.argv[3:]:
    if m == "dense":
        capi.check(capi.lib.psattn_set_dense_early(C.c_float(1e30)))
    for i in range(units):
        rc, o, res, _ = st.run_multi_head(qs[i], [lists[i]], cfg)
        r0 = ref_out[i]
        print(f"  {m} unit {i}: max|d out| {np.abs(o - r0[1]).max():.3g}, blocks "
              f"{[x.blocks_processed for x in res]} vs {[x.blocks_processed for x in r0[2]]}")
    timed(m)

