#!/usr/bin/env python3
"""PSA decode-attention benchmark (BASELINE.json config 2 on one B200, weak-scaled over N GPUs).

Workload ("step"): one decode step of Llama-3.1-8B at 128K context for a batch of
8 requests — every (request, layer, q-head) query = 8 x 32 x 32 = 8192 progressive
sparse attention queries over 2048 kv-head block lists of 8192 blocks (B=16, d=128,
bf16 KV in the unified HBM pool, eps=0.95, microbatch 1, CuboidMean). Synthetic data
from the seekable generator (planted pattern of the reference workload: skew 8,
P(planted)=1/32, i.e. 64 planted blocks per 2048; --dist iso for isotropic keys).
The pool (~144 GiB) is far larger than L2, so no explicit flush is needed.

`value`  = queries/s over the whole job, inputs resident in HBM (device-timed, max over ranks).
`e2e`    = same metric through the C ABI batch call with per-step H2D of the queries from
           pinned host memory and D2H of outputs + stats inside the timed region.
`--impl reference` times the reference's own CPU implementation (compiled from
/root/reference into oracle/_ref) on the host cores on a bounded sample.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PSA decode-attn queries/s, Llama-3.1-8B 128K ctx; HBM GB/s vs peak; KV bytes read"
UNIT = "queries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dist", default="planted", choices=["planted", "iso"])
    ap.add_argument("--requests", type=int, default=8, help="requests per GPU (weak scaling, the default)")
    ap.add_argument("--total-requests", type=int, default=0,
                    help="fixed total requests over all GPUs (strong scaling; config 5 = 64): requests shard "
                         "across ranks, (request, kv head) pairs when requests < GPUs; layers beyond the HBM "
                         "budget are not resident (a step runs the resident layers)")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--block", type=int, default=16)
    ap.add_argument("--eps", type=float, default=0.95)
    ap.add_argument("--microbatch", type=int, default=1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="budget of the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--psa-kernel", type=int, default=0, help="0 auto, 1 per q-head, 2 GQA group")
    ap.add_argument("--score-kernel", type=int, default=0, help="0 auto, 1 register-staged, 2 TMA-staged")
    ap.add_argument("--pipeline", type=int, default=1, help="0 auto, 1 off, k sub-batches")
    ap.add_argument("--graph", type=int, default=1, help="1: replay the step as a captured CUDA graph")
    ap.add_argument("--dense-early", type=float, default=2.0,
                    help="early dense hand-over of flat heads (nats between ranks 0 and 383; 0 off)")
    ap.add_argument("--dense-partial", type=int, default=1024,
                    help="dense hand-over: ranks of each head's first-round candidate prefix (0: whole lists)")
    ap.add_argument("--plan-only", action="store_true",
                    help="launcher/sharding dry run (no GPU): every rank reports its units over gloo")
    ap.add_argument("--e2e-buffers", type=int, default=1, choices=[1], help=argparse.SUPPRESS)  # (kept for old scripts)
    ap.add_argument("--dropin-groups", type=int, default=2,
                    help="(request, layer) groups timed through the drop-in C ABI (psattn_run_multi_head, "
                         "host buffers); 0: off")
    ap.add_argument("--dropin-units", dest="dropin_groups", type=int, help=argparse.SUPPRESS)  # old scripts
    ap.add_argument("--check", type=int, default=16,
                    help="after timing: units of this rank's step checked against the reference (0: off)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def synth_params(args):
    from workload import synth
    prob = 1.0 / 32.0 if args.dist == "planted" else 0.0
    return synth.params(seed=args.seed, dim=args.dim, block_tokens=args.block, skew=8.0, planted_prob=prob,
                             round_bf16=1)


# ----------------------------------------------------------------------------------------------
# Reference CPU arm: the unmodified reference library (oracle/_ref) on the host cores.
# ----------------------------------------------------------------------------------------------
class ReferenceCPU:
    kind = "reference"
    """psattn::psa_attention_multi_head (reference engine.cpp:240-260) of the unmodified reference
    library on kv-head units of the same workload shape (n = ctx/B blocks, GQA group hq/hkv, same
    synthetic bf16 values upcast to fp32), one TieredBlockStore per host thread (a shared store
    serialises on its mutex, reference store.hpp:112)."""

    def __init__(self, args, rank_offset=0):
        from oracle.pyoracle import RefDriver, make_config
        from workload import synth
        drv = RefDriver()
        p = synth_params(args)
        self.g = args.hq // args.hkv
        self.n = -(-args.ctx // args.block)
        self.threads = max(1, min(os.cpu_count() or 1, 64))
        self.stores, self.qs = [None] * self.threads, [None] * self.threads
        self.cfg = make_config(epsilon=args.eps, microbatch_size=args.microbatch)
        self.ids = np.arange(self.n, dtype=np.int64)[None, :]
        self.args = args

        def setup(t):
            uid = 10_000_000 + rank_offset + t
            k, v = synth.unit_host(p, uid, args.ctx)
            st = drv.store(capacity=0)
            r = args.ctx - (self.n - 1) * args.block  # tokens of the (possibly ragged) last block
            st.put_many(0, k[:-1], v[:-1])
            st.put(self.n - 1, k[-1, :r], v[-1, :r])
            self.stores[t] = st
            self.qs[t] = np.array([synth.query(p, uid, h) for h in range(self.g)], np.float32)
            st.multi_head(self.qs[t], self.ids, self.cfg, want_ids=False)  # warm

        ths = [threading.Thread(target=setup, args=(t,)) for t in range(self.threads)]
        [th.start() for th in ths]
        [th.join() for th in ths]

    def sample(self, seconds):
        """Every thread runs whole GQA groups until the window closes; returns queries/s."""
        counts = [0] * self.threads
        t0 = time.perf_counter()
        stop_at = t0 + seconds

        def work(t):
            while True:
                self.stores[t].multi_head(self.qs[t], self.ids, self.cfg, want_ids=False)
                counts[t] += self.g
                if time.perf_counter() >= stop_at:
                    break

        ths = [threading.Thread(target=work, args=(t,)) for t in range(self.threads)]
        [th.start() for th in ths]
        [th.join() for th in ths]
        el = time.perf_counter() - t0
        desc = (f"{self.threads} host threads, each on its own kv-head unit of {self.n} blocks "
                f"(ctx {self.args.ctx}, GQA group {self.g}) via psa_attention_multi_head, eps {self.args.eps}; "
                f"{sum(counts)} queries in {el:.1f}s")
        return sum(counts) / el, desc


class PortCPU(ReferenceCPU):
    """Fallback when oracle/_ref (the compiled reference) is absent on the box: the plain-C oracle
    port (oracle/psa_oracle.c, the reference algorithm restated) on the same units, one head at a
    time per thread, kind "port"."""
    kind = "port"

    def __init__(self, args, rank_offset=0):
        from oracle.pyoracle import BlockSet, COracle, make_config
        from workload import synth
        self.orc = COracle()
        p = synth_params(args)
        self.g = args.hq // args.hkv
        self.n = -(-args.ctx // args.block)
        self.threads = max(1, min(os.cpu_count() or 1, 64))
        self.cfg = make_config(epsilon=args.eps, microbatch_size=args.microbatch)
        self.args = args
        self.units, self.qs = [None] * self.threads, [None] * self.threads

        def setup(t):
            uid = 10_000_000 + rank_offset + t
            k, v = synth.unit_host(p, uid, args.ctx)
            r = args.ctx - (self.n - 1) * args.block
            self.units[t] = BlockSet(list(k[:-1]) + [k[-1, :r]], list(v[:-1]) + [v[-1, :r]])
            self.qs[t] = np.array([synth.query(p, uid, h) for h in range(self.g)], np.float32)

        ths = [threading.Thread(target=setup, args=(t,)) for t in range(self.threads)]
        [th.start() for th in ths]
        [th.join() for th in ths]

    def sample(self, seconds):
        counts = [0] * self.threads
        t0 = time.perf_counter()
        stop_at = t0 + seconds

        def work(t):
            while True:
                for h in range(self.g):
                    self.orc.psa(self.qs[t][h], self.units[t], self.cfg)
                counts[t] += self.g
                if time.perf_counter() >= stop_at:
                    break

        ths = [threading.Thread(target=work, args=(t,)) for t in range(self.threads)]
        [th.start() for th in ths]
        [th.join() for th in ths]
        el = time.perf_counter() - t0
        desc = (f"{self.threads} host threads, each on its own kv-head unit of {self.n} blocks "
                f"(ctx {self.args.ctx}, GQA group {self.g}) via the C oracle port (oracle/_ref absent), eps "
                f"{self.args.eps}; {sum(counts)} queries in {el:.1f}s")
        return sum(counts) / el, desc


def cpu_reference(args):
    """The compiled reference when present (kind "reference"), else the C oracle port."""
    from oracle.pyoracle import ref_available
    return ReferenceCPU(args) if ref_available() else PortCPU(args)


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    per_step = max(args.cpu_seconds / max(K + W, 1), 0.5)
    ref = cpu_reference(args)
    vals = []
    desc, threads = "", ref.threads
    for i in range(W + K):
        qps, desc = ref.sample(per_step)
        if i >= W:
            vals.append(qps)
    v = float(np.median(vals))
    cpu = os.popen("lscpu | grep 'Model name' | head -1").read().strip().split(":")[-1].strip()
    line = dict(metric=METRIC, value=v, unit=UNIT, n_gpus=args.gpus, steps=K, warmup=W, ms_per_step=None,
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f32", data="synthetic",
                impl="reference",
                config=dict(workload="config2 sample: Llama-3.1-8B shape kv-head units, 128K ctx, "
                                     f"{args.dist} keys", ctx=args.ctx, group=args.hq // args.hkv, eps=args.eps,
                            microbatch=args.microbatch),
                cpu_baseline=dict(value=v, unit=UNIT, cores=threads, kind=getattr(ref, "kind", "reference"),
                                  sample=desc, cpu=cpu),
                e2e=dict(value=v, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
# Our arm
# ----------------------------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/psa_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return dict(sm_mhz=float(np.median(sm)) if sm else None, sm_max_mhz=mx, reasons=sorted(reasons),
                    samples=len(sm))


def measured_peak():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(stage):
    """dram bytes per launch of the stage's kernel from the committed ncu summary, if any."""
    try:
        s = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return s["kernels"][stage]["dram_bytes_per_launch"]
    except Exception:
        return None


def check_step(args, p, run, q_host, unit_ids, n, g):
    """Samples `--check` units spread over this rank's step (requests x layers x kv heads) and
    compares all g heads of each with the reference on the same synthetic data (oracle/parity.py:
    compiled reference psa_attention_multi_head, C oracle for ties). Outside every timed region."""
    t0 = time.time()
    U = unit_ids.size
    pick = np.unique(np.linspace(0, U - 1, min(args.check, U)).astype(np.int64))
    out = run.out.cpu().numpy()
    bp = run.bp.cpu().numpy()
    ranked = run.ranked.cpu().numpy()
    units = []
    for u in pick:
        ids = [ranked[u * n * g + h * n: u * n * g + h * n + int(bp[u * g + h])] for h in range(g)]
        units.append(dict(uid=int(unit_ids[u]), q=q_host[u], out=out[u], bp=bp[u * g: (u + 1) * g], ids=ids))
    try:
        from oracle.parity import check_sampled_units
        r = check_sampled_units(p, units, args.ctx, args.eps, args.microbatch)
        r["ok"] = True
    except AssertionError as e:
        r = dict(ok=False, units=len(units), error=str(e)[:400])
    except Exception as e:  # noqa: BLE001  (checker unavailable: say so, never claim parity)
        r = dict(ok=None, units=len(units), error=f"checker unavailable: {e}"[:400])
    r["sampled_units"] = [int(unit_ids[u]) for u in pick]
    r["seconds"] = round(time.time() - t0, 1)
    return r


def dropin_e2e(args, p, groups, n, g, seconds=2.0):
    """`e2e_dropin`: the same queries through the reference-facing C ABI — psattn_store (blocks put as
    host fp32 K/V, reference capi.cpp:134-156) and psattn_run_multi_head (psa_attention_multi_head,
    engine.cpp:240-260) — host q in, host outputs + stats out, every copy and the host-side
    accounting inside the timed region. One call per (request, layer): its hq q-heads over its hkv
    kv-head lists, the call a decode step makes for one layer of one request (the multi-head API's
    shape). `per_kv_head` times the same store one kv-head list (g q-heads) per call — the unit the
    CPU reference arm's threads run."""
    from paper_2503_00392_b200 import capi
    from workload import synth
    hkv = args.hkv
    units = [(int(r) * args.layers + int(l)) * hkv + h for r, l in groups for h in range(hkv)]
    st = capi.Store(capacity=n * len(units), n_layers=1)
    lists, qs = [], []
    for i, uid in enumerate(units):
        k, v = synth.unit_host(p, uid, args.ctx)
        r = args.ctx - (n - 1) * args.block  # ragged last block keeps its own token count
        st.put_many(i * n, k[:-1], v[:-1])
        capi.check(st.put(i * n + n - 1, k[-1, :r], v[-1, :r]))
        del k, v
        lists.append(np.arange(i * n, (i + 1) * n, dtype=np.int64))
        qs.append(np.stack([synth.query(p, uid, h) for h in range(g)]).astype(np.float32))
    cfg = capi.config_default(epsilon=args.eps, microbatch_size=args.microbatch)
    calls_layer = [(np.concatenate(qs[j * hkv:(j + 1) * hkv]), lists[j * hkv:(j + 1) * hkv])
                   for j in range(len(groups))]
    calls_unit = [(qs[i], [lists[i]]) for i in range(len(units))]

    def timed(calls):
        for q, ls in calls:  # warm-up (the first call sizes the store's staging buffers)
            capi.check(st.run_multi_head(q, ls, cfg)[0])
        ncall, nq, t0 = 0, 0, time.perf_counter()
        while True:
            for q, ls in calls:
                capi.check(st.run_multi_head(q, ls, cfg)[0])
                ncall += 1
                nq += q.shape[0]
            el = time.perf_counter() - t0
            if el >= seconds:
                return nq / el, ncall, el

    v_layer, c_layer, s_layer = timed(calls_layer)
    v_unit, c_unit, s_unit = timed(calls_unit)
    st.close()
    return dict(value=v_layer, unit=UNIT, calls=c_layer, seconds=round(s_layer, 3),
                groups=[[int(r), int(l)] for r, l in groups], kv_dtype="fp32 host blocks via put_block (bf16-exact values: stored losslessly as bf16)",
                api=f"psattn_run_multi_head per (request, layer): {args.hq} q-heads over {hkv} kv-head lists of "
                    f"{n} blocks, host buffers",
                per_kv_head=dict(value=v_unit, unit=UNIT, calls=c_unit, seconds=round(s_unit, 3),
                                 api=f"psattn_run_multi_head per kv-head unit: {g} q-heads, one list"))


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2503_00392_b200 import batch, capi, shard

    ws, rank, local = dist_env()
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines show the rank count
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    capi.check(capi.lib.psattn_set_progressive_kernel(args.psa_kernel))
    capi.check(capi.lib.psattn_set_score_kernel(args.score_kernel))
    capi.check(capi.lib.psattn_set_pipeline(args.pipeline))
    capi.check(capi.lib.psattn_set_dense_early(args.dense_early))
    capi.check(capi.lib.psattn_set_dense_partial(args.dense_partial))
    from workload import synth
    p = synth_params(args)
    g = args.hq // args.hkv
    n = -(-args.ctx // args.block)
    # ---- units of this rank: weak scaling (requests per GPU fixed) or a fixed total (strong) ----
    strong = args.total_requests > 0
    total_req = args.total_requests if strong else args.requests * ws
    unit_ids = shard.plan_units(total_req, args.layers, args.hkv, ws, rank)
    layers_resident = args.layers
    slot_b = 2 * args.block * args.dim * 2
    meta_b1 = args.dim * (4 + 2 * 2)
    overflow = unit_ids.size * n * (slot_b + meta_b1) > torch.cuda.mem_get_info(dev)[0] - (10 << 30)
    if overflow and not strong:  # the weak-scaling shape does not fit one GPU: the resident layers (in config)
        print(f"bench: {unit_ids.size} units x {n} blocks exceed HBM; running the resident layers", file=sys.stderr)
    if strong or overflow:
        budget = torch.cuda.mem_get_info(dev)[0] - (10 << 30)
        reqs_here = max(1, len(np.unique(unit_ids // (args.layers * args.hkv))))
        layers_resident = shard.resident_layers(reqs_here, args.layers, args.hkv, n, slot_b + meta_b1, budget)
        layers_resident = int(shard.max_over_ranks(-layers_resident, dev) * -1)  # the same on every rank
        unit_ids = unit_ids[(unit_ids // args.hkv) % args.layers < layers_resident]
    U = int(unit_ids.size)
    nq = U * g
    nq_all = int(shard.sum_over_ranks(nq, dev))
    # ---- unified pool: every (request, layer, kv-head) list is n consecutive slots ----
    pool = batch.DevicePool(args.dim, args.block, capi.PSATTN_KV_BF16, U * n)
    t0 = time.time()
    synth.fill(pool, p, unit_ids, np.arange(U, dtype=np.int64) * n, np.full(U, args.ctx, np.int64))
    torch.cuda.synchronize()
    fill_s = time.time() - t0
    q_host = np.zeros((U, g, args.dim), np.float32)
    for u in range(U):
        for h in range(g):
            q_host[u, h] = synth.query(p, int(unit_ids[u]), h)
    q_dev = torch.tensor(q_host, device=dev)
    slots = torch.arange(U * n, dtype=torch.int32, device=dev)
    off = torch.arange(U + 1, dtype=torch.int64, device=dev) * n
    cfg = batch.BatchConfig(epsilon=args.eps, microbatch_size=args.microbatch)
    run = batch.BatchRun(pool, q_dev, slots, off, n, cfg, want_ranked=True)
    stream = torch.cuda.Stream()  # a non-default stream: graph capture and every launch/copy/event go here
    torch.cuda.set_stream(stream)

    def barrier():
        if ws > 1:
            dist.barrier()

    # ---- device-timed region (inputs resident) ----
    # nvidia-smi samples every 50 ms from the start of the warm-up through the timed region
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        launches_per_step = run.run()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    step = run.run
    if args.graph:
        run.capture(stream)  # one decode step = one CUDA graph replay
        step = run.run_graph
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
    phases = np.zeros(12, np.uint64)
    prof_build = capi.lib.psattn_debug_gqa_phases(phases.ctypes.data) == 0  # PROF=1 development build only
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        launches_per_step = step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    # per-stage kernel times: the same steps launched directly with CUDA events between the stages
    capi.lib.psattn_profile_read(None, None, 1)
    sstats = np.zeros(4, np.uint64)
    capi.lib.psattn_debug_stream_stats(sstats.ctypes.data)  # zero the stream kernel's fetch counters
    sprof = np.zeros(32, np.uint64)
    capi.lib.psattn_debug_stream_prof(sprof.ctypes.data)
    capi.lib.psattn_profile_enable(1)
    for _ in range(args.steps):
        run.run()
    torch.cuda.synchronize()
    capi.lib.psattn_profile_enable(0)
    capi.lib.psattn_debug_stream_stats(sstats.ctypes.data)
    capi.lib.psattn_debug_stream_prof(sprof.ctypes.data)
    if sprof.any():  # development build with the stream kernel's wait-site cycle counters
        roles, sites = ["producer", "decider", "scorer", "v"], ["total", "drain", "scored", "pub", "ktile", "vtile"]
        units = max(1.0, float(sstats[3]))
        print(json.dumps({"stream_prof_cycles_per_unit": {
            r: {k: round(float(sprof[8 * i + j]) / units) for j, k in enumerate(sites + ["idle_it", "busy_it"])}
            for i, r in enumerate(roles)}}), file=sys.stderr)
    stage_ms = np.zeros(4, np.float64)
    stage_n = np.zeros(4, np.int64)
    capi.lib.psattn_profile_read(stage_ms.ctypes.data, stage_n.ctypes.data, 1)
    if prof_build:
        capi.lib.psattn_debug_gqa_phases(phases.ctypes.data)
        names = ["init", "order", "union", "k_pass", "decide", "v_pass", "advance", "finalize"]
        tot = float(phases[:8].sum())
        print(json.dumps({"gqa_phase_share": {k: round(float(phases[i]) / tot, 4) for i, k in enumerate(names)},
                          "rounds_per_cta": float(phases[8]) / (U * args.steps),
                          "cycles_per_cta": tot / (U * args.steps),
                          "warp0_decide_chunk": round(float(phases[9]) / tot, 4),
                          "warp0_k_work": round(float(phases[10]) / tot, 4),
                          "warp0_v_work": round(float(phases[11]) / tot, 4)}), file=sys.stderr)
    ms = shard.max_over_ranks(ms, dev)
    ms_per_step = ms / args.steps
    value = nq_all * args.steps / (ms / 1e3)

    # ---- algorithmic bytes ----
    un = run.union_blocks().cpu().numpy()
    bp = run.bp.cpu().numpy()
    torch.cuda.synchronize()
    lay = pool.layout()
    meta_b = U * n * lay.meta_bytes
    kv_union_b = int(un.sum()) * lay.slot_bytes
    kv_sum_b = int(bp.sum()) * lay.slot_bytes
    qo_b = 2 * nq * args.dim * 4
    step_bytes = meta_b + kv_union_b + qo_b
    kv_full_b = U * n * lay.slot_bytes
    # physical K/V tiles the stream kernel fetched vs the algorithmic union (bounded speculation)
    fetch = None
    if int(sstats[3]) > 0:
        kt, vt = float(sstats[0]) / args.steps, float(sstats[1]) / args.steps
        tile_b = lay.slot_bytes / 2
        fetch = dict(k_tiles_per_step=kt, v_tiles_per_step=vt, union_blocks_per_step=float(un.sum()),
                     fetched_bytes_per_step=(kt + vt) * tile_b, kv_union_bytes=kv_union_b,
                     waste_frac=(kt + vt) * tile_b / max(kv_union_b, 1) - 1.0,
                     rounds_per_unit=float(sstats[2]) / max(float(sstats[3]), 1.0))
    stage_names = ["oracle", "score", "order", "progressive"]
    per_launch_ms = {s: stage_ms[i] / max(stage_n[i], 1) for i, s in enumerate(stage_names) if stage_n[i] > 0}
    stage_bytes = {"score": meta_b + nq * args.dim * 4, "progressive": kv_union_b + qo_b,
                   "order": None, "oracle": None}
    dom = max(per_launch_ms, key=per_launch_ms.get)
    peak, peak_kind = measured_peak()
    ach = (stage_bytes[dom] / (per_launch_ms[dom] / 1e3) / 1e9) if stage_bytes.get(dom) else None
    roofline = dict(bound="hbm", kernel=dom, achieved=ach, peak=peak, peak_kind=peak_kind, unit="GB/s",
                    frac=(ach / peak) if ach else None, traffic=ncu_traffic(dom),
                    algorithmic_bytes_per_launch=stage_bytes.get(dom), launch_ms=per_launch_ms[dom])
    step_gbs = step_bytes / (ms_per_step / 1e3) / 1e9

    # ---- e2e through the C ABI batch call, host buffers, copies inside the timed region ----
    # Every step: H2D of its queries from pinned host memory, the step, D2H of its outputs and stats,
    # and the host waiting for them before the next step. (A double-buffered loop overlapping the
    # copies with the neighbouring steps measured no better: 1.656 vs 1.683 M queries/s.)
    q_pin = torch.from_numpy(q_host).pin_memory()
    out_pin = torch.empty(run.out.shape, dtype=torch.float32).pin_memory()
    bp_pin = torch.empty(nq, dtype=torch.int64).pin_memory()
    est_pin = torch.empty(nq, dtype=torch.float64).pin_memory()
    term_pin = torch.empty(nq, dtype=torch.int32).pin_memory()
    h2d = q_pin.numel() * 4
    d2h = out_pin.numel() * 4 + nq * (8 + 8 + 4)

    def e2e_step():
        run.q.copy_(q_pin, non_blocking=True)
        step()
        out_pin.copy_(run.out, non_blocking=True)
        bp_pin.copy_(run.bp, non_blocking=True)
        est_pin.copy_(run.est, non_blocking=True)
        term_pin.copy_(run.term, non_blocking=True)

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
        stream.synchronize()  # the caller consumes each step's outputs on the host
    e2e_s = shard.max_over_ranks(time.perf_counter() - t0, dev)
    e2e_val = nq_all * args.steps / e2e_s

    # ---- optional final output gather over NCCL (N > 1; not part of `value`) ----
    gather = None
    if ws > 1:
        for _ in range(2):
            shard.gather_outputs(run.out)
        torch.cuda.synchronize()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            allout = shard.gather_outputs(run.out)
        g1.record(stream)
        torch.cuda.synchronize()
        gms = shard.max_over_ranks(g0.elapsed_time(g1) / args.steps, dev)
        gather = dict(ms_per_step=gms, bytes_per_step=int(allout.numel()) * 4, collective="all_gather (NCCL)",
                      value_with_gather=nq_all / ((ms_per_step + gms) / 1e3))

    # ---- parity of the benchmarked step itself (after timing; the checker is the reference) ----
    parity = None
    if args.check > 0:
        parity = check_step(args, p, run, q_host, unit_ids, n, g)  # every rank checks a sample of its own units

    # ---- the drop-in C ABI with host buffers (rank 0): psattn_run_multi_head per (request, layer) ----
    dropin = None
    if rank == 0 and args.dropin_groups > 0:
        rl = np.unique(unit_ids // args.hkv)  # this rank's (request, layer) pairs
        pick = rl[np.linspace(0, len(rl) - 1, min(args.dropin_groups, len(rl))).astype(np.int64)]
        dropin = dropin_e2e(args, p, [(x // args.layers, x % args.layers) for x in pick], n, g)

    # ---- CPU baseline (rank 0, N=1 only) ----
    cpu_base = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            ref = cpu_reference(args)
            v, desc = ref.sample(args.cpu_seconds)
            cpu_base = dict(value=v, unit=UNIT, cores=ref.threads, kind=getattr(ref, "kind", "reference"), sample=desc)
        except Exception as e:  # noqa: BLE001
            cpu_base = dict(value=None, unit=UNIT, cores=0, kind="reference", sample=f"unavailable: {e}")

    # ---- every rank's view (device, units, parity of its own sample) gathered on rank 0 ----
    me = dict(rank=rank, device=torch.cuda.get_device_name(dev), units=U, queries=nq, parity_ok=(parity or {}).get("ok"))
    ranks = [me]
    if ws > 1:
        ranks = [None] * ws
        dist.all_gather_object(ranks, me)
        if parity is not None:
            allp = [None] * ws
            dist.all_gather_object(allp, parity)
            parity = dict(ok=all(x.get("ok") for x in allp) if all(x.get("ok") is not None for x in allp) else None,
                          units=sum(x.get("units", 0) for x in allp), queries=sum(x.get("queries", 0) for x in allp),
                          exact=sum(x.get("exact", 0) for x in allp), tie=sum(x.get("tie", 0) for x in allp),
                          per_rank=allp)
    if rank == 0:
        if strong:
            wl = (f"config5: {total_req} concurrent 128K-context decodes (Llama-3.1-8B shape) over {ws} GPU(s), "
                  f"{layers_resident} of {args.layers} layers resident per step, eps {args.eps}")
        else:
            wl = f"config2: Llama-3.1-8B shape, {args.layers} layers, batch {args.requests} decode, ctx {args.ctx}, eps {args.eps}"
        line = dict(
            metric=METRIC, value=value, unit=UNIT, n_gpus=ws, steps=args.steps, warmup=args.warmup,
            ms_per_step=ms_per_step, higher_is_better=True, scaling="strong" if strong else "weak",
            vs_baseline=None, dtype="bf16",
            data=f"synthetic ({args.dist} keys, seekable generator, seed {args.seed})",
            config=dict(workload=wl, requests_total=total_req, requests_per_gpu=None if strong else args.requests,
                        layers=args.layers, layers_resident=layers_resident, ctx=args.ctx, hq=args.hq,
                        hkv=args.hkv, dim=args.dim, block=args.block, eps=args.eps, microbatch=args.microbatch,
                        queries_per_step=nq_all, kv_dtype="bf16", l2="inputs (~144 GiB/GPU) >> 126 MB L2; no flush",
                        parallelism=(f"request sharding x{ws}" if total_req >= ws else f"(request, kv head) sharding x{ws}")
                        + ", no collective on the data path"),
            world=dict(size=ws, backend="nccl" if ws > 1 else None, ranks=ranks),
            roofline=roofline,
            step_roofline=dict(per_gpu="rank 0", achieved=step_gbs, peak=peak, frac=step_gbs / peak, unit="GB/s",
                               bytes_per_step=step_bytes, meta_bytes=meta_b, kv_union_bytes=kv_union_b,
                               qo_bytes=qo_b),
            kv_fraction_read=kv_union_b / kv_full_b, kv_fraction_per_head_sum=kv_sum_b / (kv_full_b * g),
            mean_blocks_processed=float(bp.mean()), fetch=fetch,
            stage_ms_per_step={k: v for k, v in per_launch_ms.items()},
            cpu_baseline=cpu_base, parity=parity, parity_ok=(parity or {}).get("ok"),
            e2e=dict(value=e2e_val, unit=UNIT, h2d_bytes_per_step=h2d, d2h_bytes_per_step=d2h),
            e2e_dropin=dropin,
            gpu_launches=int(launches_per_step) * args.steps,
            cuda_graph=bool(args.graph), gather=gather,
            clocks=clk, setup=dict(fill_seconds=fill_s, pool_gib=(U * n * (lay.slot_bytes + lay.meta_bytes)) / 2**30),
        )
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def run_plan_only(args):
    """What each rank would own, gathered over gloo on the host (tests the N-rank launch on CPU)."""
    import torch.distributed as dist
    from paper_2503_00392_b200 import shard
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    total_req = args.total_requests if args.total_requests > 0 else args.requests * ws
    units = shard.plan_units(total_req, args.layers, args.hkv, ws, rank)
    me = dict(rank=rank, pid=os.getpid(), units=units.tolist())
    ranks = [me]
    if ws > 1:
        ranks = [None] * ws
        dist.all_gather_object(ranks, me)
    if rank == 0:
        print(json.dumps(dict(plan_only=True, n_gpus=args.gpus, world_size=ws, requests_total=total_req,
                              ranks=ranks)), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def relaunch_multi_gpu(args):
    """`--gpus N` outside torchrun: start N ranks (one process per GPU) under torch.distributed.run
    on 127.0.0.1 with this same command line and return their exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if (args.impl == "ours" or args.plan_only) and args.gpus > 1 and ws == 0:
        sys.exit(relaunch_multi_gpu(args))
    if ws and ws != args.gpus:
        print(json.dumps(dict(metric=METRIC, error=f"--gpus {args.gpus} but WORLD_SIZE {ws}")), flush=True)
        sys.exit(2)
    if args.plan_only:
        run_plan_only(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
