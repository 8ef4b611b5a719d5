"""ctypes bindings to the oracles — TEST INFRASTRUCTURE ONLY.

* ``COracle``  -> oracle/build/libpsa_oracle.so (our plain-C restatement, psa_oracle.c)
* ``RefDriver`` -> oracle/_ref/libpsattn_refdrv.so (the unmodified reference library,
  compiled from /root/reference/proj/src by oracle/Makefile, plus our shim)

Only tests/, bench.py's cpu_baseline / reference arm and __graft_entry__.smoke()
import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libpsa_oracle.so")
REFDRV_SO = os.path.join(HERE, "_ref", "libpsattn_refdrv.so")
REF_SO = os.path.join(HERE, "_ref", "libpsattn_ref.so")


class Config(C.Structure):
    """Layout of psattn_config (reference include/psattn.h:75-83)."""

    _fields_ = [
        ("epsilon", C.c_double),
        ("microbatch_size", C.c_int32),
        ("block_size", C.c_int32),
        ("estimator", C.c_int32),
        ("ranking_mode", C.c_int32),
        ("audit_coverage", C.c_int32),
        ("scale_override", C.c_double),
    ]


def make_config(epsilon=0.95, microbatch_size=1, block_size=32, estimator=2, ranking_mode=0,
                audit_coverage=0, scale_override=0.0) -> Config:
    """Defaults = psattn_config_default (reference capi.cpp:194-203)."""
    return Config(epsilon, microbatch_size, block_size, estimator, ranking_mode, audit_coverage,
                  scale_override)


class _OrcResult(C.Structure):
    _fields_ = [
        ("blocks_processed", C.c_uint64),
        ("total_blocks", C.c_uint64),
        ("n_iterations", C.c_uint64),
        ("estimated_coverage", C.c_double),
        ("true_coverage", C.c_double),
        ("terminated_early", C.c_int32),
        ("status", C.c_int32),
    ]


class _OrcBlocks(C.Structure):
    _fields_ = [
        ("keys", C.c_void_p),
        ("values", C.c_void_p),
        ("row_off", C.c_void_p),
        ("ntok", C.c_void_p),
        ("ids", C.c_void_p),
        ("n", C.c_size_t),
        ("d", C.c_int32),
    ]


@dataclass
class QueryResult:
    output: np.ndarray
    blocks_processed: int
    total_blocks: int
    estimated_coverage: float
    true_coverage: float | None
    terminated_early: bool
    processed_ids: np.ndarray
    iteration_estimates: np.ndarray = field(default_factory=lambda: np.zeros(0))
    status: int = 0


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class BlockSet:
    """A list of KV blocks flattened for the oracles: rows of d floats."""

    def __init__(self, keys: list[np.ndarray], values: list[np.ndarray], ids=None):
        assert len(keys) == len(values) and len(keys) > 0
        self.d = int(keys[0].shape[1])
        self.ntok = np.array([k.shape[0] for k in keys], dtype=np.int32)
        self.row_off = np.zeros(len(keys), dtype=np.int64)
        self.row_off[1:] = np.cumsum(self.ntok[:-1])
        self.keys = np.ascontiguousarray(np.concatenate(keys, 0), dtype=np.float32)
        self.values = np.ascontiguousarray(np.concatenate(values, 0), dtype=np.float32)
        self.ids = (np.arange(len(keys), dtype=np.int64) if ids is None
                    else np.ascontiguousarray(ids, dtype=np.int64))
        self.n = len(keys)

    def block(self, i):
        a, b = self.row_off[i], self.row_off[i] + self.ntok[i]
        return self.keys[a:b], self.values[a:b]

    def _c(self) -> _OrcBlocks:
        return _OrcBlocks(self.keys.ctypes.data, self.values.ctypes.data, self.row_off.ctypes.data,
                          self.ntok.ctypes.data, self.ids.ctypes.data, self.n, self.d)


class COracle:
    """The plain-C restatement of the reference path (psa_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = C.CDLL(path)
        self.L = L
        L.orc_build_metadata.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_criticality.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                      C.c_double]
        L.orc_criticality.restype = C.c_double
        L.orc_rank_by_scores.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.orc_block_partial.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_float,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_block_partial.restype = C.c_float
        L.orc_block_log_as_oracle.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_double]
        L.orc_block_log_as_oracle.restype = C.c_double
        L.orc_exact_attention_blocks.argtypes = [C.c_void_p, C.POINTER(_OrcBlocks), C.c_void_p, C.c_size_t,
                                                 C.c_double, C.c_void_p]
        L.orc_estimate_coverage.argtypes = [C.c_double, C.c_double, C.c_uint64]
        L.orc_estimate_coverage.restype = C.c_double
        L.orc_psa.argtypes = [C.c_void_p, C.POINTER(_OrcBlocks), C.POINTER(Config), C.c_uint64, C.c_void_p,
                              C.POINTER(_OrcResult), C.c_void_p, C.c_void_p]
        L.orc_plan.argtypes = [C.c_void_p, C.POINTER(_OrcBlocks), C.POINTER(Config), C.c_void_p, C.c_void_p]
        L.orc_cache_create.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32]
        L.orc_cache_create.restype = C.c_void_p
        L.orc_cache_destroy.argtypes = [C.c_void_p]
        L.orc_cache_put.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_int64)]
        L.orc_cache_load.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.POINTER(C.c_int64)]
        L.orc_cache_release.argtypes = [C.c_void_p, C.c_int64, C.c_int32]
        L.orc_cache_resident.argtypes = [C.c_void_p, C.c_int64, C.c_int32]
        L.orc_cache_stats.argtypes = [C.c_void_p, C.c_void_p]

    # -- math ------------------------------------------------------------
    def build_metadata(self, keys: np.ndarray):
        keys = np.ascontiguousarray(keys, dtype=np.float32)
        n, d = keys.shape
        mean, lo, hi = (np.zeros(d, np.float32) for _ in range(3))
        st = self.L.orc_build_metadata(n, d, _p(keys), _p(mean), _p(lo), _p(hi))
        if st:
            raise ValueError("build_metadata: empty block")
        return mean, lo, hi

    def criticality(self, q, mean, lo, hi, estimator=2, scale=None):
        q = np.ascontiguousarray(q, np.float32)
        d = q.size
        scale = 1.0 / np.sqrt(d) if scale is None else scale
        arr = [np.ascontiguousarray(a, np.float32) for a in (mean, lo, hi)]
        return self.L.orc_criticality(_p(q), d, _p(arr[0]), _p(arr[1]), _p(arr[2]), estimator, scale)

    def rank_by_scores(self, scores, ids):
        scores = np.ascontiguousarray(scores, np.float64)
        ids = np.ascontiguousarray(ids, np.int64)
        out = np.zeros(scores.size, np.int64)
        self.L.orc_rank_by_scores(_p(scores), _p(ids), scores.size, _p(out))
        return out

    def block_partial(self, q, keys, values, scale):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        out = np.zeros(q.size, np.float32)
        mx, es = C.c_float(), C.c_float()
        la = self.L.orc_block_partial(_p(q), q.size, k.shape[0], _p(k), _p(v), scale, C.byref(mx), C.byref(es),
                                      _p(out))
        return dict(max_score=mx.value, exp_sum=es.value, log_as=la, out_unnorm=out)

    def block_log_as_oracle(self, q, keys, scale):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(keys, np.float32)
        return self.L.orc_block_log_as_oracle(_p(q), q.size, k.shape[0], _p(k), scale)

    def exact_attention_blocks(self, q, bs: BlockSet, sel, scale):
        q = np.ascontiguousarray(q, np.float32)
        sel = np.ascontiguousarray(sel, np.int64)
        out = np.zeros(bs.d, np.float64)
        cb = bs._c()
        self.L.orc_exact_attention_blocks(_p(q), C.byref(cb), _p(sel), sel.size, scale, _p(out))
        return out

    def estimate_coverage(self, acc, mn, n_left):
        return self.L.orc_estimate_coverage(acc, mn, n_left)

    def plan(self, q, bs: BlockSet, cfg: Config):
        q = np.ascontiguousarray(q, np.float32)
        ranked = np.zeros(bs.n, np.int64)
        scores = np.zeros(bs.n, np.float64)
        cb = bs._c()
        st = self.L.orc_plan(_p(q), C.byref(cb), C.byref(cfg), _p(ranked), _p(scores))
        if st:
            raise ValueError(f"plan failed with status {st}")
        return ranked, scores

    def psa(self, q, bs: BlockSet, cfg: Config, topk: int = 0) -> QueryResult:
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(bs.d, np.float32)
        pid = np.zeros(bs.n, np.int64)
        it = np.zeros(bs.n, np.float64)
        r = _OrcResult()
        cb = bs._c()
        st = self.L.orc_psa(_p(q), C.byref(cb), C.byref(cfg), topk, _p(out), C.byref(r), _p(pid), _p(it))
        bp = int(r.blocks_processed)
        return QueryResult(out, bp, int(r.total_blocks), r.estimated_coverage,
                           None if r.true_coverage < 0 else r.true_coverage, bool(r.terminated_early),
                           pid[:bp].copy(), it[: int(r.n_iterations)].copy(), st)


class RefDriver:
    """The UNMODIFIED reference (libpsattn_ref.so) through our shim (ref_driver.cpp)."""

    def __init__(self, path: str = REFDRV_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(path)
        self.L = L
        L.refdrv_last_error.restype = C.c_char_p
        L.refdrv_store_create.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_double]
        L.refdrv_store_create.restype = C.c_void_p
        L.refdrv_store_destroy.argtypes = [C.c_void_p]
        L.refdrv_put.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                 C.c_void_p]
        L.refdrv_release.argtypes = [C.c_void_p, C.c_int64]
        L.refdrv_put_many.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                      C.c_void_p, C.c_void_p]
        L.refdrv_stats.argtypes = [C.c_void_p, C.c_void_p]
        L.refdrv_layer_stats.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.refdrv_contains.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int32)]
        L.refdrv_enable_trace.argtypes = [C.c_void_p]
        L.refdrv_trace.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.refdrv_trace.restype = C.c_int64
        L.refdrv_query.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64, C.POINTER(Config),
                                   C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]
        L.refdrv_pipeline.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64,
                                      C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
        L.refdrv_multi_head.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                        C.c_uint64, C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
        L.refdrv_batched.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_uint64,
                                     C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.POINTER(C.c_uint64)]
        L.refdrv_build_metadata.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.refdrv_criticality.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                         C.c_double]
        L.refdrv_criticality.restype = C.c_double
        L.refdrv_block_log_as_oracle.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_double]
        L.refdrv_block_log_as_oracle.restype = C.c_double

    def error(self) -> str:
        return self.L.refdrv_last_error().decode()

    def criticality(self, q, mean, lo, hi, estimator=2, scale=None):
        """The reference's criticality_score (metadata.cpp:60-72), compiled."""
        q = np.ascontiguousarray(q, np.float32)
        scale = 1.0 / np.sqrt(q.size) if scale is None else scale
        arr = [np.ascontiguousarray(a, np.float32) for a in (mean, lo, hi)]
        return self.L.refdrv_criticality(_p(q), q.size, _p(arr[0]), _p(arr[1]), _p(arr[2]), estimator, scale)

    def store(self, capacity=256, n_layers=1, partitioned=0, fifo=0, miss_ms=0.0) -> "RefStore":
        return RefStore(self, capacity, n_layers, partitioned, fifo, miss_ms)

    def workload(self, **spec) -> "RefWorkload":
        """The reference's generate_workload (workload.cpp:49-153) with a WorkloadSpec's fields."""
        return RefWorkload(self, **spec)


class RefWorkload:
    """Requests of the reference's synthetic workload generator: blocks (ids, layers, n_tokens, K/V
    zero-padded to block_size), per-layer block lists and per-step queries."""

    FIELDS = ("n_requests", "dim", "block_size", "n_layers", "context_min", "context_max", "decode_steps", "rho",
              "skew", "planted_blocks", "planted_blocks_alt", "seed")

    def __init__(self, drv: RefDriver, **spec):
        L = drv.L
        L.refdrv_workload_create.argtypes = [C.c_int32] * 7 + [C.c_double, C.c_double, C.c_int32, C.c_int32,
                                                              C.c_uint64]
        L.refdrv_workload_create.restype = C.c_void_p
        L.refdrv_workload_destroy.argtypes = [C.c_void_p]
        L.refdrv_workload_n_requests.argtypes = [C.c_void_p]
        L.refdrv_workload_request.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.refdrv_workload_blocks.argtypes = [C.c_void_p, C.c_int32, C.c_int32] + [C.c_void_p] * 5
        L.refdrv_workload_layer_list.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        L.refdrv_workload_query.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
        sp = dict(n_requests=1, dim=64, block_size=32, n_layers=1, context_min=1024, context_max=1024,
                  decode_steps=8, rho=0.0, skew=0.0, planted_blocks=0, planted_blocks_alt=0, seed=1)
        sp.update(spec)
        self.spec = sp
        self.L = L
        self.h = L.refdrv_workload_create(*[sp[k] for k in self.FIELDS])
        if not self.h:
            raise RuntimeError(drv.error())
        self.requests = []
        d, B = sp["dim"], sp["block_size"]
        for r in range(L.refdrv_workload_n_requests(self.h)):
            info = np.zeros(5, np.int64)
            L.refdrv_workload_request(self.h, r, _p(info))
            nb = int(info[3])
            ids, lay, nt = np.zeros(nb, np.int64), np.zeros(nb, np.int32), np.zeros(nb, np.int32)
            k, v = np.zeros((nb, B, d), np.float32), np.zeros((nb, B, d), np.float32)
            L.refdrv_workload_blocks(self.h, r, B, _p(ids), _p(lay), _p(nt), _p(k), _p(v))
            lists = []
            for l in range(sp["n_layers"]):
                li = np.zeros(int(info[4]), np.int64)
                L.refdrv_workload_layer_list(self.h, r, l, _p(li))
                lists.append(li)
            qs = np.zeros((int(info[2]), sp["n_layers"], d), np.float32)
            for t in range(int(info[2])):
                for l in range(sp["n_layers"]):
                    L.refdrv_workload_query(self.h, r, t, l, _p(qs[t, l]))
            self.requests.append(dict(request_id=int(info[0]), context=int(info[1]), steps=int(info[2]), ids=ids,
                                      layers=lay, ntok=nt, keys=k, values=v, lists=lists, queries=qs))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.refdrv_workload_destroy(self.h)
            self.h = None


class RefStore:
    def __init__(self, drv: RefDriver, capacity, n_layers, partitioned, fifo, miss_ms):
        self.drv, self.L = drv, drv.L
        self.h = self.L.refdrv_store_create(capacity, n_layers, partitioned, fifo, miss_ms)
        if not self.h:
            raise RuntimeError(drv.error())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.refdrv_store_destroy(self.h)
            self.h = None

    def put(self, block_id, keys, values, layer=0, owner=0):
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        st = self.L.refdrv_put(self.h, block_id, layer, owner, k.shape[0], k.shape[1], _p(k), _p(v))
        if st:
            raise RuntimeError(f"status {st}: {self.drv.error()}")

    def put_many(self, first_id, keys, values, layer=0, owner=0):
        """keys/values [n, ntok, d] fp32."""
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        st = self.L.refdrv_put_many(self.h, k.shape[0], first_id, layer, owner, k.shape[1], k.shape[2], _p(k), _p(v))
        if st:
            raise RuntimeError(f"status {st}: {self.drv.error()}")

    def put_blockset(self, bs: BlockSet, layer=0, owner=0):
        for i in range(bs.n):
            k, v = bs.block(i)
            self.put(int(bs.ids[i]), k, v, layer, owner)

    def release(self, owner) -> int:
        return self.L.refdrv_release(self.h, owner)

    def stats(self):
        out = np.zeros(4, np.uint64)
        self.L.refdrv_stats(self.h, _p(out))
        return dict(zip(("hits", "misses", "evictions", "bytes_transferred"), map(int, out)))

    def layer_stats(self, layer):
        out = np.zeros(4, np.uint64)
        self.L.refdrv_layer_stats(self.h, layer, _p(out))
        return dict(zip(("hits", "misses", "evictions", "bytes_transferred"), map(int, out)))

    def contains(self, block_id):
        r = C.c_int32(-1)
        st = self.L.refdrv_contains(self.h, block_id, C.byref(r))
        return None if st else bool(r.value)

    def enable_trace(self):
        self.L.refdrv_enable_trace(self.h)

    def trace(self) -> str:
        n = self.L.refdrv_trace(self.h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self.L.refdrv_trace(self.h, buf, n + 1)
        return buf.value.decode()

    def query(self, q, ids, cfg: Config, topk: int = 0) -> QueryResult:
        q = np.ascontiguousarray(q, np.float32)
        ids = np.ascontiguousarray(ids, np.int64)
        n = ids.size
        out = np.zeros(q.size, np.float32)
        su = np.zeros(3, np.uint64)
        sf = np.zeros(2, np.float64)
        term = C.c_int32()
        pid = np.zeros(max(n, 1), np.int64)
        it = np.zeros(max(n, 1), np.float64)
        st = self.L.refdrv_query(self.h, _p(q), q.size, _p(ids), n, C.byref(cfg), topk, _p(out), _p(su), _p(sf),
                                 C.byref(term), _p(pid), _p(it))
        if st:
            return QueryResult(out, 0, 0, 0.0, None, False, np.zeros(0, np.int64), status=st)
        bp = int(su[0])
        return QueryResult(out, bp, int(su[1]), float(sf[0]), None if sf[1] < 0 else float(sf[1]),
                           bool(term.value), pid[:bp].copy(), it[: int(su[2])].copy(), 0)

    def pipeline(self, q, ids, cfg: Config, pipelined=True) -> QueryResult:
        q = np.ascontiguousarray(q, np.float32)
        ids = np.ascontiguousarray(ids, np.int64)
        out = np.zeros(q.size, np.float32)
        su = np.zeros(3, np.uint64)
        sf = np.zeros(2, np.float64)
        term = C.c_int32()
        pid = np.zeros(max(ids.size, 1), np.int64)
        st = self.L.refdrv_pipeline(self.h, int(pipelined), _p(q), q.size, _p(ids), ids.size, C.byref(cfg),
                                    _p(out), _p(su), _p(sf), C.byref(term), _p(pid))
        if st:
            raise RuntimeError(self.drv.error())
        bp = int(su[0])
        return QueryResult(out, bp, int(su[1]), float(sf[0]), None if sf[1] < 0 else float(sf[1]),
                           bool(term.value), pid[:bp].copy())

    def multi_head(self, qs, kv_ids, cfg: Config, want_ids=True):
        """qs [hq,d]; kv_ids [hkv,n]. Returns (list[QueryResult], fetched_union)."""
        qs = np.ascontiguousarray(qs, np.float32)
        kv_ids = np.ascontiguousarray(kv_ids, np.int64)
        hq, d = qs.shape
        hkv, n = kv_ids.shape
        outs = np.zeros((hq, d), np.float32)
        su = np.zeros((hq, 3), np.uint64)
        sf = np.zeros((hq, 2), np.float64)
        term = np.zeros(hq, np.int32)
        pid = np.zeros((hq, n), np.int64) if want_ids else None
        uni = np.zeros(hkv * n, np.int64)
        un = C.c_uint64()
        st = self.L.refdrv_multi_head(self.h, _p(qs), hq, d, _p(kv_ids), hkv, n, C.byref(cfg), _p(outs), _p(su),
                                      _p(sf), _p(term), _p(pid) if want_ids else None, _p(uni), C.byref(un))
        if st:
            raise RuntimeError(f"status {st}: {self.drv.error()}")
        res = []
        for h in range(hq):
            bp = int(su[h, 0])
            res.append(QueryResult(outs[h], bp, int(su[h, 1]), float(sf[h, 0]),
                                   None if sf[h, 1] < 0 else float(sf[h, 1]), bool(term[h]),
                                   pid[h, :bp].copy() if want_ids else np.zeros(0, np.int64)))
        return res, uni[: un.value].copy()

    def batched(self, qs, ids, cfg: Config):
        qs = np.ascontiguousarray(qs, np.float32)
        ids = np.ascontiguousarray(ids, np.int64)
        nq, d = qs.shape
        n = ids.shape[1]
        outs = np.zeros((nq, d), np.float32)
        su = np.zeros((nq, 3), np.uint64)
        sf = np.zeros((nq, 2), np.float64)
        term = np.zeros(nq, np.int32)
        rounds = C.c_uint64()
        st = self.L.refdrv_batched(self.h, _p(qs), nq, d, _p(ids), n, C.byref(cfg), _p(outs), _p(su), _p(sf),
                                   _p(term), C.byref(rounds))
        if st:
            raise RuntimeError(self.drv.error())
        return [QueryResult(outs[i], int(su[i, 0]), int(su[i, 1]), float(sf[i, 0]),
                            None if sf[i, 1] < 0 else float(sf[i, 1]), bool(term[i]), np.zeros(0, np.int64))
                for i in range(nq)], int(rounds.value)


def _batched_ragged(self, qs, ids, off, cfg: Config):
    """psa_attention_batched over ragged lists ids[off[i]:off[i+1]]; returns (results with processed ids, rounds)."""
    L = self.L
    L.refdrv_batched_ragged.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                        C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.POINTER(C.c_uint64)]
    qs = np.ascontiguousarray(qs, np.float32)
    ids = np.ascontiguousarray(ids, np.int64)
    off = np.ascontiguousarray(off, np.int64)
    nq, d = qs.shape
    outs = np.zeros((nq, d), np.float32)
    su = np.zeros((nq, 3), np.uint64)
    sf = np.zeros((nq, 2), np.float64)
    term = np.zeros(nq, np.int32)
    pids = np.zeros(ids.size, np.int64)
    rounds = C.c_uint64()
    st = L.refdrv_batched_ragged(self.h, _p(qs), nq, d, _p(ids), _p(off), C.byref(cfg), _p(outs), _p(su), _p(sf),
                                 _p(term), _p(pids), C.byref(rounds))
    if st:
        raise RuntimeError(self.drv.error())
    return [QueryResult(outs[i], int(su[i, 0]), int(su[i, 1]), float(sf[i, 0]),
                        None if sf[i, 1] < 0 else float(sf[i, 1]), bool(term[i]),
                        pids[off[i]: off[i] + int(su[i, 0])].copy()) for i in range(nq)], int(rounds.value)


RefStore.batched_ragged = _batched_ragged


def _load_ids(self, ids):
    self.L.refdrv_load_ids.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    ids = np.ascontiguousarray(ids, np.int64)
    st = self.L.refdrv_load_ids(self.h, _p(ids), ids.size)
    if st:
        raise RuntimeError(self.drv.error())


RefStore.load_ids = _load_ids


def ref_available() -> bool:
    return os.path.exists(REFDRV_SO)
