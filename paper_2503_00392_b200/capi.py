"""ctypes mirror of the C ABI (include/psattn.h, include/psattn_b200.h).

Names, argument meaning and status codes follow the reference's C ABI
(/root/reference/proj/include/psattn.h). Every compute call goes to the CUDA
library ``_lib/libpsattn_b200.so``; there is no Python or CPU fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSATTN_B200_LIB") or os.path.join(_HERE, "_lib", "libpsattn_b200.so")

PSATTN_OK = 0
PSATTN_ERR_INVALID_ARGUMENT = 1
PSATTN_ERR_NOT_FOUND = 2
PSATTN_ERR_RUNTIME = 3

PSATTN_POOL_UNIFIED, PSATTN_POOL_LAYER_PARTITIONED = 0, 1
PSATTN_EVICT_LRU, PSATTN_EVICT_FIFO = 0, 1
PSATTN_EST_MEAN, PSATTN_EST_CUBOID_UPPER, PSATTN_EST_CUBOID_MEAN = 0, 1, 2
PSATTN_RANK_ESTIMATED, PSATTN_RANK_ORACLE = 0, 1
PSATTN_KV_F32, PSATTN_KV_BF16 = 0, 1
PSATTN_METHOD_PSA, PSATTN_METHOD_TOPK, PSATTN_METHOD_EXACT = 0, 1, 2


class StoreOptions(C.Structure):
    _fields_ = [("fast_capacity_slots", C.c_int32), ("n_layers", C.c_int32), ("pool_policy", C.c_int32),
                ("eviction_policy", C.c_int32), ("miss_latency_ms", C.c_double)]


class Config(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("microbatch_size", C.c_int32), ("block_size", C.c_int32),
                ("estimator", C.c_int32), ("ranking_mode", C.c_int32), ("audit_coverage", C.c_int32),
                ("scale_override", C.c_double)]


class RunStats(C.Structure):
    _fields_ = [("blocks_processed", C.c_uint64), ("total_blocks", C.c_uint64), ("estimated_coverage", C.c_double),
                ("true_coverage", C.c_double), ("terminated_early", C.c_int32)]


class CacheStats(C.Structure):
    _fields_ = [("hits", C.c_uint64), ("misses", C.c_uint64), ("evictions", C.c_uint64),
                ("bytes_transferred", C.c_uint64)]


class PoolDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("block_tokens", C.c_int32), ("kv_dtype", C.c_int32), ("reserved", C.c_int32),
                ("n_slots", C.c_int64)]


class PoolLayout(C.Structure):
    _fields_ = [("kv", C.c_void_p), ("meta", C.c_void_p), ("ntok", C.c_void_p), ("slot_bytes", C.c_int64),
                ("meta_bytes", C.c_int64)]


class Batch(C.Structure):
    _fields_ = [("n_units", C.c_int32), ("group", C.c_int32), ("dim", C.c_int32), ("max_blocks", C.c_int32),
                ("total_blocks", C.c_int64),
                ("q", C.c_void_p), ("slots", C.c_void_p), ("list_off", C.c_void_p),
                ("epsilon", C.c_double), ("microbatch_size", C.c_int32), ("estimator", C.c_int32),
                ("ranking_mode", C.c_int32), ("audit_coverage", C.c_int32), ("scale_override", C.c_double),
                ("topk", C.c_int64),
                ("out", C.c_void_p), ("blocks_processed", C.c_void_p), ("est_coverage", C.c_void_p),
                ("true_coverage", C.c_void_p), ("terminated", C.c_void_p), ("ranked_pos", C.c_void_p),
                ("iter_est", C.c_void_p)]


class TradeoffReport(C.Structure):
    _fields_ = [("target_coverage", C.c_double), ("n_queries", C.c_int64), ("max_blocks", C.c_int64),
                ("k_min", C.c_int64), ("worst_coverage_at_kmin", C.c_double),
                ("worst_coverage_below_kmin", C.c_double), ("psa_mean_blocks", C.c_double),
                ("psa_p99_blocks", C.c_double), ("psa_mean_coverage", C.c_double),
                ("block_access_ratio", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class TierDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("block_tokens", C.c_int32), ("kv_dtype", C.c_int32), ("n_layers", C.c_int32),
                ("n_blocks", C.c_int64), ("fast_slots", C.c_int64), ("pool_policy", C.c_int32),
                ("eviction_policy", C.c_int32)]


class ServingCost(C.Structure):
    _fields_ = [("miss_cost_ms", C.c_double), ("hit_cost_ms", C.c_double), ("compute_cost_ms", C.c_double),
                ("overlap", C.c_int32), ("reserved", C.c_int32)]


class ServingReport(C.Structure):
    _fields_ = [("mean_blocks", C.c_double), ("p99_blocks", C.c_double), ("kv_fraction", C.c_double),
                ("mean_coverage", C.c_double), ("min_coverage", C.c_double), ("hit_ratio", C.c_double),
                ("tbt_p50_ms", C.c_double), ("tbt_p99_ms", C.c_double), ("overlap_eff", C.c_double),
                ("store_stats", CacheStats), ("n_calls", C.c_int64), ("n_steps", C.c_int64),
                ("completed_requests", C.c_int64), ("device_batches", C.c_int64), ("sim_time_ms", C.c_double),
                ("gpu_ms", C.c_double)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "store_stats"}
        s = self.store_stats
        d["store_stats"] = dict(hits=s.hits, misses=s.misses, evictions=s.evictions,
                                bytes_transferred=s.bytes_transferred)
        return d


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the PSA path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64, dbl, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
    L.psattn_last_error.restype = C.c_char_p
    L.psattn_version.restype = C.c_char_p
    L.psattn_store_options_default.argtypes = [C.POINTER(StoreOptions)]
    L.psattn_store_create.argtypes = [C.POINTER(StoreOptions), C.POINTER(vp)]
    L.psattn_store_destroy.argtypes = [vp]
    L.psattn_store_put_block.argtypes = [vp, i64, i32, i64, i32, i32, vp, vp]
    L.psattn_store_release_request.argtypes = [vp, i64]
    L.psattn_store_contains.argtypes = [vp, i64, C.POINTER(C.c_int)]
    L.psattn_store_stats.argtypes = [vp, C.POINTER(CacheStats)]
    L.psattn_config_default.argtypes = [C.POINTER(Config)]
    L.psattn_run_query.argtypes = [vp, vp, i32, vp, sz, C.POINTER(Config), vp, C.POINTER(RunStats)]
    L.psattn_run_topk.argtypes = [vp, vp, i32, vp, sz, sz, C.POINTER(Config), vp, C.POINTER(RunStats)]
    L.psattn_run_multi_head.argtypes = [vp, vp, i32, i32, vp, vp, i32, C.POINTER(Config), vp, vp, vp]
    L.psattn_pool_create.argtypes = [C.POINTER(PoolDesc), C.POINTER(vp)]
    L.psattn_pool_destroy.argtypes = [vp]
    L.psattn_pool_get_desc.argtypes = [vp, C.POINTER(PoolDesc)]
    L.psattn_pool_get_layout.argtypes = [vp, C.POINTER(PoolLayout)]
    L.psattn_pool_put_blocks.argtypes = [vp, i64, vp, vp, vp, vp]
    L.psattn_pool_build_metadata.argtypes = [vp, i64, i64, vp]
    L.psattn_pool_read_metadata.argtypes = [vp, i64, vp, vp, vp]
    L.psattn_pool_append_tokens.argtypes = [vp, i32, vp, vp, vp, vp, vp]
    L.psattn_batch_workspace_bytes.argtypes = [C.POINTER(Batch)]
    L.psattn_batch_workspace_bytes.restype = sz
    L.psattn_run_batch.argtypes = [vp, C.POINTER(Batch), vp, vp]
    L.psattn_rank_batch.argtypes = [vp, C.POINTER(Batch), vp, vp]
    L.psattn_batch_union_blocks.argtypes = [C.POINTER(Batch), vp, vp, vp]
    L.psattn_batch_last_launches.argtypes = [C.POINTER(i32)]
    L.psattn_set_progressive_kernel.argtypes = [i32]
    L.psattn_debug_stream_stats.argtypes = [vp]
    L.psattn_debug_stream_prof.argtypes = [vp]
    L.psattn_set_dense_early.argtypes = [C.c_float]
    L.psattn_set_dense_partial.argtypes = [i32]
    L.psattn_debug_gqa_phases.argtypes = [vp]
    L.psattn_debug_stream_attach.argtypes = []
    L.psattn_debug_stream_attach.restype = C.POINTER(C.c_int)
    L.psattn_set_score_kernel.argtypes = [i32]
    L.psattn_set_pipeline.argtypes = [i32]
    L.psattn_profile_enable.argtypes = [i32]
    L.psattn_profile_read.argtypes = [vp, vp, i32]
    L.psattn_set_dense.argtypes = [i32]
    L.psattn_graph_create.argtypes = [vp, C.POINTER(Batch), vp, vp, C.POINTER(vp)]
    L.psattn_graph_launch.argtypes = [vp, vp]
    L.psattn_graph_destroy.argtypes = [vp]
    L.psattn_exact_attention.argtypes = [vp, C.POINTER(Batch), vp, vp]
    L.psattn_criticality_scores.argtypes = [vp, i32, vp, vp, vp, i64, i32, dbl, vp]
    L.psattn_rank_by_scores.argtypes = [vp, vp, i64, vp]
    L.psattn_tradeoff.argtypes = [vp, C.POINTER(Batch), dbl, C.POINTER(TradeoffReport), vp]
    L.psattn_tier_create.argtypes = [C.POINTER(TierDesc), C.POINTER(vp)]
    L.psattn_tier_destroy.argtypes = [vp]
    L.psattn_tier_put_blocks.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp]
    L.psattn_tier_release_request.argtypes = [vp, i64]
    L.psattn_tier_run_batch.argtypes = [vp, C.POINTER(Batch), vp, vp]
    L.psattn_tier_stats.argtypes = [vp, i32, C.POINTER(CacheStats)]
    L.psattn_tier_resident.argtypes = [vp, i64, C.POINTER(i32)]
    L.psattn_tier_h2d_bytes.argtypes = [vp, C.POINTER(u64)]
    L.psattn_tier_pool.argtypes = [vp]
    L.psattn_tier_pool.restype = vp
    L.psattn_serving_create.argtypes = [C.POINTER(TierDesc), C.POINTER(Config), C.POINTER(ServingCost), C.POINTER(vp)]
    L.psattn_serving_destroy.argtypes = [vp]
    L.psattn_serving_add_request.argtypes = [vp, i64, dbl, i32, i32, i64, vp, i64, vp, vp, vp, vp, vp, vp]
    L.psattn_serving_run.argtypes = [vp, i32, dbl, i64, C.POINTER(ServingReport)]
    return L


lib = _load()

# Every function include/psattn.h and include/psattn_b200.h declare.
EXPORTED = [
    "psattn_last_error", "psattn_version", "psattn_store_options_default", "psattn_store_create",
    "psattn_store_destroy", "psattn_store_put_block", "psattn_store_release_request", "psattn_store_contains",
    "psattn_store_stats", "psattn_config_default", "psattn_run_query", "psattn_run_topk",
    "psattn_cmd_run", "psattn_cmd_tradeoff", "psattn_cmd_equivalence",
    "psattn_pool_create", "psattn_pool_destroy", "psattn_pool_get_desc", "psattn_pool_get_layout",
    "psattn_pool_put_blocks", "psattn_pool_build_metadata", "psattn_pool_read_metadata",
    "psattn_pool_append_tokens",
    "psattn_batch_workspace_bytes", "psattn_run_batch", "psattn_batch_union_blocks", "psattn_batch_last_launches",
    "psattn_profile_enable", "psattn_profile_read", "psattn_set_progressive_kernel",
    "psattn_debug_stream_stats", "psattn_debug_stream_prof", "psattn_set_dense_early", "psattn_set_dense_partial", "psattn_debug_gqa_phases", "psattn_debug_stream_attach",
    "psattn_set_score_kernel", "psattn_set_pipeline", "psattn_set_dense",
    "psattn_graph_create", "psattn_graph_launch", "psattn_graph_destroy",
    "psattn_exact_attention", "psattn_tradeoff", "psattn_rank_batch", "psattn_run_multi_head",
    "psattn_criticality_scores", "psattn_rank_by_scores",
    "psattn_tier_create", "psattn_tier_destroy", "psattn_tier_put_blocks", "psattn_tier_release_request",
    "psattn_tier_run_batch", "psattn_tier_stats", "psattn_tier_resident", "psattn_tier_h2d_bytes", "psattn_tier_pool",
    "psattn_serving_create", "psattn_serving_destroy", "psattn_serving_add_request", "psattn_serving_run",
]


def last_error() -> str:
    return lib.psattn_last_error().decode()


class PsattnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != PSATTN_OK:
        raise PsattnError(rc, last_error())


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def store_options_default() -> StoreOptions:
    o = StoreOptions()
    lib.psattn_store_options_default(C.byref(o))
    return o


def config_default(**kw) -> Config:
    c = Config()
    lib.psattn_config_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@dataclass
class QueryOut:
    output: np.ndarray
    blocks_processed: int
    total_blocks: int
    estimated_coverage: float
    true_coverage: float
    terminated_early: bool


class Store:
    """psattn_store: device-resident block store (reference TieredBlockStore via C ABI)."""

    def __init__(self, capacity=256, n_layers=1, policy=PSATTN_POOL_UNIFIED, eviction=PSATTN_EVICT_LRU,
                 miss_latency_ms=0.0):
        o = StoreOptions(capacity, n_layers, policy, eviction, miss_latency_ms)
        self.h = C.c_void_p()
        check(lib.psattn_store_create(C.byref(o), C.byref(self.h)))

    def close(self):
        if lib is not None and getattr(self, "h", None) is not None and self.h.value:
            lib.psattn_store_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def put(self, block_id, keys, values, layer=0, owner=0) -> int:
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        return lib.psattn_store_put_block(self.h, block_id, layer, owner, k.shape[0], k.shape[1], _p(k), _p(v))

    def put_blockset(self, bs, layer=0, owner=0):
        for i in range(bs.n):
            k, v = bs.block(i)
            check(self.put(int(bs.ids[i]), k, v, layer, owner))

    def release(self, owner) -> int:
        return lib.psattn_store_release_request(self.h, owner)

    def contains(self, block_id):
        r = C.c_int(-1)
        rc = lib.psattn_store_contains(self.h, block_id, C.byref(r))
        return rc, bool(r.value)

    def stats(self) -> dict:
        s = CacheStats()
        check(lib.psattn_store_stats(self.h, C.byref(s)))
        return dict(hits=s.hits, misses=s.misses, evictions=s.evictions, bytes_transferred=s.bytes_transferred)

    def _run(self, fn, q, ids, cfg, k=None):
        q = np.ascontiguousarray(q, np.float32)
        ids = np.ascontiguousarray(ids, np.int64)
        out = np.zeros(q.size, np.float32)
        st = RunStats()
        args = [self.h, _p(q), q.size, _p(ids), ids.size]
        if k is not None:
            args.append(k)
        args += [C.byref(cfg) if cfg is not None else None, _p(out), C.byref(st)]
        rc = fn(*args)
        return rc, QueryOut(out, int(st.blocks_processed), int(st.total_blocks), st.estimated_coverage,
                            st.true_coverage, bool(st.terminated_early))

    def run_query(self, q, ids, cfg=None):
        return self._run(lib.psattn_run_query, q, ids, cfg)

    def run_topk(self, q, ids, k, cfg=None):
        return self._run(lib.psattn_run_topk, q, ids, cfg, k)

    def put_many(self, first_id, keys, values, layer=0, owner=0):
        """Blocks keys[i] / values[i] ([n, T, d]) as ids first_id + i."""
        for i in range(keys.shape[0]):
            check(self.put(first_id + i, keys[i], values[i], layer, owner))

    def run_multi_head(self, qs, kv_ids, cfg=None):
        """psattn_run_multi_head (reference psa_attention_multi_head): qs [Hq, d], kv_ids: list of
        Hkv id arrays. Returns (rc, outputs [Hq, d], per-head QueryOut list, fetched-union size)."""
        qs = np.ascontiguousarray(qs, np.float32)
        lists = [np.ascontiguousarray(x, np.int64) for x in kv_ids]
        ids = np.ascontiguousarray(np.concatenate(lists), np.int64)
        off = np.zeros(len(lists) + 1, np.int64)
        off[1:] = np.cumsum([x.size for x in lists])
        out = np.zeros(qs.shape, np.float32)
        st = (RunStats * qs.shape[0])()
        un = C.c_int64(0)
        rc = lib.psattn_run_multi_head(self.h, _p(qs), qs.shape[0], qs.shape[1], _p(ids), _p(off), len(lists),
                                       C.byref(cfg) if cfg is not None else None, _p(out), st, C.byref(un))
        res = [QueryOut(out[h], int(st[h].blocks_processed), int(st[h].total_blocks), st[h].estimated_coverage,
                        st[h].true_coverage, bool(st[h].terminated_early)) for h in range(qs.shape[0])]
        return rc, out, res, int(un.value)


def criticality_scores(q, mean, lo, hi, estimator=2, scale=None) -> np.ndarray:
    """criticality_score (reference src/metadata.cpp:60-72) of every record: mean/lo/hi [n, d]."""
    q = np.ascontiguousarray(q, np.float32)
    arr = [np.ascontiguousarray(x, np.float32).reshape(-1, q.size) for x in (mean, lo, hi)]
    n = arr[0].shape[0]
    scale = 1.0 / np.sqrt(q.size) if scale is None else float(scale)
    out = np.zeros(n, np.float64)
    check(lib.psattn_criticality_scores(_p(q), q.size, _p(arr[0]), _p(arr[1]), _p(arr[2]), n, estimator, scale,
                                        _p(out)))
    return out


def rank_by_scores(scores, block_ids) -> np.ndarray:
    """rank_by_scores (reference src/metadata.cpp:87-96): descending score, ties by block id."""
    s = np.ascontiguousarray(scores, np.float64)
    ids = np.ascontiguousarray(block_ids, np.int64)
    if s.size != ids.size:
        raise ValueError("rank_by_scores: scores and block ids differ in length")
    out = np.zeros(s.size, np.int64)
    check(lib.psattn_rank_by_scores(_p(s), _p(ids), s.size, _p(out)))
    return out


def rank_blocks(q, mean, lo, hi, block_ids, estimator=2, scale=None) -> np.ndarray:
    """rank_blocks (reference src/metadata.cpp:74-85)."""
    if len(block_ids) == 0:
        raise ValueError("rank_blocks: empty metadata list")
    return rank_by_scores(criticality_scores(q, mean, lo, hi, estimator, scale), block_ids)


class Serving:
    """psattn_serving: the batched FCFS serving loop over the two-tier store (reference run_serving)."""

    def __init__(self, store: TierDesc, engine: Config, cost: ServingCost):
        self.h = C.c_void_p()
        check(lib.psattn_serving_create(C.byref(store), C.byref(engine), C.byref(cost), C.byref(self.h)))

    def close(self):
        if lib is not None and getattr(self, "h", None) is not None and self.h.value:
            lib.psattn_serving_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def add_request(self, request_id, arrival_s, steps, layer_blocks, block_ids, block_layers, ntok, keys, values,
                    queries):
        lb = np.ascontiguousarray(layer_blocks, np.int64)
        ids = np.ascontiguousarray(block_ids, np.int64)
        ly = np.ascontiguousarray(block_layers, np.int32)
        nt = np.ascontiguousarray(ntok, np.int32)
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        check(lib.psattn_serving_add_request(self.h, request_id, arrival_s, steps, lb.shape[0], lb.shape[1], _p(lb),
                                             ids.size, _p(ids), _p(ly), _p(nt), _p(k), _p(v), _p(q)))

    def run(self, method: int, epsilon: float = 0.95, k: int = 0) -> dict:
        rep = ServingReport()
        check(lib.psattn_serving_run(self.h, method, epsilon, k, C.byref(rep)))
        return rep.as_dict()
