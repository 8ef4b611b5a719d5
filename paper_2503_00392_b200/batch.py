"""torch-tensor helpers around the device-batched C ABI (include/psattn_b200.h).

torch provides device memory and the stream; every kernel launched here is one
of ours (libpsattn_b200.so). Nothing in this module computes attention.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import capi
from .capi import Batch, PoolDesc, PoolLayout, check, lib


def _stream_ptr(stream) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dp(t: torch.Tensor | None) -> C.c_void_p | None:
    return None if t is None else C.c_void_p(t.data_ptr())


class DevicePool:
    """psattn_pool: the unified paged KV block pool in HBM (slots shared by all layers)."""

    def __init__(self, dim: int, block_tokens: int, kv_dtype: int, n_slots: int):
        d = PoolDesc(dim, block_tokens, kv_dtype, 0, n_slots)
        self.h = C.c_void_p()
        check(lib.psattn_pool_create(C.byref(d), C.byref(self.h)))
        self.dim, self.block_tokens, self.kv_dtype, self.n_slots = dim, block_tokens, kv_dtype, n_slots

    def close(self):
        if lib is not None and getattr(self, "h", None) is not None and self.h.value:
            lib.psattn_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def layout(self) -> PoolLayout:
        lay = PoolLayout()
        check(lib.psattn_pool_get_layout(self.h, C.byref(lay)))
        return lay

    def put_blocks(self, slots, ntok, keys, values):
        s = np.ascontiguousarray(slots, np.int32)
        n = np.ascontiguousarray(ntok, np.int32)
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        check(lib.psattn_pool_put_blocks(self.h, s.size, capi._p(s), capi._p(n), capi._p(k), capi._p(v)))

    def build_metadata(self, s0, s1, stream=None):
        check(lib.psattn_pool_build_metadata(self.h, s0, s1, _stream_ptr(stream)))

    def append_tokens(self, tail_slots: torch.Tensor, keys: torch.Tensor, values: torch.Tensor, stream=None) -> int:
        """One decode step's KV append (device tensors): int32 [n] tail slots, fp32 [n, dim] K and V.
        Returns 1 if some tail slot was already full (that sequence's token was not written)."""
        status = torch.zeros(1, dtype=torch.int32, device=keys.device)
        check(lib.psattn_pool_append_tokens(self.h, int(tail_slots.numel()), _dp(tail_slots.contiguous()),
                                            _dp(keys.contiguous()), _dp(values.contiguous()), _dp(status),
                                            _stream_ptr(stream)))
        return int(status.item())

    def read_metadata(self, slot):
        m, lo, hi = (np.zeros(self.dim, np.float32) for _ in range(3))
        check(lib.psattn_pool_read_metadata(self.h, slot, capi._p(m), capi._p(lo), capi._p(hi)))
        return m, lo, hi


class DeviceTier:
    """psattn_tier: pinned-host backing tier + HBM fast tier (LRU/FIFO, unified or layer-partitioned)
    with the reference TieredBlockStore's accounting. Batches over it take block indices as slots."""

    def __init__(self, dim, block_tokens, kv_dtype, n_layers, n_blocks, fast_slots,
                 policy=capi.PSATTN_POOL_UNIFIED, eviction=capi.PSATTN_EVICT_LRU):
        d = capi.TierDesc(dim, block_tokens, kv_dtype, n_layers, n_blocks, fast_slots, policy, eviction)
        self.t = C.c_void_p()
        check(lib.psattn_tier_create(C.byref(d), C.byref(self.t)))
        self.h = C.c_void_p(lib.psattn_tier_pool(self.t))
        self.dim, self.block_tokens, self.n_layers = dim, block_tokens, n_layers

    def close(self):
        if lib is not None and getattr(self, "t", None) is not None and self.t.value:
            lib.psattn_tier_destroy(self.t)
            self.t = None

    def __del__(self):
        self.close()

    def put_blocks(self, blocks, layers, ntok, keys, values, owners=None):
        b = np.ascontiguousarray(blocks, np.int64)
        ly = np.ascontiguousarray(layers, np.int32)
        nt = np.ascontiguousarray(ntok, np.int32)
        ow = None if owners is None else np.ascontiguousarray(owners, np.int64)
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        check(lib.psattn_tier_put_blocks(self.t, b.size, capi._p(b), capi._p(ly), capi._p(nt),
                                         None if ow is None else capi._p(ow), capi._p(k), capi._p(v)))

    def release(self, owner):
        check(lib.psattn_tier_release_request(self.t, owner))

    def stats(self, layer=-1) -> dict:
        s = capi.CacheStats()
        check(lib.psattn_tier_stats(self.t, layer, C.byref(s)))
        return dict(hits=s.hits, misses=s.misses, evictions=s.evictions, bytes_transferred=s.bytes_transferred)

    def resident_slot(self, block) -> int:
        out = C.c_int32()
        check(lib.psattn_tier_resident(self.t, block, C.byref(out)))
        return out.value

    def h2d_bytes(self) -> int:
        out = C.c_uint64()
        check(lib.psattn_tier_h2d_bytes(self.t, C.byref(out)))
        return out.value


@dataclass
class BatchConfig:
    epsilon: float = 0.95
    microbatch_size: int = 1
    estimator: int = capi.PSATTN_EST_CUBOID_MEAN
    ranking_mode: int = capi.PSATTN_RANK_ESTIMATED
    audit_coverage: int = 0
    scale_override: float = 0.0
    topk: int = 0


class BatchRun:
    """One psattn_batch: device page tables + outputs + workspace, launched on a torch stream."""

    def __init__(self, pool: DevicePool, q: torch.Tensor, slots: torch.Tensor, list_off: torch.Tensor,
                 max_blocks: int, cfg: BatchConfig, want_ranked: bool = False, want_iter: bool = False):
        assert q.is_cuda and q.dtype == torch.float32 and q.dim() == 3
        assert slots.dtype == torch.int32 and list_off.dtype == torch.int64
        self.pool = pool
        self.n_units, self.group, self.dim = q.shape
        self.total = int(slots.numel())
        dev = q.device
        nq = self.n_units * self.group
        self.q, self.slots, self.list_off = q.contiguous(), slots.contiguous(), list_off.contiguous()
        self.out = torch.empty((self.n_units, self.group, self.dim), dtype=torch.float32, device=dev)
        self.bp = torch.empty(nq, dtype=torch.int64, device=dev)
        self.est = torch.empty(nq, dtype=torch.float64, device=dev)
        self.tcov = torch.empty(nq, dtype=torch.float64, device=dev)
        self.term = torch.empty(nq, dtype=torch.int32, device=dev)
        self.ranked = torch.empty(self.total * self.group, dtype=torch.int32, device=dev) if want_ranked else None
        self.iest = torch.empty(self.total * self.group, dtype=torch.float64, device=dev) if want_iter else None
        b = Batch()
        b.n_units, b.group, b.dim, b.max_blocks, b.total_blocks = self.n_units, self.group, self.dim, max_blocks, \
            self.total
        b.q, b.slots, b.list_off = _dp(self.q), _dp(self.slots), _dp(self.list_off)
        b.epsilon, b.microbatch_size, b.estimator = cfg.epsilon, cfg.microbatch_size, cfg.estimator
        b.ranking_mode, b.audit_coverage, b.scale_override, b.topk = cfg.ranking_mode, cfg.audit_coverage, \
            cfg.scale_override, cfg.topk
        b.out, b.blocks_processed, b.est_coverage = _dp(self.out), _dp(self.bp), _dp(self.est)
        b.true_coverage, b.terminated = _dp(self.tcov), _dp(self.term)
        b.ranked_pos, b.iter_est = _dp(self.ranked), _dp(self.iest)
        self.b = b
        ws = int(lib.psattn_batch_workspace_bytes(C.byref(b)))
        self.ws = torch.empty(max(ws, 256), dtype=torch.uint8, device=dev)
        self.union = torch.zeros(self.n_units, dtype=torch.int64, device=dev)

    def run(self, stream=None) -> int:
        if isinstance(self.pool, DeviceTier):
            check(lib.psattn_tier_run_batch(self.pool.t, C.byref(self.b), _dp(self.ws), _stream_ptr(stream)))
        else:
            check(lib.psattn_run_batch(self.pool.h, C.byref(self.b), _dp(self.ws), _stream_ptr(stream)))
        n = C.c_int32()
        lib.psattn_batch_last_launches(C.byref(n))
        return n.value

    def capture(self, stream=None):
        """Records this batch's launch sequence as a CUDA graph; run_graph() replays it."""
        self.graph = C.c_void_p()
        check(lib.psattn_graph_create(self.pool.h, C.byref(self.b), _dp(self.ws), _stream_ptr(stream),
                                      C.byref(self.graph)))

    def run_graph(self, stream=None) -> int:
        check(lib.psattn_graph_launch(self.graph, _stream_ptr(stream)))
        n = C.c_int32()
        lib.psattn_batch_last_launches(C.byref(n))
        return n.value

    def __del__(self):
        if lib is not None and getattr(self, "graph", None) is not None and self.graph.value:
            lib.psattn_graph_destroy(self.graph)
            self.graph = None

    def union_blocks(self, stream=None) -> torch.Tensor:
        check(lib.psattn_batch_union_blocks(C.byref(self.b), _dp(self.ws), _dp(self.union), _stream_ptr(stream)))
        return self.union

    def exact_attention(self, stream=None) -> torch.Tensor:
        """fp64 exact attention over every block of each list (reference exact_attention_blocks)."""
        out = torch.empty((self.n_units, self.group, self.dim), dtype=torch.float64, device=self.q.device)
        check(lib.psattn_exact_attention(self.pool.h, C.byref(self.b), _dp(out), _stream_ptr(stream)))
        return out

    def tradeoff(self, target: float, stream=None) -> dict:
        """Reference run_tradeoff on device: k_min of a uniform top-k vs PSA at epsilon = target."""
        rep = capi.TradeoffReport()
        check(lib.psattn_tradeoff(self.pool.h, C.byref(self.b), target, C.byref(rep), _stream_ptr(stream)))
        return rep.as_dict()
