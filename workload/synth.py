"""ctypes binding of the seekable synthetic generator (workload/psattn_synth.h).

Host functions come from ``libpsattn_synth_host.so`` (no CUDA: the reference arm of the
benchmark builds its CPU inputs with it and never maps the product library); the device
pool fill from ``libpsattn_synth_dev.so``, which takes the pool's raw layout and leaves the
metadata build to the product (psattn_pool_build_metadata).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_lib")


class SynthParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("dim", C.c_int32), ("block_tokens", C.c_int32), ("skew", C.c_float),
                ("planted_prob", C.c_float), ("round_bf16", C.c_int32), ("reserved", C.c_int32)]


def _bind(L):
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    P = C.POINTER(SynthParams)
    L.psattn_synth_direction.argtypes = [P, i64, vp]
    L.psattn_synth_query.argtypes = [P, i64, i32, vp]
    L.psattn_synth_unit_host.argtypes = [P, i64, i64, i64, i64, vp, vp]
    L.psattn_synth_is_planted.argtypes = [P, i64, i64]
    if hasattr(L, "psattn_synth_fill"):
        L.psattn_synth_fill.argtypes = [P, vp, vp, i64, i32, i64, i32, vp, vp, vp, vp]
    return L


def _load(name):
    path = os.path.join(_LIB, name)
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `make -C workload` (or __graft_entry__.build())")
    return _bind(C.CDLL(path))


host = _load("libpsattn_synth_host.so")
_dev = None


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def params(seed=1, dim=128, block_tokens=16, skew=8.0, planted_prob=0.0, round_bf16=1) -> SynthParams:
    return SynthParams(seed, dim, block_tokens, skew, planted_prob, round_bf16, 0)


def query(p: SynthParams, unit_id: int, head: int) -> np.ndarray:
    out = np.zeros(p.dim, np.float32)
    host.psattn_synth_query(C.byref(p), unit_id, head, _p(out))
    return out


def direction(p: SynthParams, unit_id: int) -> np.ndarray:
    out = np.zeros(p.dim, np.float32)
    host.psattn_synth_direction(C.byref(p), unit_id, _p(out))
    return out


def unit_host(p: SynthParams, unit_id: int, n_tokens: int, first_block=0, n_blocks=None):
    """Host copy of a unit's K/V blocks: arrays [n_blocks, block_tokens, dim] (zero past n_tokens)."""
    T = p.block_tokens
    nb_total = (n_tokens + T - 1) // T
    n_blocks = nb_total - first_block if n_blocks is None else n_blocks
    k = np.zeros((n_blocks, T, p.dim), np.float32)
    v = np.zeros((n_blocks, T, p.dim), np.float32)
    host.psattn_synth_unit_host(C.byref(p), unit_id, first_block, n_blocks, n_tokens, _p(k), _p(v))
    return k, v


def is_planted(p: SynthParams, unit_id: int, block: int) -> bool:
    return bool(host.psattn_synth_is_planted(C.byref(p), unit_id, block))


def fill(pool, p: SynthParams, unit_ids, slot_off, tokens, stream=None):
    """Writes the units' blocks into a DevicePool (paper_2503_00392_b200.batch) and builds their
    metadata with the product's own kernel (psattn_pool_build_metadata)."""
    global _dev
    import torch
    if _dev is None:
        _dev = _load("libpsattn_synth_dev.so")
    if p.dim != pool.dim or p.block_tokens != pool.block_tokens:
        raise ValueError("synth params do not match the pool")
    u = np.ascontiguousarray(unit_ids, np.int64)
    s = np.ascontiguousarray(slot_off, np.int64)
    t = np.ascontiguousarray(tokens, np.int64)
    if u.size == 0:
        return
    lay = pool.layout()
    st = stream if stream is not None else torch.cuda.current_stream()
    sp = C.c_void_p(st.cuda_stream)
    rc = _dev.psattn_synth_fill(C.byref(p), C.c_void_p(lay.kv), C.c_void_p(lay.ntok), lay.slot_bytes, pool.kv_dtype,
                                pool.n_slots, u.size, _p(u), _p(s), _p(t), sp)
    if rc != 0:
        raise RuntimeError(f"psattn_synth_fill failed (cudaError {rc})")
    nb = (t + p.block_tokens - 1) // p.block_tokens
    lo, hi = int(s.min()), int((s + nb).max())
    pool.build_metadata(lo, hi, stream=st)
    st.synchronize()
