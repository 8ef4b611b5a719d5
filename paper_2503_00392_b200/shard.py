"""Multi-GPU plumbing for the PSA path: one process per GPU.

(request, layer, kv-head) units share nothing (reference engine.cpp:240-260;
batched == solo, test_engine.cpp:280-327), so the data path has NO collective:
each rank owns whole requests in its own HBM pool. torch.distributed carries
only the benchmark barrier / max-over-ranks timing and the optional final
output gather (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_requests(n_requests: int, world: int, rank: int) -> np.ndarray:
    """Requests owned by `rank`: contiguous, balanced (sizes differ by at most one)."""
    base, extra = divmod(n_requests, world)
    start = rank * base + min(rank, extra)
    return np.arange(start, start + base + (1 if rank < extra else 0), dtype=np.int64)


def shard_kv_heads(n_kv_heads: int, world: int, rank: int) -> np.ndarray:
    """Secondary split when requests < GPUs (config-1-like): kv heads of one request."""
    return shard_requests(n_kv_heads, world, rank)


def unit_ids(requests: np.ndarray, layers: int, kv_heads: int) -> np.ndarray:
    """Global unit id = (request * layers + layer) * kv_heads + kv_head, for each owned request."""
    r = np.asarray(requests, np.int64)[:, None, None]
    l = np.arange(layers, dtype=np.int64)[None, :, None]
    h = np.arange(kv_heads, dtype=np.int64)[None, None, :]
    return ((r * layers + l) * kv_heads + h).reshape(-1)


def plan_units(n_requests: int, layers: int, kv_heads: int, world: int, rank: int) -> np.ndarray:
    """Units (global ids, see unit_ids) owned by `rank` (SURVEY §8e partitioning).

    Primary: whole requests (every layer and kv head of a request on one GPU) when there are at
    least as many requests as ranks. Secondary, when requests < ranks (config-1-like): the
    (request, kv-head) pairs are split contiguously, so each rank owns some kv heads of a request
    with all their layers. Either way every unit is owned by exactly one rank; no collective."""
    if n_requests >= world:
        return unit_ids(shard_requests(n_requests, world, rank), layers, kv_heads)
    pairs = shard_requests(n_requests * kv_heads, world, rank)  # flattened (request, kv head)
    r, h = pairs // kv_heads, pairs % kv_heads
    l = np.arange(layers, dtype=np.int64)
    return ((r[:, None] * layers + l[None, :]) * kv_heads + h[:, None]).reshape(-1)


def resident_layers(requests_on_rank: int, layers: int, kv_heads: int, blocks: int, bytes_per_block: int,
                    budget_bytes: int) -> int:
    """Config 5 (64 x 128K decodes on 2/4 GPUs exceeds HBM, SURVEY §7 hard part 7): how many layers
    of every owned request fit the pool budget; a step then runs those resident layers."""
    per_layer = requests_on_rank * kv_heads * blocks * bytes_per_block
    return int(max(1, min(layers, budget_bytes // max(per_layer, 1))))


def max_over_ranks(x: float, device=None) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_outputs(out: torch.Tensor) -> torch.Tensor:
    """Optional final output gather: every rank's [units, g, d] outputs, concatenated in rank order."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return out
    ws = dist.get_world_size()
    n = torch.tensor([out.shape[0]], dtype=torch.int64, device=out.device)
    sizes = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(sizes, n)
    mx = int(max(int(s.item()) for s in sizes))
    pad = torch.zeros((mx,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    pad[: out.shape[0]] = out
    parts = [torch.empty_like(pad) for _ in range(ws)]
    dist.all_gather(parts, pad)
    return torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)], 0)
