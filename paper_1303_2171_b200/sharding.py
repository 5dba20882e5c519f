"""Device-side partitioner for the GPU share across a group of GPUs.

One process per GPU (torch.distributed; NCCL over NVLink on the B200 box,
gloo in the CPU tests).  `fraction_a` stays the host share chosen by the
reference's Partitionable.partition; the DeviceB part is split again here
into G contiguous shards, one per rank, with the reference's own rounding
rule floor(k·n/G) (kernels_regular.py:143, :501), and the per-rank partials
are merged with the one collective each workload really needs
(SURVEY §8e): histogram → all-reduce of 256 counts; row-sharded outputs →
all-gather of the strips; sort → sample-merge exchange (sort_exchange.py).

Without an active group (the default) the whole GPU share runs on the
calling process's current device.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass
from typing import Any, Callable, Iterator

import numpy as np

from .gpu import is_device_array

_active: "ShardGroup | None" = None


@dataclass(frozen=True)
class ShardGroup:
    """A torch.distributed process group whose ranks share the GPU work."""

    group: Any
    rank: int
    world: int
    device: Any  # torch.device the collectives run on ("cuda:i" for NCCL, "cpu" for gloo)


def shard_bounds(n: int, world: int) -> list[int]:
    """G+1 boundaries floor(k·n/G), k = 0..G (reference strip rule)."""
    return [(k * n) // world for k in range(world + 1)]


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    b = shard_bounds(n, world)
    return b[rank], b[rank + 1]


def active_group() -> "ShardGroup | None":
    return _active


def set_group(group: "ShardGroup | None") -> None:
    global _active
    _active = group


def group_from_default() -> "ShardGroup | None":
    """ShardGroup over torch.distributed's default group (None if world == 1)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return None
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    return ShardGroup(dist.group.WORLD, dist.get_rank(), dist.get_world_size(), dev)


@contextlib.contextmanager
def gpu_group(group: "ShardGroup | None") -> Iterator["ShardGroup | None"]:
    prev = _active
    set_group(group)
    try:
        yield group
    finally:
        set_group(prev)


def _length(part: Any) -> int:
    return int(part.numel() if is_device_array(part) else len(part))


# ---------------------------------------------------------------- collectives


def allreduce_sum_i64(counts: np.ndarray, g: ShardGroup) -> np.ndarray:
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int64)).to(g.device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=g.group)
    return t.cpu().numpy()


def allgather_rows(local: np.ndarray, bounds: list[int], g: ShardGroup) -> np.ndarray:
    """Concatenate per-rank row blocks (unequal sizes) in rank order."""
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local)
    tail = local.shape[1:]
    row_elems = int(np.prod(tail)) if tail else 1
    width = max(bounds[k + 1] - bounds[k] for k in range(g.world)) * row_elems
    send = torch.zeros(width, dtype=_torch_dtype(local.dtype), device=g.device)
    flat = torch.from_numpy(local.reshape(-1))
    send[: flat.numel()] = flat.to(g.device)
    recv = [torch.empty_like(send) for _ in range(g.world)]
    dist.all_gather(recv, send, group=g.group)
    pieces = [recv[k][: (bounds[k + 1] - bounds[k]) * row_elems].cpu().numpy() for k in range(g.world)]
    out = np.concatenate(pieces)
    return out.reshape((bounds[-1] - bounds[0],) + tail)


def _torch_dtype(dt: np.dtype):
    import torch

    return {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
            np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
            np.dtype(np.uint8): torch.uint8}[np.dtype(dt)]


# ---------------------------------------------------------------- workloads


def run_sharded_histogram(part: Any, bin_count: int, local: Callable | None = None) -> np.ndarray:
    """DeviceB histogram share: rank r counts shard r, all-reduce the counts."""
    if local is None:
        from .kernels_regular import gpu_histogram as local
    g = _active
    if g is None or g.world == 1:
        return np.asarray(to_numpy(local(part, bin_count)), dtype=np.int64)
    lo, hi = shard_range(_length(part), g.rank, g.world)
    counts = np.asarray(to_numpy(local(part[lo:hi], bin_count)), dtype=np.int64)
    return allreduce_sum_i64(counts, g)


def run_sharded_rows(row0: int, row1: int, local: Callable[[int, int], np.ndarray]) -> np.ndarray:
    """Row-range share [row0, row1): rank r computes its strip, all ranks
    receive the concatenation (the reference's vstack/concatenate merge)."""
    g = _active
    if g is None or g.world == 1:
        return to_numpy(local(row0, row1))
    bounds = [row0 + b for b in shard_bounds(row1 - row0, g.world)]
    mine = to_numpy(local(bounds[g.rank], bounds[g.rank + 1]))
    return allgather_rows(mine, bounds, g)


def to_numpy(x: Any) -> np.ndarray:
    if is_device_array(x):
        return x.cpu().numpy()
    return np.asarray(x)


def run_sharded_sort(keys: Any, payload: Any = None, local: Callable | None = None):
    """DeviceB sort share.  Single GPU: one LSD radix sort.  GPU group: the
    sample-merge of sort_exchange.py (local sort, splitter all-gather,
    all-to-all, local merge); every rank returns the full sorted array."""
    if local is None:
        from .kernels_regular import gpu_sort as local
    g = _active
    if g is None or g.world == 1:
        return local(keys, payload)
    from .sort_exchange import sample_merge_sort

    return sample_merge_sort(keys, payload, g, local)
