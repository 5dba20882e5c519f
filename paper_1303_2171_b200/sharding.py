"""DeviceB as a group of GPUs: the device-side partitioner and the merges.

One process per GPU (torch.distributed; NCCL over NVLink on the B200 box,
gloo in the CPU tests and the 1-GPU functional runs).  `fraction_a` stays
the host share chosen by the reference's Partitionable.partition
(worksharing.py:264-281); the DeviceB part is split again here into G
contiguous shards, one per rank, and each rank's partial is merged with the
one collective the workload needs:

  histogram   floor(k·n/G) element shards (kernels_regular.py:143)
              → all-reduce of the bin counts;
  row strips  floor(k·rows/G) strips (kernels_regular.py:501) → all-gather of
              the strips (the reference's vstack, :510-511);
  SpMV        equal-nnz row shards found ON THE DEVICE by hb_partition_nnz
              (SpmvWorkload's searchsorted rule, kernels_irregular.py:243-245,
              at k/G) → all-gather of y_perm, un-permute by hb_scatter_perm;
  sort        sample-merge exchange (sort_exchange.py);
  ranking     sublist-split list ranking (kernels_irregular.list_rank_sharded).

Data stays where it lives: CUDA-tensor inputs give CUDA-tensor results and
every collective runs on device memory under NCCL — nothing round-trips
through the host.  Host (numpy) inputs give numpy results.  Under gloo the
collective tensors bounce through host memory (gloo's wire is the host);
the kernels are the same libhb200 calls either way.

Without an active group (the default) the whole GPU share runs on the
calling process's current device.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass
from typing import Any, Callable, Iterator, Sequence

import numpy as np

from .gpu import is_device_array

_active: "ShardGroup | None" = None


@dataclass(frozen=True)
class ShardGroup:
    """A torch.distributed process group whose ranks share the GPU work.
    `device` is where the backend's collectives take their tensors: the
    rank's GPU under NCCL, the host under gloo."""

    group: Any
    rank: int
    world: int
    device: Any


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


def multi(g: "ShardGroup | None" = None) -> bool:
    g = _active if g is None else g
    return g is not None and g.world > 1


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
# Collectives move 32/64-bit unsigned values as their signed bits (the
# backends need not support torch.uint32/uint64); the bits are unchanged.


def _wire_view(t):
    import torch

    if t.dtype == getattr(torch, "uint32", None):
        return t.view(torch.int32)
    if t.dtype == getattr(torch, "uint64", None):
        return t.view(torch.int64)
    return t


def _to_wire(t, g: ShardGroup):
    """`t` as the backend takes it (same storage when already there)."""
    w = _wire_view(t)
    return w if w.device == g.device else w.to(g.device)


def _tensor(x: Any, g: ShardGroup):
    """numpy → torch on the collective device; tensors pass through."""
    import torch

    if isinstance(x, torch.Tensor):
        return x
    return torch.from_numpy(np.ascontiguousarray(x)).to(g.device)


def all_reduce_sum(t, g: ShardGroup):
    """In-place sum across ranks of a tensor (returned; same device as `t`)."""
    import torch.distributed as dist

    w = _to_wire(t, g)
    dist.all_reduce(w, op=dist.ReduceOp.SUM, group=g.group)
    if w.data_ptr() != _wire_view(t).data_ptr():
        _wire_view(t).copy_(w)
    return t


def gather_blocks(local, counts: Sequence[int], g: ShardGroup):
    """Concatenation in rank order of per-rank blocks (dim 0), rank r holding
    counts[r] rows; one all-gather on the wire (padded to the largest block
    when the sizes differ).  Result on `local`'s device."""
    import torch
    import torch.distributed as dist

    counts = [int(c) for c in counts]
    if local.shape[0] != counts[g.rank]:
        raise ValueError(f"rank {g.rank} holds {local.shape[0]} rows, expected {counts[g.rank]}")
    w = _to_wire(local.contiguous(), g)
    tail = tuple(w.shape[1:])
    width = max(counts)
    if width == 0:
        return local[:0].clone()
    if any(c != width for c in counts):
        send = torch.zeros((width,) + tail, dtype=w.dtype, device=w.device)
        send[: counts[g.rank]].copy_(w)
    else:
        send = w
    out = torch.empty((g.world * width,) + tail, dtype=w.dtype, device=w.device)
    dist.all_gather_into_tensor(out, send, group=g.group)
    if any(c != width for c in counts):
        out = torch.cat([out[r * width : r * width + counts[r]] for r in range(g.world)])
    if out.device != local.device:
        out = out.to(local.device)
    return out.view(local.dtype) if out.dtype != local.dtype else out


def all_to_all_v(send, send_counts: Sequence[int], recv_counts: Sequence[int], g: ShardGroup):
    """Variable-size all-to-all of a 1-D tensor; result on `send`'s device."""
    import torch
    import torch.distributed as dist

    w = _to_wire(send.contiguous(), g)
    out = torch.empty(int(sum(recv_counts)), dtype=w.dtype, device=w.device)
    dist.all_to_all_single(out, w, [int(c) for c in recv_counts], [int(c) for c in send_counts], group=g.group)
    if out.device != send.device:
        out = out.to(send.device)
    return out.view(send.dtype) if out.dtype != send.dtype else out


def all_gather_small(t, g: ShardGroup):
    """[world, *t.shape] stack of every rank's (small) tensor."""
    import torch
    import torch.distributed as dist

    w = _to_wire(t.contiguous().reshape((1,) + tuple(t.shape)), g)
    out = torch.empty((g.world,) + tuple(t.shape), dtype=w.dtype, device=w.device)
    dist.all_gather_into_tensor(out, w, group=g.group)  # dim-0 concatenation of [1, ...] blocks
    out = out.to(t.device) if out.device != t.device else out
    return out.view(t.dtype) if out.dtype != t.dtype else out


def gather_rows(mine: Any, bounds: Sequence[int], g: ShardGroup) -> Any:
    """All ranks receive the row blocks [bounds[r], bounds[r+1]) concatenated
    in rank order.  CUDA tensor in → CUDA tensor out (device-resident
    all-gather); numpy in → numpy out."""
    counts = [bounds[k + 1] - bounds[k] for k in range(g.world)]
    if is_device_array(mine):
        return gather_blocks(mine, counts, g)
    t = _tensor(mine, g)
    return gather_blocks(t, counts, g).cpu().numpy()


# ---------------------------------------------------------------- workloads


def run_sharded_histogram(part: Any, bin_count: int, local: Callable | None = None) -> Any:
    """DeviceB histogram share: rank r counts shard r, all-reduce the counts.
    Host part → int64 numpy counts; CUDA part → int64 CUDA tensor."""
    if local is None:
        from .kernels_regular import gpu_histogram as local
    g = _active
    if not multi(g):
        counts = local(part, bin_count)
        return counts if is_device_array(counts) else np.asarray(counts, dtype=np.int64)
    lo, hi = shard_range(_length(part), g.rank, g.world)
    counts = local(part[lo:hi], bin_count)
    t = _tensor(np.asarray(counts, dtype=np.int64) if not is_device_array(counts) else counts, g)
    all_reduce_sum(t, g)
    return t if is_device_array(part) else t.cpu().numpy()


def run_sharded_rows(row0: int, row1: int, local: Callable[[int, int], Any]) -> Any:
    """Row-range share [row0, row1): rank r computes strip r (floor(k·n/G)
    rule), all ranks receive the concatenation (the reference's
    vstack/concatenate merge)."""
    g = _active
    if not multi(g):
        return local(row0, row1)
    bounds = [row0 + b for b in shard_bounds(row1 - row0, g.world)]
    return gather_rows(local(bounds[g.rank], bounds[g.rank + 1]), bounds, g)


def to_numpy(x: Any) -> np.ndarray:
    if is_device_array(x):
        return x.cpu().numpy()
    return np.asarray(x)


def run_sharded_sort(keys: Any, payload: Any = None, local: Callable | None = None):
    """DeviceB sort share.  Single GPU: one LSD radix sort.  GPU group: the
    sample-merge of sort_exchange.py (local sort, splitter all-gather,
    all-to-all, G-way merge); every rank returns the full sorted array."""
    if local is None:
        from .kernels_regular import gpu_sort as local
    g = _active
    if not multi(g):
        return local(keys, payload)
    from .sort_exchange import sample_merge_sort

    return sample_merge_sort(keys, payload, g)
