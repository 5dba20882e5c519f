"""Multi-GPU sample-merge sort (the one exchange step of the sort path,
SURVEY §8e; the reference's single-node analogue is the splitter binning +
concatenation of sample_sort_hybrid, kernels_regular.py:264-310).

With G ranks, each holding a shard of keys plus their global indices:
  1. local LSD radix sort (hb_sort) of (key, index) — stable;
  2. S regular samples per rank, all-gathered; G-1 splitters picked at the
     equal-mass positions of the sorted sample set.  Splitters are
     (key, global index) pairs, so ties between equal keys on different ranks
     split exactly where a stable sort puts them;
  3. split points of the local run at the splitters (hb_sort_bounds);
  4. all-to-all of the key / index ranges (NCCL over NVLink on the box);
  5. stable local sort of the received runs (runs arrive in rank order, which
     is the original order of equal keys, so the result is the stable order).
Rank r ends with the r-th splitter interval of the globally sorted sequence.

Indices travel as int32 (the uint32 payload slot of hb_sort; n < 2^31).
The per-rank compute is injected (`local_sort`, `split_points`) so the
exchange logic is covered by world-size-2 gloo tests on CPU.
"""

from __future__ import annotations

from typing import Any, Callable

import numpy as np

from .sharding import ShardGroup, shard_bounds

SAMPLES_PER_RANK = 256


def gpu_local_sort(keys, idx):
    from .kernels_regular import gpu_sort

    k, v, _ = gpu_sort(keys, idx)
    return k, v


def gpu_split_points(keys, idx, probe_k, probe_i):
    import torch

    from . import _lib
    from .gpu import current_stream_handle, vp
    from .kernels_regular import _SORT_CODES

    out = torch.empty(probe_k.numel(), dtype=torch.int64, device=keys.device)
    code = _SORT_CODES[np.dtype(str(keys.dtype).replace("torch.", ""))]
    _lib.call(
        "hb_sort_bounds", vp(keys.data_ptr()), code, vp(idx.data_ptr()), keys.numel(),
        vp(probe_k.data_ptr()), vp(probe_i.data_ptr()), probe_k.numel(), vp(out.data_ptr()),
        _lib.HB_DEVICE_PTRS, current_stream_handle(keys),
    )
    return out


def host_local_sort(keys, idx):
    """CPU stand-in (tests): stable sort of (key, index) tensors."""
    import torch

    order = np.argsort(keys.numpy(), kind="stable")
    return keys[torch.from_numpy(order)], idx[torch.from_numpy(order)]


def host_split_points(keys, idx, probe_k, probe_i):
    """CPU stand-in (tests): lexicographic lower bounds."""
    import torch

    k, v = keys.numpy(), idx.numpy()
    out = []
    for a, b in zip(probe_k.numpy().tolist(), probe_i.numpy().tolist()):
        lo = int(np.searchsorted(k, a, side="left"))
        hi = int(np.searchsorted(k, a, side="right"))
        out.append(lo + int(np.searchsorted(v[lo:hi], b, side="left")))
    return torch.tensor(out, dtype=torch.int64)


def _wire(t):
    """Collectives move 32-bit unsigned keys as their int32 bits (NCCL/gloo
    need not support torch.uint32); the key order is unaffected."""
    import torch

    return t.view(torch.int32) if t.dtype == torch.uint32 else t


def sample_positions(n: int, samples: int):
    """Regular sample positions round(j·(n-1)/(samples-1)), j = 0..samples-1,
    in exact integer arithmetic (a float32 linspace rounds n-1 up past the
    end of the array once n >= 2^24)."""
    import torch

    j = torch.arange(samples, dtype=torch.int64)
    if samples == 1:
        return torch.zeros(1, dtype=torch.int64)
    return (2 * j * (n - 1) + (samples - 1)) // (2 * (samples - 1))


def exchange_sort(
    keys: Any,
    idx: Any,
    g: ShardGroup,
    local_sort: Callable = gpu_local_sort,
    split_points: Callable = gpu_split_points,
    samples: int = SAMPLES_PER_RANK,
):
    """Distributed stable sort of sharded (keys, int32 global index) tensors.
    Returns this rank's (keys, idx) range of the global order."""
    import torch
    import torch.distributed as dist

    keys, idx = local_sort(keys, idx)
    n = keys.numel()
    if n:
        pick = sample_positions(n, samples).to(keys.device)
        sk, si = _wire(keys)[pick].to(torch.int64), idx[pick].to(torch.int64)
        if keys.dtype == torch.uint32:
            sk = sk & 0xFFFFFFFF  # the unsigned key value
        ok = torch.ones(samples, dtype=torch.int64, device=keys.device)
    else:
        sk = si = ok = torch.zeros(samples, dtype=torch.int64, device=keys.device)
    packed = torch.stack([sk, si, ok]).to(g.device)
    gathered = [torch.empty_like(packed) for _ in range(g.world)]
    dist.all_gather(gathered, packed, group=g.group)
    allp = torch.cat(gathered, dim=1).cpu().numpy()
    allp = allp[:, allp[2] == 1]
    order = np.lexsort((allp[1], allp[0]))
    sk_all, si_all = allp[0][order], allp[1][order]
    m = sk_all.size
    picks = [min(m - 1, (j * m) // g.world) for j in range(1, g.world)] if m else []
    pk64 = sk_all[picks].astype(np.int64)
    if keys.dtype == torch.uint32:  # back to the int32 bits, moved, then viewed as u32
        probe_k = torch.from_numpy(pk64.astype(np.uint32).view(np.int32)).to(keys.device).view(torch.uint32)
    else:
        probe_k = torch.from_numpy(pk64).to(keys.dtype).to(keys.device)
    probe_i = torch.from_numpy(si_all[picks].astype(np.int64)).to(idx.dtype).to(keys.device)
    if n and picks:
        cuts = split_points(keys, idx, probe_k, probe_i).to(torch.int64).cpu().tolist()
    else:
        cuts = [0 if not n else n] * (g.world - 1)
    bounds = [0] + list(cuts) + [n]
    send = [bounds[j + 1] - bounds[j] for j in range(g.world)]
    sc = torch.tensor(send, dtype=torch.int64, device=g.device)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=g.group)
    recv = rc.cpu().tolist()
    k_out = torch.empty(sum(recv), dtype=_wire(keys).dtype, device=g.device)
    i_out = torch.empty(sum(recv), dtype=idx.dtype, device=g.device)
    dist.all_to_all_single(k_out, _wire(keys.contiguous()).to(g.device), recv, send, group=g.group)
    dist.all_to_all_single(i_out, idx.contiguous().to(g.device), recv, send, group=g.group)
    return local_sort(k_out.to(keys.device).view(keys.dtype), i_out.to(keys.device))


def sample_merge_sort(keys: Any, payload: Any, g: ShardGroup, local_sort: Callable | None = None,
                      split_points: Callable | None = None):
    """API form (replicated input → replicated output): shard by floor(k·n/G),
    exchange_sort, all-gather the ranges.  Returns (keys, payload, passes)
    like gpu_sort (payload None sorts keys only)."""
    import torch
    import torch.distributed as dist

    from .gpu import is_device_array

    local_sort = local_sort or gpu_local_sort
    split_points = split_points or gpu_split_points
    host_in = not is_device_array(keys)
    dev = torch.device("cpu") if g.device.type == "cpu" else g.device
    k_t = torch.from_numpy(np.ascontiguousarray(keys)).to(dev) if host_in else keys
    n = k_t.numel()
    b = shard_bounds(n, g.world)
    lo, hi = b[g.rank], b[g.rank + 1]
    gidx = torch.arange(lo, hi, dtype=torch.int32).to(dev)
    mk, mi = exchange_sort(k_t[lo:hi].contiguous(), gidx, g, local_sort, split_points)
    cnt = torch.tensor([mk.numel()], dtype=torch.int64, device=g.device)
    cnts = [torch.empty_like(cnt) for _ in range(g.world)]
    dist.all_gather(cnts, cnt, group=g.group)
    sizes = [int(c.item()) for c in cnts]
    width = max(sizes)
    pk = torch.zeros(width, dtype=_wire(mk).dtype, device=g.device)
    pi = torch.zeros(width, dtype=mi.dtype, device=g.device)
    pk[: mk.numel()] = _wire(mk).to(g.device)
    pi[: mi.numel()] = mi.to(g.device)
    gk = [torch.empty_like(pk) for _ in range(g.world)]
    gi = [torch.empty_like(pi) for _ in range(g.world)]
    dist.all_gather(gk, pk, group=g.group)
    dist.all_gather(gi, pi, group=g.group)
    out_k = torch.cat([gk[r][: sizes[r]] for r in range(g.world)]).view(mk.dtype)
    order = torch.cat([gi[r][: sizes[r]] for r in range(g.world)]).to(torch.int64)
    out_p = None
    if payload is not None:
        p_t = torch.from_numpy(np.ascontiguousarray(payload)) if not is_device_array(payload) else payload
        out_p = p_t[order.to(p_t.device)]
    if host_in:
        out_k = out_k.cpu().numpy()
        out_p = out_p.cpu().numpy() if out_p is not None else None
    elif out_k.device != keys.device:
        out_k = out_k.to(keys.device)
    constant = n > 0 and bool(out_k[0] == out_k[-1])
    return out_k, out_p, 0 if constant else 1
