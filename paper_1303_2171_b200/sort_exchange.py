"""Multi-GPU sample-merge sort (the one exchange step of the sort path,
SURVEY §8e; the reference's single-node analogue is the splitter binning +
concatenation of sample_sort_hybrid, kernels_regular.py:264-310).

With G ranks, each holding a shard of keys plus their global indices (the
shards are contiguous index ranges in rank order):
  1. local LSD radix sort (hb_sort) of (key, index) — stable;
  2. S regular samples per rank, all-gathered on the device; G-1 splitters
     at the equal-mass positions of the sorted sample set.  Splitters are
     (key, global index) pairs, so ties between equal keys on different ranks
     split exactly where a stable sort puts them;
  3. split points of the local run at the splitters (hb_sort_bounds);
  4. all-to-all of the key / index ranges (NCCL over NVLink on the box);
  5. G-way stable merge of the received runs (hb_merge_runs): the runs
     arrive in rank order, and a run-order tie break is the original order
     of equal keys, so the result is the stable order.
Rank r ends with the r-th splitter interval of the globally sorted
sequence — the sort's natural, distributed output.  `sample_merge_sort`
(the API form) additionally all-gathers the intervals so that every rank
returns the whole sorted array, like the reference's single return value.

Indices travel as int32 (the uint32 payload slot of hb_sort; n < 2^31).
The per-rank compute is injected (`local_sort`, `split_points`,
`merge_runs`) so the exchange logic is covered by gloo tests on CPU.
"""

from __future__ import annotations

from typing import Any, Callable

import numpy as np

from .sharding import ShardGroup, all_gather_small, all_to_all_v, gather_blocks, shard_bounds

SAMPLES_PER_RANK = 256


# ---------------------------------------------------------------- per-rank compute (GPU)
def gpu_local_sort(keys, idx):
    from .kernels_regular import gpu_sort

    k, v, _ = gpu_sort(keys, idx)
    return k, v


def _key_code(keys) -> int:
    from .kernels_regular import _SORT_CODES

    return _SORT_CODES[np.dtype(str(keys.dtype).replace("torch.", ""))]


def gpu_split_points(keys, idx, probe_k, probe_i):
    import torch

    from . import _lib
    from .gpu import current_stream_handle, vp

    out = torch.empty(probe_k.numel(), dtype=torch.int64, device=keys.device)
    _lib.call(
        "hb_sort_bounds", vp(keys.data_ptr()), _key_code(keys), vp(idx.data_ptr()), keys.numel(),
        vp(probe_k.data_ptr()), vp(probe_i.data_ptr()), probe_k.numel(), vp(out.data_ptr()),
        _lib.HB_DEVICE_PTRS, current_stream_handle(keys),
    )
    return out


def gpu_merge_runs(keys, idx, counts):
    """Stable merge of the back-to-back sorted runs (hb_merge_runs)."""
    import torch

    from . import _lib
    from .gpu import current_stream_handle, vp

    offs = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(counts, out=offs[1:])
    ko = torch.empty_like(keys)
    io = torch.empty_like(idx)
    if keys.numel():
        _lib.call("hb_merge_runs", vp(keys.data_ptr()), _key_code(keys), vp(idx.data_ptr()), keys.numel(),
                  vp(offs.ctypes.data), len(counts), vp(ko.data_ptr()), vp(io.data_ptr()),
                  _lib.HB_DEVICE_PTRS | _lib.HB_ASYNC, current_stream_handle(keys))
    return ko, io


# ---------------------------------------------------------------- CPU stand-ins (tests)
def host_local_sort(keys, idx):
    """Stable sort of (key, index) CPU tensors."""
    import torch

    order = np.argsort(_np(keys), kind="stable")
    return keys[torch.from_numpy(order)], idx[torch.from_numpy(order)]


def host_split_points(keys, idx, probe_k, probe_i):
    """Lexicographic lower bounds of (probe key, probe index) pairs."""
    import torch

    k, v = _np(keys), idx.numpy()
    out = []
    for a, b in zip(_np(probe_k).tolist(), probe_i.numpy().tolist()):
        lo = int(np.searchsorted(k, a, side="left"))
        hi = int(np.searchsorted(k, a, side="right"))
        out.append(lo + int(np.searchsorted(v[lo:hi], b, side="left")))
    return torch.tensor(out, dtype=torch.int64)


def host_merge_runs(keys, idx, counts):
    """Runs in order + stable sort == stable run merge."""
    return host_local_sort(keys, idx)


def _np(t):
    import torch

    if t.dtype == getattr(torch, "uint32", None):
        return t.view(torch.int32).numpy().view(np.uint32)
    if t.dtype == getattr(torch, "uint64", None):
        return t.view(torch.int64).numpy().view(np.uint64)
    return t.numpy()


# ---------------------------------------------------------------- exchange
def sample_positions(n: int, samples: int):
    """Regular sample positions round(j·(n-1)/(samples-1)), j = 0..samples-1,
    in exact integer arithmetic (a float32 linspace rounds n-1 up past the
    end of the array once n >= 2^24)."""
    import torch

    j = torch.arange(samples, dtype=torch.int64)
    if samples == 1:
        return torch.zeros(1, dtype=torch.int64)
    return (2 * j * (n - 1) + (samples - 1)) // (2 * (samples - 1))


def _ordered_int64(t, pick):
    """int64 values of keys[pick] whose signed order is the key order (u32
    keys by value; u64 keys with the top bit flipped).  Unsigned tensors are
    indexed through their signed view (torch kernels for uint32/uint64 are
    sparse)."""
    import torch

    if t.dtype == getattr(torch, "uint32", None):
        return t.view(torch.int32)[pick].to(torch.int64) & 0xFFFFFFFF
    if t.dtype == getattr(torch, "uint64", None):
        return t.view(torch.int64)[pick] ^ _TOP
    return t[pick].to(torch.int64)


_TOP = -(1 << 63)


def choose_splitters(keys, idx, g: ShardGroup, samples: int):
    """G-1 (key, index) splitters from S regular samples per rank, selected
    on the device: all-gather (key, index, valid) triples, lexicographic
    order, picks at j·m/G of the m valid samples."""
    import torch

    n = keys.numel()
    dev = keys.device
    if n:
        pick = sample_positions(n, samples).to(dev)
        sk, si = _ordered_int64(keys, pick), idx[pick].to(torch.int64)
        ok = torch.ones(samples, dtype=torch.int64, device=dev)
    else:
        sk = si = ok = torch.zeros(samples, dtype=torch.int64, device=dev)
    allp = all_gather_small(torch.stack([sk, si, ok]), g)  # [G, 3, S]
    allp = allp.permute(1, 0, 2).reshape(3, -1)
    valid = allp[2] == 1
    k_all, i_all = allp[0][valid], allp[1][valid]
    # lexicographic (key, index): stable sort by index, then stable by key
    o = torch.argsort(i_all, stable=True)
    k_all, i_all = k_all[o], i_all[o]
    o = torch.argsort(k_all, stable=True)
    k_all, i_all = k_all[o], i_all[o]
    m = int(k_all.numel())
    if m == 0:
        return None, None
    picks = torch.tensor([min(m - 1, (j * m) // g.world) for j in range(1, g.world)], dtype=torch.int64, device=dev)
    pk, pi = k_all[picks], i_all[picks]
    if keys.dtype == getattr(torch, "uint32", None):  # back to u32 bits
        probe_k = pk.to(torch.int32).view(torch.uint32)  # two's-complement wrap keeps the low 32 bits
    elif keys.dtype == getattr(torch, "uint64", None):
        probe_k = (pk ^ _TOP).view(torch.uint64)
    else:
        probe_k = pk.to(keys.dtype)
    return probe_k.contiguous(), pi.to(idx.dtype).contiguous()


def exchange_sort(
    keys: Any,
    idx: Any,
    g: ShardGroup,
    local_sort: Callable = gpu_local_sort,
    split_points: Callable = gpu_split_points,
    samples: int = SAMPLES_PER_RANK,
    merge_runs: Callable = gpu_merge_runs,
    presorted: bool = False,
):
    """Distributed stable sort of sharded (keys, int32 global index) tensors.
    Returns this rank's (keys, idx) interval of the global order.
    `presorted`: the shard is already locally sorted (step 1 done)."""
    import torch

    if not presorted:
        keys, idx = local_sort(keys, idx)
    n = keys.numel()
    probe_k, probe_i = choose_splitters(keys, idx, g, samples)
    if n and probe_k is not None and g.world > 1:
        cuts = split_points(keys, idx, probe_k, probe_i).to(torch.int64).cpu().tolist()
    else:
        cuts = [n] * (g.world - 1)
    bounds = [0] + list(cuts) + [n]
    send = [bounds[j + 1] - bounds[j] for j in range(g.world)]
    sizes = all_gather_small(torch.tensor(send, dtype=torch.int64, device=keys.device), g).cpu()
    recv = sizes[:, g.rank].tolist()  # what every rank sends to me
    k_out = all_to_all_v(keys, send, recv, g)
    i_out = all_to_all_v(idx, send, recv, g)
    return merge_runs(k_out, i_out, recv)


def sample_merge_sort(keys: Any, payload: Any, g: ShardGroup, local_sort: Callable | None = None,
                      split_points: Callable | None = None, merge_runs: Callable | None = None):
    """API form (replicated input → replicated output): shard by floor(k·n/G),
    exchange_sort, all-gather the intervals.  Returns (keys, payload, passes)
    like gpu_sort (payload None sorts keys only; passes 0 ⇔ constant keys).
    CUDA tensors stay on the device; numpy input gives numpy output."""
    import torch

    from .gpu import is_device_array

    local_sort = local_sort or gpu_local_sort
    split_points = split_points or gpu_split_points
    merge_runs = merge_runs or gpu_merge_runs
    host_in = not is_device_array(keys)
    if host_in:
        dev = torch.device("cuda", torch.cuda.current_device()) if local_sort is gpu_local_sort else torch.device("cpu")
        arr = np.ascontiguousarray(keys)
        signed = {np.dtype(np.uint32): (np.int32, torch.uint32), np.dtype(np.uint64): (np.int64, torch.uint64)}
        if arr.dtype in signed:  # moved as the signed bits, viewed back on the device
            k_t = torch.from_numpy(arr.view(signed[arr.dtype][0])).to(dev).view(signed[arr.dtype][1])
        else:
            k_t = torch.from_numpy(arr).to(dev)
    else:
        k_t, dev = keys, keys.device
    n = k_t.numel()
    b = shard_bounds(n, g.world)
    lo, hi = b[g.rank], b[g.rank + 1]
    gidx = torch.arange(lo, hi, dtype=torch.int32, device=dev)
    mk, mi = exchange_sort(k_t[lo:hi].contiguous(), gidx, g, local_sort, split_points, merge_runs=merge_runs)
    sizes = all_gather_small(torch.tensor([mk.numel()], dtype=torch.int64, device=dev), g).reshape(-1).tolist()
    out_k = gather_blocks(mk, sizes, g)
    order = gather_blocks(mi, sizes, g).to(torch.int64)
    out_p = None
    if payload is not None:
        p_t = payload if is_device_array(payload) else torch.from_numpy(np.ascontiguousarray(payload))
        out_p = p_t[order.to(p_t.device)]
    from .sharding import _wire_view

    constant = n > 0 and bool(_wire_view(out_k)[0] == _wire_view(out_k)[-1])
    if host_in:
        out_k = _np(out_k.cpu())
        out_p = out_p.cpu().numpy() if out_p is not None else None
    return out_k, out_p, 0 if constant else 1
