"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: the device-side
partitioner, the histogram all-reduce, the row-strip all-gather and the
sort sample-merge exchange.  The per-rank compute is the CPU oracle here;
on the B200 box the same code paths call libhb200 and NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1303_2171_b200.sharding import shard_bounds, shard_range


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn_name, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, globals()[fn_name](rank, world)))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def run_world(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return out


def _group():
    from paper_1303_2171_b200.sharding import group_from_default

    return group_from_default()


# ---------------------------------------------------------------- rank bodies
def hist_body(rank, world):
    from oracle import datasets as ods
    from oracle import hist as ohist
    from paper_1303_2171_b200 import sharding

    data = ods.hist_values(10_001, 42, 256).astype(np.uint8)
    with sharding.gpu_group(_group()):
        got = sharding.run_sharded_histogram(data, 256, local=lambda p, b: ohist.side_counts(p, b, 1))
    return bool(np.array_equal(got, np.bincount(data, minlength=256)))


def rows_body(rank, world):
    from oracle import bilateral as obil
    from oracle import datasets as ods
    from paper_1303_2171_b200 import sharding

    img = ods.image(37, 5)
    sp, rg = obil.lut(2, 1.5, 20.0)
    with sharding.gpu_group(_group()):
        got = sharding.run_sharded_rows(7, 37, lambda a, b: obil.rows(img, sp, rg, 2, a, b))
    return bool(np.array_equal(got, obil.rows(img, sp, rg, 2, 7, 37)))


def sort_body(rank, world):
    from oracle import datasets as ods
    from paper_1303_2171_b200 import sharding
    from paper_1303_2171_b200.sort_exchange import host_local_sort, host_split_points, sample_merge_sort

    keys = (ods.sort_keys(20_000, 3) % 50).astype(np.int64)  # heavy ties across ranks
    payload = np.arange(keys.size, dtype=np.int64) * 7
    g = _group()
    k, p, passes = sample_merge_sort(keys, payload, g, host_local_sort, host_split_points)
    order = np.argsort(keys, kind="stable")
    ok = np.array_equal(k, keys[order]) and np.array_equal(p, payload[order]) and passes == 1
    const = np.full(999, 5, dtype=np.int64)
    k2, _, passes2 = sample_merge_sort(const, None, g, host_local_sort, host_split_points)
    return bool(ok and np.array_equal(k2, const) and passes2 == 0)


def sort_uneven_body(rank, world):
    """Each rank holds a different-size shard (weak-scaling layout): the
    exchange must return globally ordered, stable ranges."""
    import torch
    import torch.distributed as dist

    from oracle import datasets as ods
    from paper_1303_2171_b200.sort_exchange import exchange_sort, host_local_sort, host_split_points

    sizes = [3000, 5000, 1, 0][:world]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    allk = ods.sort_keys(int(offs[-1]), 9) % 1000
    mine = torch.from_numpy(allk[offs[rank] : offs[rank + 1]].astype(np.int64))
    idx = torch.arange(int(offs[rank]), int(offs[rank + 1]), dtype=torch.int32)
    k, i = exchange_sort(mine, idx, _group(), host_local_sort, host_split_points, samples=64)
    parts = [None] * world
    dist.all_gather_object(parts, (k.numpy(), i.numpy()))
    gk = np.concatenate([a for a, _ in parts])
    gi = np.concatenate([b for _, b in parts])
    order = np.argsort(allk, kind="stable")
    return bool(np.array_equal(gk, allk[order]) and np.array_equal(gi, order))


def sort_u32_body(rank, world):
    """u32 keys with the top bit set (the benchmark's key type): the exchange
    must order them unsigned end to end (samples, splitters, wire format)."""
    import torch
    import torch.distributed as dist

    from oracle import datasets as ods
    from paper_1303_2171_b200.sort_exchange import exchange_sort, host_local_sort, host_split_points

    n = 6000
    allk = ods.sort_keys(n * world, 11).astype(np.uint32)  # uniform over [0, 2^32)
    assert (allk >= 1 << 31).any()
    mine = torch.from_numpy(allk[rank * n : (rank + 1) * n].copy()).view(torch.uint32)
    idx = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int32)
    k, i = exchange_sort(mine, idx, _group(), host_local_sort, host_split_points, samples=64)
    assert k.dtype == torch.uint32
    parts = [None] * world
    dist.all_gather_object(parts, (k.view(torch.int32).numpy().view(np.uint32), i.numpy()))
    gk = np.concatenate([a for a, _ in parts])
    gi = np.concatenate([b for _, b in parts])
    order = np.argsort(allk, kind="stable")
    return bool(np.array_equal(gk, allk[order]) and np.array_equal(gi, order))


# ---------------------------------------------------------------- tests
def test_shard_bounds_rule():
    assert shard_bounds(10, 3) == [0, 3, 6, 10]
    assert shard_range(7, 1, 2) == (3, 7)
    assert shard_bounds(0, 4) == [0, 0, 0, 0, 0]


@pytest.mark.parametrize("body", ["hist_body", "rows_body", "sort_body", "sort_u32_body"])
def test_world2(body):
    res = run_world(body, 2)
    assert res == {0: True, 1: True}, res


def test_world3_uneven_sort_exchange():
    res = run_world("sort_uneven_body", 3)
    assert res == {0: True, 1: True, 2: True}, res


def test_sample_positions_exact_at_benchmark_sizes():
    # the 2^28-key-per-rank sort: float32 linspace would index past the end
    from paper_1303_2171_b200.sort_exchange import sample_positions

    for n in (1, 2, 255, 256, 1 << 24, (1 << 28) + 3, 1 << 28):
        p = sample_positions(n, 256)
        assert int(p[0]) == 0 and int(p[-1]) == n - 1 and bool((p[1:] >= p[:-1]).all())
