"""World-size-2/3 gloo tests (CPU) of the multi-GPU logic: the partitioner
rules, the histogram all-reduce, the row-strip and SpMV y all-gathers and
the sort sample-merge exchange.  The per-rank compute is the CPU oracle
here; tests/test_gpu_sharded.py runs the same paths with the libhb200
kernels (gloo ranks sharing the box's GPU), and NCCL on an 8-GPU node."""

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
    from paper_1303_2171_b200.sort_exchange import host_local_sort, host_merge_runs, host_split_points, sample_merge_sort

    keys = (ods.sort_keys(20_000, 3) % 50).astype(np.int64)  # heavy ties across ranks
    payload = np.arange(keys.size, dtype=np.int64) * 7
    g = _group()
    k, p, passes = sample_merge_sort(keys, payload, g, host_local_sort, host_split_points, host_merge_runs)
    order = np.argsort(keys, kind="stable")
    ok = np.array_equal(k, keys[order]) and np.array_equal(p, payload[order]) and passes == 1
    const = np.full(999, 5, dtype=np.int64)
    k2, _, passes2 = sample_merge_sort(const, None, g, host_local_sort, host_split_points, host_merge_runs)
    return bool(ok and np.array_equal(k2, const) and passes2 == 0)


def sort_uneven_body(rank, world):
    """Each rank holds a different-size shard (weak-scaling layout): the
    exchange must return globally ordered, stable ranges."""
    import torch
    import torch.distributed as dist

    from oracle import datasets as ods
    from paper_1303_2171_b200.sort_exchange import exchange_sort, host_local_sort, host_merge_runs, host_split_points

    sizes = [3000, 5000, 1, 0][:world]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    allk = ods.sort_keys(int(offs[-1]), 9) % 1000
    mine = torch.from_numpy(allk[offs[rank] : offs[rank + 1]].astype(np.int64))
    idx = torch.arange(int(offs[rank]), int(offs[rank + 1]), dtype=torch.int32)
    k, i = exchange_sort(mine, idx, _group(), host_local_sort, host_split_points, samples=64,
                         merge_runs=host_merge_runs)
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
    from paper_1303_2171_b200.sort_exchange import exchange_sort, host_local_sort, host_merge_runs, host_split_points

    n = 6000
    allk = ods.sort_keys(n * world, 11).astype(np.uint32)  # uniform over [0, 2^32)
    assert (allk >= 1 << 31).any()
    mine = torch.from_numpy(allk[rank * n : (rank + 1) * n].copy()).view(torch.uint32)
    idx = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int32)
    k, i = exchange_sort(mine, idx, _group(), host_local_sort, host_split_points, samples=64,
                         merge_runs=host_merge_runs)
    assert k.dtype == torch.uint32
    parts = [None] * world
    dist.all_gather_object(parts, (k.view(torch.int32).numpy().view(np.uint32), i.numpy()))
    gk = np.concatenate([a for a, _ in parts])
    gi = np.concatenate([b for _, b in parts])
    order = np.argsort(allk, kind="stable")
    return bool(np.array_equal(gk, allk[order]) and np.array_equal(gi, order))


def spmv_body(rank, world):
    """SpMV shard rule (equal nnz, SpmvWorkload's searchsorted at k/G) +
    y_perm all-gather + un-permute, oracle row sums per rank."""
    from oracle import datasets as ods
    from oracle import rng as orng
    from oracle import spmv as ospmv
    from paper_1303_2171_b200 import sharding
    from paper_1303_2171_b200.kernels_irregular import nnz_bounds_host

    ptr, col, val = ods.csr(500, 500, 42, 0.03)
    x = orng.uniform_floats(7, 500)
    perm, (pp, pc, pv), _ = ospmv.preprocess(ptr, col, val, 1.0, 3.0, None)
    split = 123
    g = _group()
    b = nnz_bounds_host(pp, split, 500, world)
    nz = [int(pp[b[k + 1]] - pp[b[k]]) for k in range(world)]
    ok = b[0] == split and b[-1] == 500 and max(nz) - min(nz) <= 31  # one row of slack
    mine = ospmv.range_matvec(pp, pc, pv, x, b[rank], b[rank + 1])
    y_b = sharding.gather_rows(mine, b, g)
    y_perm = np.concatenate([ospmv.range_matvec(pp, pc, pv, x, 0, split), y_b])
    y = np.empty_like(y_perm)
    y[perm] = y_perm
    want = ospmv.hybrid(perm, (pp, pc, pv), split, x)
    return bool(ok and np.array_equal(y.view(np.uint64), want.view(np.uint64)))


def collectives_body(rank, world):
    """Device-agnostic collective helpers: uneven blocks, u32 bits, all-to-all."""
    import torch

    from paper_1303_2171_b200 import sharding

    g = _group()
    counts = [3, 0, 5][:world]
    mine = torch.arange(counts[rank], dtype=torch.int64) + 100 * rank
    got = sharding.gather_blocks(mine, counts, g)
    want = torch.cat([torch.arange(counts[r], dtype=torch.int64) + 100 * r for r in range(world)])
    ok = torch.equal(got, want)
    u = torch.tensor([2**32 - 1 - rank, rank], dtype=torch.int64).to(torch.int32).view(torch.uint32)
    gu = sharding.gather_blocks(u, [2] * world, g)
    ok &= gu.dtype == torch.uint32 and gu.view(torch.int32).tolist()[2 * rank] == -1 - rank
    t = torch.full((4,), rank + 1, dtype=torch.int64)
    sharding.all_reduce_sum(t, g)
    ok &= t.tolist() == [world * (world + 1) // 2] * 4
    send = torch.arange(world, dtype=torch.int64) + 10 * rank
    recv = sharding.all_to_all_v(send, [1] * world, [1] * world, g)
    ok &= recv.tolist() == [10 * r + rank for r in range(world)]
    return bool(ok)


# ---------------------------------------------------------------- tests
def test_shard_bounds_rule():
    assert shard_bounds(10, 3) == [0, 3, 6, 10]
    assert shard_range(7, 1, 2) == (3, 7)
    assert shard_bounds(0, 4) == [0, 0, 0, 0, 0]


@pytest.mark.parametrize("body", ["hist_body", "rows_body", "sort_body", "sort_u32_body", "spmv_body",
                                  "collectives_body"])
def test_world2(body):
    res = run_world(body, 2)
    assert res == {0: True, 1: True}, res


@pytest.mark.parametrize("body", ["sort_uneven_body", "spmv_body", "collectives_body"])
def test_world3(body):
    res = run_world(body, 3)
    assert res == {0: True, 1: True, 2: True}, res


def test_sample_positions_exact_at_benchmark_sizes():
    # the 2^28-key-per-rank sort: float32 linspace would index past the end
    from paper_1303_2171_b200.sort_exchange import sample_positions

    for n in (1, 2, 255, 256, 1 << 24, (1 << 28) + 3, 1 << 28):
        p = sample_positions(n, 256)
        assert int(p[0]) == 0 and int(p[-1]) == n - 1 and bool((p[1:] >= p[:-1]).all())
