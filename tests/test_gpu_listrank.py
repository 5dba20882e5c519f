"""List ranking GPU parity: ranks identical to the reference's own outputs
(golden) and to pointer chasing; malformed lists raise StructuralError.
Mirrors tests/test_kernels_irregular.py:214-266 and acceptance :204-229."""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import datasets as ods
from oracle import listrank as olr
from oracle import rng as orng
from paper_1303_2171_b200.errors import StructuralError
from paper_1303_2171_b200.kernels_irregular import (
    LinkedListArr,
    gpu_list_rank,
    list_rank_hybrid,
    list_rank_with_stats,
    validate_list,
)

pytestmark = pytest.mark.gpu


def test_golden_ranks(platform13):
    g = golden("listrank")
    for i in range(6):
        lst = LinkedListArr(g[f"succ_{i}"], int(g[f"head_{i}"][0]))
        assert np.array_equal(list_rank_hybrid(lst, platform13, int(g[f"seed_{i}"][0])), g[f"rank_{i}"])


def test_singleton_and_ordered_chain(platform13):
    assert list_rank_hybrid(LinkedListArr(np.array([-1]), 0), platform13, 1).tolist() == [0]
    assert list_rank_hybrid(LinkedListArr(np.array([1, 2, 3, -1]), 0), platform13, 1).tolist() == [0, 1, 2, 3]


@pytest.mark.parametrize("n", [2, 63, 64, 65, 4095, 4096, 4097, 300_001, 2_000_000])
def test_random_lists_match_chase(n):
    succ, head = ods.linked_list(n, n)
    order = np.argsort(orng.draws(n, n), kind="stable")
    want = olr.ranks_from_order(order)
    assert np.array_equal(gpu_list_rank(succ, head), want)
    assert np.array_equal(gpu_list_rank(succ.astype(np.int32), head), want)


def test_structural_invariants_50_lists(platform13):
    for i in range(50):
        n = 100 + (orng.mix_seed(i, 5) % 9_901)
        succ, head = ods.linked_list(int(n), i)
        r = list_rank_hybrid(LinkedListArr(succ, head), platform13, i)
        assert np.array_equal(r, olr.chase(succ, head))
        assert r[head] == 0
        inner = succ >= 0
        assert np.array_equal(r[succ[inner]], r[inner] + 1)


def test_pathological_orders():
    n = 100_000
    ordered = np.arange(1, n + 1, dtype=np.int64); ordered[-1] = -1
    assert np.array_equal(gpu_list_rank(ordered, 0), np.arange(n))
    rev = np.arange(-1, n - 1, dtype=np.int64)  # n-1 -> n-2 -> ... -> 0
    assert np.array_equal(gpu_list_rank(rev, n - 1), np.arange(n)[::-1])
    # non-multiples of 64 first, then multiples: one very long first sublist
    order = np.concatenate([np.flatnonzero(np.arange(n) % 64 != 0), np.arange(0, n, 64)])
    succ = np.full(n, -1, dtype=np.int64); succ[order[:-1]] = order[1:]
    assert np.array_equal(gpu_list_rank(succ, int(order[0])), olr.ranks_from_order(order))


def test_device_resident():
    import torch

    succ, head = ods.linked_list(1_000_000, 42)
    got = gpu_list_rank(torch.from_numpy(succ.astype(np.int32)).cuda(), head)
    assert np.array_equal(got.cpu().numpy(), olr.chase(succ, head))


@pytest.mark.parametrize("dtype", ["int32", "int64"])
def test_unaligned_device_views_and_range_check(dtype):
    """Device successors passed as views at every 4/8-byte offset inside a
    16-byte vector (the pre-check reads aligned arrays with 16-byte loads),
    valid and with one out-of-range successor at the start, the middle and
    the scalar tail."""
    import torch

    tdt = getattr(torch, dtype)
    n = 1_000_003
    succ, head = ods.linked_list(n, 7)
    want = olr.chase(succ, head)
    for off in range(16 // torch.tensor([], dtype=tdt).element_size()):
        big = torch.zeros(n + off, dtype=tdt, device="cuda")
        view = big[off:]
        view.copy_(torch.from_numpy(succ.astype(dtype)))
        assert np.array_equal(gpu_list_rank(view, head).cpu().numpy(), want), off
        for at in (0, n // 2, n - 1):
            bad = view.clone() if off == 0 else view
            keep = int(bad[at])
            bad[at] = n + 5
            with pytest.raises(StructuralError):
                gpu_list_rank(bad, head)
            bad[at] = keep


def test_broken_lists_raise():
    for succ, head in ((np.array([1, 0]), 0), (np.array([-1, -1]), 0), (np.array([5]), 0), (np.array([-1]), 3)):
        with pytest.raises(StructuralError):
            gpu_list_rank(succ, head)
        with pytest.raises(StructuralError):
            validate_list(LinkedListArr(succ, head))
    # big broken cases: a detached cycle, and two chains
    n = 100_000
    succ, head = ods.linked_list(n, 3)
    cyc = succ.copy()
    tail = int(np.flatnonzero(cyc == -1)[0])
    order = olr.chase(succ, head).argsort()
    # cut the chain 10 nodes before the end and close those nodes into a ring
    a = order[-10]
    cyc[order[-11]] = -1
    cyc[tail] = a
    with pytest.raises(StructuralError):
        gpu_list_rank(cyc, head)
    two = succ.copy()
    two[order[n // 2]] = -1  # second half detached: two tails
    with pytest.raises(StructuralError):
        gpu_list_rank(two, head)


def test_device_list_generator_matches_reference():
    from paper_1303_2171_b200.datasets import device_gen_list

    g = golden("listrank")
    succ, head = device_gen_list(10_000, 42, np.int64)
    assert np.array_equal(succ.cpu().numpy(), g["succ_0"]) and head == int(g["head_0"][0])
    for n, seed in ((5, 7), (4097, 11), (100_000, 3)):
        s2, h2 = device_gen_list(n, seed)
        want_s, want_h = ods.linked_list(n, seed)
        assert np.array_equal(s2.cpu().numpy(), want_s) and h2 == want_h


def test_golden_stats_identical(platform13):
    g = golden("listrank")
    for i in range(6):
        lst = LinkedListArr(g[f"succ_{i}"], int(g[f"head_{i}"][0]))
        rank, st = list_rank_with_stats(lst, platform13, int(g[f"seed_{i}"][0]))
        assert np.array_equal(rank, g[f"rank_{i}"])
        assert [st.fis_rounds, st.reduced_size, st.removed_total, st.sublist_count] == g[f"stats_{i}"].tolist()
        assert list(st.round_sizes) == g[f"sizes_{i}"].tolist()


def test_stats_match_oracle_many_lists(platform13):
    for i in range(12):
        n = 100 + (orng.mix_seed(i, 5) % 20_000)
        succ, head = ods.linked_list(int(n), i)
        rank, st = list_rank_with_stats(LinkedListArr(succ, head), platform13, i)
        want_rank, (rounds, sizes, reduced, removed, subl) = olr.list_rank_with_stats(succ, head, i)
        assert np.array_equal(rank, want_rank)
        assert (st.fis_rounds, st.round_sizes, st.reduced_size, st.removed_total, st.sublist_count) == (
            rounds, sizes, reduced, removed, subl)
        assert st.reduced_size <= n / math.log2(n)


def test_stats_large_list_device():
    import torch

    from paper_1303_2171_b200.datasets import device_gen_list
    from paper_1303_2171_b200.kernels_irregular import gpu_list_fis_stats

    n = 1 << 20
    succ_d, head = device_gen_list(n, 42)
    st = gpu_list_fis_stats(succ_d, head, 7, 32)
    succ, head2 = ods.linked_list(n, 42)
    assert head2 == head
    _, (rounds, sizes, reduced, removed, subl) = olr.list_rank_with_stats(succ, head, 7)
    assert (st.fis_rounds, st.round_sizes, st.reduced_size, st.removed_total, st.sublist_count) == (
        rounds, sizes, reduced, removed, subl)


@pytest.mark.parametrize("order", ["identity", "reverse", "random", "blocks"])
@pytest.mark.parametrize("n", [(1 << 20), (1 << 20) + 37, 3_000_001])
def test_logged_walk_orders(n, order):
    """Lists of >= 2^20 nodes take the logged level-1 walk (sequential
    (node, offset) log + bucketed scatter of the ranks): every ordering,
    heads on and off the 64-node grid, sizes not a power of two."""
    rs = np.random.default_rng(n)
    if order == "identity":
        seq = np.arange(n)
    elif order == "reverse":
        seq = np.arange(n)[::-1].copy()
    elif order == "random":
        seq = rs.permutation(n)
    else:  # long runs of consecutive nodes in random block order
        blk = 1000
        starts = rs.permutation((n + blk - 1) // blk) * blk
        seq = np.concatenate([np.arange(s0, min(n, s0 + blk)) for s0 in starts])
    succ = np.full(n, -1, dtype=np.int64)
    succ[seq[:-1]] = seq[1:]
    head = int(seq[0])
    want = np.empty(n, dtype=np.int64)
    want[seq] = np.arange(n)
    got = gpu_list_rank(succ.astype(np.int32), head)
    assert np.array_equal(got, want), (n, order)


def test_ballot_ranking_fallback_paths():
    """With the ballot ranking forced (HB_SORT_RANK=ballot, read once per
    process: a subprocess), every sort-based path takes its general branch —
    the logged walk's node sort included (two pair arrays + sort + widen
    instead of the fused packed sort) — and gives the same results."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = (
        "import numpy as np, torch\n"
        "from oracle import datasets as ods\n"
        "from oracle import listrank as olr\n"
        "from oracle import sort as osort\n"
        "from paper_1303_2171_b200.kernels_irregular import gpu_list_rank\n"
        "from paper_1303_2171_b200.kernels_regular import gpu_sort\n"
        "succ, head = ods.linked_list(1_500_000, 77)\n"
        "got = gpu_list_rank(torch.from_numpy(succ.astype(np.int32)).cuda(), head).cpu().numpy()\n"
        "assert np.array_equal(got, olr.chase(succ, head)), 'ranks'\n"
        "k = (np.random.default_rng(3).integers(0, 7, size=300_001)).astype(np.uint32)\n"
        "sk, sv, _ = gpu_sort(k, np.arange(k.size, dtype=np.uint32))\n"
        "assert osort.check_stable_payload(k, sk, sv), 'stable payload'\n"
        "print('ok')\n"
    )
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, HB_SORT_RANK="ballot", PYTHONPATH=str(root) + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("pinned", [False, True])
def test_host_lists_large(pinned):
    """Host lists of 2^23+ nodes (many 32 MB pinned-stage chunks, a ragged
    last chunk), pageable and page-locked int64 successors and int32
    successors: identical to the device-resident ranking; a successor outside
    int32 anywhere (first chunk, last element) raises validate_list's range
    error, and one inside int32 but >= n the same."""
    import torch

    n = (1 << 23) + 4099
    seq = np.random.default_rng(7).permutation(n)
    succ = np.full(n, -1, dtype=np.int64)
    succ[seq[:-1]] = seq[1:]
    head = int(seq[0])
    want = np.empty(n, dtype=np.int64)
    want[seq] = np.arange(n)
    if pinned:
        t = torch.empty(n, dtype=torch.int64, pin_memory=True)
        t.numpy()[...] = succ
        succ = t.numpy()
    got = gpu_list_rank(succ, head)
    assert got.dtype == np.int64 and np.array_equal(got, want)
    assert np.array_equal(gpu_list_rank(np.asarray(succ, dtype=np.int32), head), want)
    dev = gpu_list_rank(torch.from_numpy(np.array(succ)).cuda(), head).cpu().numpy()
    assert np.array_equal(dev, want)
    for pos, bad in ((5, 1 << 40), (n - 1, -(1 << 35)), (n // 2, n)):
        s2 = np.array(succ)
        s2[seq[pos]] = bad
        with pytest.raises(StructuralError, match="out of range"):
            gpu_list_rank(s2, head)
