"""Oracle: FIS-reduction list ranking (reference kernels_irregular.py:356-508).
Test infrastructure / CPU baseline."""

from __future__ import annotations

import math

import numpy as np

from .rng import draws, mix_seed

END = -1  # LIST_END, kernels_irregular.py:29


class Broken(Exception):
    """Stands in for the reference's StructuralError inside the oracle."""


def validate(succ: np.ndarray, head: int) -> None:
    """:377-393: range check, then a walk from head covering every node."""
    n = succ.size
    if not 0 <= head < n:
        raise Broken("head out of range")
    if n and (succ.min() < END or succ.max() >= n):
        raise Broken("successor index out of range")
    seen, cur = 0, head
    while cur != END:
        seen += 1
        if seen > n:
            raise Broken("list contains a cycle")
        cur = int(succ[cur])
    if seen != n:
        raise Broken(f"chain covers {seen} of {n} nodes (broken list)")


def fis_reduce(succ_in: np.ndarray, head: int, seed: int, target: int):
    """:396-428: per round r, bit(i) = draw_i(mix_seed(seed, r)) & 1; remove
    nodes with bit 1 whose successor has bit 0 (never the head); splice each
    removed node out through its predecessor, which absorbs its weight."""
    n = succ_in.size
    succ = succ_in.copy()
    weight = np.ones(n, dtype=np.int64)
    alive = np.ones(n, dtype=bool)
    events, sizes = [], []
    live, rounds = n, 0
    while live > target and rounds < 1000:
        sizes.append(live)
        bit = (draws(mix_seed(seed, rounds), n) & np.uint64(1)).astype(np.int64)
        nxt_bit = np.where(succ >= 0, bit[np.clip(succ, 0, n - 1)], 0)
        removable = alive & (bit == 1) & (nxt_bit == 0)
        removable[head] = False
        has_next = alive & (succ >= 0)
        pred = np.flatnonzero(has_next)
        pred = pred[removable[succ[pred]]]
        gone = succ[pred]
        rounds += 1
        if gone.size == 0:
            continue
        events.append((gone, pred, weight[pred].copy()))
        weight[pred] += weight[gone]
        succ[pred] = succ[gone]
        alive[gone] = False
        live -= gone.size
    if live > target:
        raise Broken("independent-set reduction failed to converge")
    return succ, weight, alive, events, sizes


def rank_reduced(succ, weight, alive, head, seed, sublists):
    """:431-478: s random sublist heads (smallest draws among survivors, in
    survivor order) + the head; weighted local ranks; prefix over heads."""
    n = succ.size
    surv = np.flatnonzero(alive)
    s = max(1, min(sublists, surv.size))
    chosen = surv[np.argsort(draws(mix_seed(seed, 0x5EED), surv.size), kind="stable")[: s - 1]]
    is_head = np.zeros(n, dtype=bool)
    is_head[chosen] = True
    is_head[head] = True
    rank = np.zeros(n, dtype=np.int64)
    owner = np.full(n, -1, dtype=np.int64)
    link = {}
    for h0 in np.flatnonzero(is_head).tolist():
        owner[h0] = h0
        acc = int(weight[h0])
        cur = int(succ[h0])
        while cur != END and not is_head[cur]:
            rank[cur] = acc
            owner[cur] = h0
            acc += int(weight[cur])
            cur = int(succ[cur])
        link[h0] = (cur, acc)
    base = np.zeros(n, dtype=np.int64)
    cur, off, hops = int(head), 0, 0
    while cur != END:
        base[cur] = off
        cur, length = link[cur]
        off += length
        hops += 1
        if hops > n:
            raise Broken("sublist chain does not terminate")
    rank[alive] += base[owner[alive]]
    return rank, int(is_head.sum())


def list_rank_with_stats(succ: np.ndarray, head: int, seed: int, workers_total: int = 8):
    """:481-502 → (rank, (fis_rounds, round_sizes, reduced, removed, sublists))."""
    validate(succ, head)
    n = succ.size
    if n == 1:
        return np.zeros(1, dtype=np.int64), (0, (), 1, 0, 1)
    target = max(int(n / math.log2(n)), 2) if n > 2 else 2
    s2, w2, alive, events, sizes = fis_reduce(succ, head, seed, target)
    rank, used = rank_reduced(s2, w2, alive, head, seed, 4 * workers_total)
    for gone, pred, w_pred in reversed(events):
        rank[gone] = rank[pred] + w_pred
    kept = int(alive.sum())
    return rank, (len(sizes), tuple(sizes), kept, n - kept, used)


def chase(succ: np.ndarray, head: int) -> np.ndarray:
    """Pointer-chasing ranks (reference tests/oracles.py:103-110)."""
    rank = np.zeros(succ.size, dtype=np.int64)
    cur, r = int(head), 0
    while cur != END:
        rank[cur] = r
        r += 1
        cur = int(succ[cur])
    return rank


def ranks_from_order(order: np.ndarray) -> np.ndarray:
    """For lists built by datasets.linked_list: rank = inverse(order)."""
    rank = np.empty(order.size, dtype=np.int64)
    rank[order] = np.arange(order.size, dtype=np.int64)
    return rank
