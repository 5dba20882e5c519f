"""The multi-GPU work-partitioned path with the libhb200 kernels.

Part 1 (one process): the device halves of the sharded merges — the device
partitioner (hb_partition_nnz) against SpmvWorkload's host split rule, the
stable G-way run merge (hb_merge_runs) against numpy's stable sort, and the
phased list ranking (hb_lr_walk_part / hb_lr_finish_part) with G parts
emulated on one GPU against the oracle's ranks.

Part 2 (2 and 3 gloo ranks sharing the box's GPU — the pool has one GPU per
box; NCCL needs one GPU per rank): every workload through the PUBLIC API
inside `sharding.gpu_group`, so each rank runs its shard on libhb200 and the
merge is the real collective: histogram all-reduce, SpMV y all-gather +
device un-permute, filter strip all-gathers, sort sample-merge exchange,
sharded list ranking — compared bit for bit with the oracle."""

import os
import socket

import numpy as np
import pytest

from oracle import bilateral as obil
from oracle import conv as oconv
from oracle import datasets as ods
from oracle import hist as ohist
from oracle import listrank as olr
from oracle import rng as orng
from oracle import spmv as ospmv

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


# ---------------------------------------------------------------- part 1: one process
def test_device_partitioner_matches_split_rule():
    import torch

    from paper_1303_2171_b200 import _lib
    from paper_1303_2171_b200.gpu import vp
    from paper_1303_2171_b200.kernels_irregular import CsrMatrix, nnz_bounds_host, partition_nnz

    rs = np.random.default_rng(3)
    for rows in (1, 7, 1000, 65_537):
        counts = rs.integers(0, 40, rows)
        counts[rs.random(rows) < 0.2] = 0  # empty rows
        ptr = np.zeros(rows + 1, dtype=np.int64)
        np.cumsum(counts, out=ptr[1:])
        col = np.concatenate([np.sort(rs.choice(1000, c, replace=False)) for c in counts]).astype(np.int64) \
            if ptr[-1] else np.zeros(0, np.int64)
        m = CsrMatrix(rows, 1000, ptr, col, np.ones(int(ptr[-1])))
        for idx_dt in (np.int32, np.int64):
            dm = m.to_device(idx_dt)
            for parts in (1, 2, 3, 8, 13):
                for r0, r1 in ((0, rows), (rows // 3, rows), (rows // 2, rows // 2)):
                    want = nnz_bounds_host(ptr, r0, r1, parts)
                    assert partition_nnz(dm, r0, r1, parts) == want, (rows, parts, r0, r1)
                    # host pointer path of the same C entry (only the window is staged)
                    out = np.zeros(parts + 1, dtype=np.int64)
                    hp = ptr.astype(idx_dt) if idx_dt == np.int32 else ptr
                    _lib.call("hb_partition_nnz", vp(hp.ctypes.data), 6 if idx_dt == np.int32 else 8, r0, r1, parts,
                              vp(out.ctypes.data), 0, None)
                    assert out.tolist() == want
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype", ["uint32", "int32", "uint64", "int64"])
def test_merge_runs_stable(dtype):
    import torch

    from paper_1303_2171_b200.sort_exchange import gpu_merge_runs

    rs = np.random.default_rng(5)
    for nruns in (1, 2, 3, 5, 8, 9):
        sizes = rs.integers(0, 5000, nruns)
        sizes[rs.random(nruns) < 0.2] = 0
        runs = [np.sort(rs.integers(0, 300, s)).astype(dtype) for s in sizes]  # heavy ties
        if dtype.startswith("u") and runs:
            runs[0] = np.sort(np.concatenate([runs[0], np.array([np.iinfo(dtype).max] * 3, dtype=dtype)]))
            sizes[0] = runs[0].size
        keys = np.concatenate(runs) if runs else np.zeros(0, dtype)
        idx = np.arange(keys.size, dtype=np.int32)
        tdt = getattr(torch, dtype)
        if dtype in ("uint32", "uint64"):
            kt = torch.from_numpy(keys.view(dtype.replace("u", ""))).cuda().view(tdt)
        else:
            kt = torch.from_numpy(keys).cuda()
        ko, io = gpu_merge_runs(kt, torch.from_numpy(idx).cuda(), sizes.tolist())
        order = np.argsort(keys, kind="stable")
        got_k = ko.view(getattr(torch, dtype.replace("u", ""))).cpu().numpy().view(dtype) if dtype[0] == "u" else ko.cpu().numpy()
        assert np.array_equal(got_k, keys[order]), nruns
        assert np.array_equal(io.cpu().numpy(), order), nruns


def _emulated_parts_rank(succ, head, parts):
    """The sharded ranking's phases with `parts` ranks emulated on one GPU."""
    import ctypes

    import torch

    from paper_1303_2171_b200 import _lib
    from paper_1303_2171_b200.gpu import vp
    from paper_1303_2171_b200.sharding import shard_bounds

    n = succ.size
    sd = torch.from_numpy(succ.astype(np.int32)).cuda()
    nsub, sh = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.call("hb_lr_layout", n, head, ctypes.byref(nsub), ctypes.byref(sh))
    nsub, sh = nsub.value, sh.value
    b = shard_bounds(nsub, parts)
    nxt = torch.empty(nsub, dtype=torch.int64, device="cuda")
    ln = torch.empty(nsub, dtype=torch.int64, device="cuda")
    packed = []
    for k in range(parts):
        r = torch.empty(n, dtype=torch.int64, device="cuda")
        _lib.call("hb_lr_walk_part", vp(sd.data_ptr()), 6, n, head, b[k], b[k + 1], vp(r.data_ptr()),
                  vp(nxt.data_ptr()), vp(ln.data_ptr()), _lib.HB_DEVICE_PTRS, None)
        packed.append(r)
    total = torch.zeros(n, dtype=torch.int64, device="cuda")
    for k in range(parts):
        _lib.call("hb_lr_finish_part", vp(nxt.data_ptr()), vp(ln.data_ptr()), nsub, sh, n, b[k], b[k + 1],
                  vp(packed[k].data_ptr()), _lib.HB_DEVICE_PTRS, None)
        total += packed[k]
    return total.cpu().numpy()


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_lr_phases_emulated(parts):
    for n, seed in ((1, 1), (2, 2), (63, 3), (64, 4), (65, 5), (5000, 6), (300_001, 7)):
        succ, head = ods.linked_list(n, seed)
        got = _emulated_parts_rank(succ, head, parts)
        assert np.array_equal(got, olr.chase(succ, head)), (n, parts)


def test_lr_phases_detect_malformed_lists():
    from paper_1303_2171_b200.errors import StructuralError

    succ, head = ods.linked_list(10_000, 9)
    cyc = succ.copy()
    tail = int(np.flatnonzero(cyc == -1)[0])
    cyc[tail] = head  # one cycle through every node: no tail
    with pytest.raises(StructuralError):
        _emulated_parts_rank(cyc, head, 3)
    # a tail, plus a detached cycle of sublist heads (nodes 0 and 64): the
    # chain from the head covers fewer than n nodes
    br, h2 = ods.linked_list(10_000, 10)
    a, b = 0, 64
    assert h2 not in (a, b)
    # splice a and b out of the list and make them a 2-cycle
    for v in (a, b):
        p = int(np.flatnonzero(br == v)[0]) if (br == v).any() else None
        if p is not None:
            br[p] = br[v]
    br[a], br[b] = b, a
    assert (br == -1).sum() == 1
    with pytest.raises(StructuralError):
        _emulated_parts_rank(br, h2, 2)


# ---------------------------------------------------------------- part 2: gloo ranks on the GPU
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _all_workloads(rank, world)))
    except Exception as exc:  # surfaced by the parent
        import traceback

        q.put((rank, repr(exc) + traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


def _all_workloads(rank, world):
    import torch

    from paper_1303_2171_b200 import kernels_irregular as ki
    from paper_1303_2171_b200 import kernels_regular as kr
    from paper_1303_2171_b200 import sharding
    from paper_1303_2171_b200.platform import Platform
    from paper_1303_2171_b200.worksharing import WorkShare, calibrate_measured

    p = Platform.build(1.0, 3.0)
    g = sharding.group_from_default()
    assert g is not None and g.world == world
    res = {}
    with sharding.gpu_group(g):
        # histogram: host data and device data, host share 0 and 0.3
        data = ods.hist_values(300_007, 42, 256).astype(np.uint8)
        want = np.bincount(data, minlength=256)
        for sh in (0.0, 0.3):
            got = kr.hybrid_histogram(data, 256, p, WorkShare.manual(sh)).bins
            res[f"hist_host_{sh}"] = np.array_equal(got, want)
            got = kr.hybrid_histogram(torch.from_numpy(data).cuda(), 256, p, WorkShare.manual(sh)).bins
            res[f"hist_dev_{sh}"] = np.array_equal(got, want)
        part = torch.from_numpy(data).cuda()
        out = kr.HistogramWorkload(part, 256).run_part(p.device_b, part)
        res["hist_run_part_on_device"] = bool(out.is_cuda) and np.array_equal(out.cpu().numpy(), want)

        # SpMV: host matrix and device matrix (device partitioner + y gather + scatter)
        ptr, col, val = ods.csr(3000, 3000, 42, 0.005)
        x = 2.0 * orng.uniform_floats(orng.mix_seed(42, 0xDEC0), 3000) - 1.0
        m = ki.CsrMatrix(3000, 3000, ptr, col, val)
        for sh in (0.0, 0.4):
            prep = ki.spmv_preprocess(m, p, WorkShare.manual(sh))
            perm, permuted, split = ospmv.preprocess(ptr, col, val, 1.0, 3.0, sh)
            want = ospmv.hybrid(perm, permuted, split, x)
            res[f"spmv_host_{sh}"] = np.array_equal(bits(ki.spmv_hybrid(prep, x)), bits(want))
            dprep = ki.spmv_preprocess(m.to_device(), p, WorkShare.manual(sh))
            y = ki.spmv_hybrid(dprep, torch.from_numpy(x).cuda())
            res[f"spmv_dev_{sh}"] = bool(y.is_cuda) and np.array_equal(bits(y.cpu().numpy()), bits(want))
            wl = ki.SpmvWorkload(dprep, torch.from_numpy(x).cuda())
            from paper_1303_2171_b200.worksharing import run_workshared

            yw, _ = run_workshared(p, wl, WorkShare.manual(sh), baselines=False)
            res[f"spmv_workload_{sh}"] = np.array_equal(bits(yw), bits(want))

        # filters: host image and device image, strips all-gathered
        img = ods.image(97, 4)
        lut = kr.build_bilateral_lut(3, 1.5, 30.0)
        sp, rg = obil.lut(3, 1.5, 30.0)
        want = obil.rows(img, sp, rg, 3, 0, 97)
        for sh in (0.0, 0.25):
            got = kr.hybrid_bilateral(kr.Image(img), lut, p, WorkShare.manual(sh)).pixels
            res[f"bilat_host_{sh}"] = np.array_equal(bits(got), bits(want))
            got = kr.hybrid_bilateral(kr.Image(torch.from_numpy(img).cuda()), lut, p, WorkShare.manual(sh)).pixels
            res[f"bilat_dev_{sh}"] = np.array_equal(bits(sharding.to_numpy(got)), bits(want))
        fk = kr.FilterKernel.gaussian(2)
        want = oconv.rows(img, fk.weights, 0, 97)
        got = kr.hybrid_convolve(kr.Image(torch.from_numpy(img).cuda()), fk, p, WorkShare.manual(0.0)).pixels
        res["conv_dev"] = np.array_equal(bits(sharding.to_numpy(got)), bits(want))
        dimg = torch.from_numpy(img).cuda()
        strip = kr.BilateralApplyWorkload(kr.Image(dimg), lut).run_part(p.device_b, (0, 97))
        res["bilat_run_part_on_device"] = bool(strip.is_cuda)

        # sort: sample-merge through the public API (host u32 keys, device keys, ties)
        keys = ods.sort_keys(40_001, 3).astype(np.uint32)
        out, wa, wb = kr.sample_sort_hybrid(keys, p, share=WorkShare.manual(0.0))
        res["sort_host_u32"] = np.array_equal(out, np.sort(keys)) and (wa, wb) == (0.0, float(keys.size))
        tk = torch.from_numpy((keys % 97).astype(np.int32)).cuda()
        out, _, _ = kr.sample_sort_hybrid(tk, p, share=WorkShare.manual(0.0))
        res["sort_dev_i32_ties"] = np.array_equal(out.cpu().numpy(), np.sort(keys % 97).astype(np.int32))
        fl = (ods.sort_keys(5000, 4).astype(np.float64) - 2.0**31) / 7.0
        out, _, _ = kr.sample_sort_hybrid(fl, p, share=WorkShare.manual(0.0))
        res["sort_host_f64"] = out.dtype == np.float64 and np.array_equal(out, np.sort(fl))
        # distributed exchange with the GPU kernels: stable (key, global index)
        from paper_1303_2171_b200.sort_exchange import exchange_sort

        allk = ods.sort_keys(30_000 * world, 11).astype(np.uint32) % 5000
        lo, hi = rank * 30_000, (rank + 1) * 30_000
        mk = torch.from_numpy(allk[lo:hi].view(np.int32)).cuda().view(torch.uint32)
        mi = torch.arange(lo, hi, dtype=torch.int32, device="cuda")
        k, i = exchange_sort(mk.clone(), mi, g)
        gk = sharding.gather_blocks(k, sharding.all_gather_small(torch.tensor([k.numel()], device="cuda"), g)
                                    .reshape(-1).tolist(), g)
        sizes = sharding.all_gather_small(torch.tensor([k.numel()], device="cuda"), g).reshape(-1).tolist()
        gi = sharding.gather_blocks(i, sizes, g)
        order = np.argsort(allk, kind="stable")
        res["exchange_stable"] = (np.array_equal(gk.view(torch.int32).cpu().numpy().view(np.uint32), allk[order])
                                  and np.array_equal(gi.cpu().numpy(), order))

        # list ranking: sharded sublists (host succ and device succ)
        succ, head = ods.linked_list(200_003, 8)
        want = olr.chase(succ, head)
        lst = ki.LinkedListArr(succ, head)
        res["lr_host"] = np.array_equal(ki.list_rank_hybrid(lst, p, 7), want)
        dl = ki.LinkedListArr(torch.from_numpy(succ.astype(np.int32)).cuda(), head)
        r = ki.list_rank_hybrid(dl, p, 7)
        res["lr_dev"] = bool(r.is_cuda) and np.array_equal(r.cpu().numpy(), want)
        bad = succ.copy()
        bad[int(np.flatnonzero(bad == -1)[0])] = head
        try:
            ki.list_rank_hybrid(ki.LinkedListArr(bad, head), p, 7)
            res["lr_cycle_raises"] = False
        except ki.StructuralError:
            res["lr_cycle_raises"] = True

        # measured calibration agrees across ranks (same fraction everywhere)
        sh = calibrate_measured(kr.HistogramWorkload(data, 256), p, max_refinements=2, repeats=1)
        fr = sharding.all_gather_small(torch.tensor([sh.fraction_a], dtype=torch.float64, device="cuda"), g)
        res["calibrate_agrees"] = len(set(fr.reshape(-1).cpu().tolist())) == 1
    bad = sorted(k for k, v in res.items() if not v)
    return True if not bad else f"failed: {bad}"


def _run(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_public_api_under_gpu_group(world):
    res = _run(world)
    assert res == {r: True for r in range(world)}, res
