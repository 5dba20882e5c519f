"""Benchmark driver for the B200 work-partitioned hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload hist|…|all]
                    [--impl ours|reference] [--scaling weak|strong] [--shape config|largest]

Prints ONE compact JSON line (rank 0; the full per-workload record goes to
gpurun_out/bench_detail.json).  The headline is BASELINE.json configs[1] —
256-bin histogram over 2^30 uint8 per GPU — and every other configured
workload is summarised under "workloads".  A step is one pass of the hot
path over one batch of synthetic input already resident in HBM (`value`);
`e2e` is the same metric through the public drop-in API on host buffers
(H2D + D2H inside the timed region).

Multi-GPU (torchrun, one process per GPU): every rank runs the workload
through the public API's sharded DeviceB path inside
`sharding.gpu_group` — its shard on libhb200 plus the workload's merge
collective (histogram all-reduce, SpMV device partitioner + y all-gather +
un-permute, filter strip all-gather, sort sample-merge exchange, sharded
list ranking), all on device memory.  `--scaling weak` (default): every GPU
owns a config-sized share of a G-times larger global input; list ranking
is always the config list (one list cannot be given a fixed per-GPU
share).  `--scaling strong`: the global input is the config (or, with
`--shape largest`, the larger shapes named in DESIGN.md §6) for every N.

`--impl reference` times the UNMODIFIED reference package (baseline/_ref,
bench_reference.py) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ARGS = argparse.Namespace(e2e_share="auto", scaling="weak", shape="config")  # set by main()

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
TRAFFIC_FILE = ROOT / "profiles" / "traffic.json"
DETAIL_FILE = ROOT / "gpurun_out" / "bench_detail.json"

RANDOM_READ_PEAK = 42.2   # G dependent random 4-B reads/s (~118 B of HBM each), scripts/micro/rand_read.cu
FP64_PEAK_GFLOPS = 18370.0  # non-FMA fp64 instructions/s, scripts/micro/fp64peak.cu
METRIC = "per-workload throughput (SpMV GFLOP/s, sort Mkeys/s) and HBM-roofline fraction"


# ---------------------------------------------------------------- utilities
def hbm_peak() -> tuple[float, str]:
    try:
        return float(json.loads(PEAKS_FILE.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return FALLBACK_HBM_GBS, "B200_PROFILING.md fallback"


def traffic_of(kernel: str):
    try:
        return json.loads(TRAFFIC_FILE.read_text()).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """Polls NVML (SM clock + clock-event reasons) on a thread; `summary()`
    returns the samples that fall inside [t0, t1]."""

    REASONS = {
        "hw_slowdown": 0x8,
        "hw_thermal_slowdown": 0x40,
        "sw_thermal_slowdown": 0x20,
        "sw_power_cap": 0x4,
        "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.samples: list[tuple[float, int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self) -> None:
        nv = self._nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)

    def summary(self, t0: float, t1: float) -> dict:
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        window = "timed"
        if not inside:  # region shorter than the polling period: nearest samples
            inside = sorted(self.samples, key=lambda s: min(abs(s[0] - t0), abs(s[0] - t1)))[:5]
            window = "adjacent"
        reasons = set()
        for _, _, rs in inside:
            for name, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        mhz = [m for _, m, _ in inside]
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(mhz), "window": window}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def coll_device():
    """Device of bench-level collective tensors: the GPU under NCCL, the host under gloo."""
    import torch.distributed as dist

    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def reduce_over_ranks(x: float, world: int, op: str) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
    return float(t.item())


def host_platform():
    """Platform for the end-to-end legs: DeviceA = the box's host cores (all
    but one, which drives the GPU copies), DeviceB = the B200 (group)."""
    from paper_1303_2171_b200.platform import Platform

    return Platform.build(1.0, 3.0, workers_a=max(1, (os.cpu_count() or 2) - 1))


def e2e_share(args, workload, platform, world):
    """`--e2e-share gpu` → all on the GPU; `calibrated` → calibrate_measured
    on this box (the paper's hybrid host+GPU split, measured; untimed);
    `auto` → calibrated at N=1, all-GPU when several ranks share the host."""
    from paper_1303_2171_b200.worksharing import WorkShare, calibrate_measured

    if args.e2e_share == "gpu" or workload is None or (args.e2e_share == "auto" and world > 1):
        return WorkShare.manual(0.0)
    return calibrate_measured(workload, platform, max_refinements=6, repeats=2)


def share_info(wl):
    sh = getattr(wl, "share", None)
    return None if sh is None else round(sh.fraction_a, 4)


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """A page-locked host copy (the bench's e2e inputs)."""
    import torch

    from paper_1303_2171_b200.gpu import _np_to_torch

    t = torch.empty(a.shape, dtype=_np_to_torch(a.dtype), pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


# ---------------------------------------------------------------- workloads
class Bench:
    """One BASELINE workload.  Subclasses define the input, the N=1 step
    (the kernel on device-resident data), the N>1 step (the public API's
    sharded DeviceB path inside gpu_group), the checks and the e2e leg."""

    name = unit = kernel = ""
    per_rank_input = False  # True: each rank holds only its shard (sort)
    always_strong = False   # list ranking: one global list for every N

    def configure(self, rank: int, world: int):
        import torch

        self.rank, self.world = rank, world
        self.mode = "strong" if (ARGS.scaling == "strong" or self.always_strong) else "weak"
        self.g = None
        if world > 1:
            from paper_1303_2171_b200.sharding import group_from_default

            self.g = group_from_default()
        self.stream = torch.cuda.current_stream()

    def group(self):
        from paper_1303_2171_b200.sharding import gpu_group

        return gpu_group(self.g)

    def roofline_extra(self, ms):
        return {}


class HistBench(Bench):
    """BASELINE configs[1]: 256-bin histogram over 2^30 uint8 per GPU."""

    name, unit, kernel = "hist", "Gelem/s", "hist_striped_kernel"
    CONFIG, LARGEST = 1 << 30, 1 << 33

    def __init__(self, seed: int = 42, bins: int = 256):
        self.seed, self.bins = seed, bins

    def setup(self, rank, world):
        import torch

        from paper_1303_2171_b200 import _lib
        from paper_1303_2171_b200.rng import device_splitmix

        self.configure(rank, world)
        base = self.LARGEST if ARGS.shape == "largest" else self.CONFIG
        self.n = base * world if self.mode == "weak" else base
        # the API's input: the whole (global) array on every rank; the sharded
        # run_part counts this rank's floor(k·n/G) slice and all-reduces
        self.x = torch.empty(self.n, dtype=torch.uint8, device="cuda")
        device_splitmix(self.x, self.seed, _lib.HB_GEN_LOW8)
        self.out = torch.empty(self.bins, dtype=torch.int64, device="cuda")
        if world > 1:
            from paper_1303_2171_b200.kernels_regular import HistogramWorkload

            self.wl = HistogramWorkload(self.x, self.bins)
            self.side_b = host_platform().device_b

    def config(self):
        return {"workload": f"hist: 256-bin histogram, 2^{self.n.bit_length() - 1} uint8 global"
                            f" ({self.mode}, floor(k*n/G) shards + all-reduce)",
                "n_global": self.n, "l2": "input > L2: no flush needed"}

    def step(self):
        if self.world == 1:
            from paper_1303_2171_b200.kernels_regular import gpu_histogram

            gpu_histogram(self.x, self.bins, self.out, asynchronous=True)
            return 1
        with self.group():
            self.out = self.wl.run_part(self.side_b, self.x)  # shard + on-device all-reduce
        return 1

    def units_per_step(self):
        return self.n

    def bytes_per_launch(self):
        return self.n // self.world + self.bins * 8

    def verify(self):
        from paper_1303_2171_b200.kernels_regular import gpu_histogram

        if self.world > 1:  # the sharded merge equals the one-GPU count of the whole array
            whole = gpu_histogram(self.x, self.bins)
            return bool(np.array_equal(whole.cpu().numpy(), self.out.cpu().numpy()))
        from oracle import hist as ohist

        m = 1 << 24
        got = gpu_histogram(self.x[:m], self.bins)
        ok = np.array_equal(got.cpu().numpy(), ohist.side_counts(self.x[:m].cpu().numpy(), self.bins, 1))
        return bool(ok and int(self.out.sum().item()) == self.n)

    # e2e: the public API on host buffers; at N>1 the config-size input (strong)
    def e2e_setup(self):
        from paper_1303_2171_b200.kernels_regular import HistogramWorkload

        m = self.CONFIG
        self.host_np = pinned_copy(self.x[:m].cpu().numpy())
        self.platform = host_platform()
        self.share = e2e_share(ARGS, HistogramWorkload(self.host_np, self.bins), self.platform, self.world)
        self.e2e_units = m

    def e2e_pageable(self):
        from paper_1303_2171_b200.kernels_regular import HistogramWorkload

        self.host_np = np.array(self.host_np)  # a plain (pageable) numpy copy
        # a caller calibrates on the buffers it holds: pageable inputs spend
        # host threads on the staging copy, so their best split differs
        self.share = e2e_share(ARGS, HistogramWorkload(self.host_np, self.bins), self.platform, self.world)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_regular import hybrid_histogram

        with self.group():
            return hybrid_histogram(self.host_np, self.bins, self.platform, self.share)

    def e2e_verify(self, res):
        from paper_1303_2171_b200.kernels_regular import gpu_histogram

        ref = gpu_histogram(self.x[: self.e2e_units], self.bins)
        return bool(np.array_equal(np.asarray(res.bins), ref.cpu().numpy()))

    def e2e_bytes(self):
        gpu = self.e2e_units - int(math.floor(self.share.fraction_a * self.e2e_units))
        return gpu // self.world, self.bins * 8

    def cpu_sample(self):
        import bench_reference as br

        return br.hist_leg(self.CONFIG, x=self.host_np)


class SpmvBench(Bench):
    """BASELINE configs[0]: CSR SpMV, 1M x 1M, ~16 nnz/row, fp64 (gen_csr seed
    42, density 1.6e-5, generated on the device bit-identically), rows
    nnz-sorted by the device spmv_preprocess; one step = y = A x over all
    rows, original row order."""

    name, unit, kernel = "spmv", "GFLOP/s", "spmv_sell_kernel"
    CONFIG, LARGEST = 1_000_000, 1 << 24
    AVG_DENSITY_COLS = 16.000000000000004  # 1.6e-5 * 1e6: the config's nnz/row target

    def __init__(self, seed: int = 42):
        self.seed = seed

    def setup(self, rank, world):
        import torch

        from paper_1303_2171_b200.datasets import device_gen_csr
        from paper_1303_2171_b200.kernels_irregular import spmv_preprocess
        from paper_1303_2171_b200.platform import Platform
        from paper_1303_2171_b200.rng import mix_seed, uniform_floats
        from paper_1303_2171_b200.worksharing import WorkShare

        self.configure(rank, world)
        base = self.LARGEST if ARGS.shape == "largest" else self.CONFIG
        self.rows = base * world if self.mode == "weak" else base
        self.density = 1.6e-5 * self.CONFIG / self.rows  # ~16 nnz per row at every size
        m = device_gen_csr(self.rows, self.rows, self.seed, self.density)
        self.nnz = m.nnz
        self.x_host = 2.0 * uniform_floats(mix_seed(self.seed, 0xDEC0), self.rows) - 1.0
        self.x = torch.from_numpy(self.x_host).cuda()
        self.prep = spmv_preprocess(m, Platform.build(1.0, 3.0), WorkShare.manual(0.0))  # on the device
        del m
        self.dm = self.prep.permuted
        self.perm = self.prep.perm
        self.y = torch.empty(self.rows, dtype=torch.float64, device="cuda")

    def config(self):
        return {"workload": f"spmv: CSR {self.rows}x{self.rows}, ~16 nnz/row (nnz {self.nnz}), fp64 bit-exact"
                            f" ({self.mode}, device partitioner + y all-gather)",
                "n_global": self.rows, "l2": "matrix > L2; x L2-resident by design"}

    def step(self):
        if self.world == 1:
            from paper_1303_2171_b200.kernels_irregular import gpu_spmv

            gpu_spmv(self.dm, self.x, 0, self.rows, y=self.y, perm=self.perm, asynchronous=True)
            return 1
        from paper_1303_2171_b200.kernels_irregular import spmv_hybrid

        with self.group():
            self.y = spmv_hybrid(self.prep, self.x)  # partition_nnz + shard + all-gather + hb_scatter_perm
        return 3

    def units_per_step(self):
        return 2 * self.nnz

    def bytes_per_launch(self):
        r = self.rows
        return (12 * self.nnz + 4 * (r + 1) + 8 * r + 12 * r) // self.world + 8 * r * (self.world > 1)

    def verify(self):
        if self.world > 1:  # equals the one-GPU fused path bit for bit
            from paper_1303_2171_b200.kernels_irregular import gpu_spmv

            one = gpu_spmv(self.dm, self.x, 0, self.rows, perm=self.perm)
            return bool(np.array_equal(one.cpu().numpy().view(np.uint64), self.y.cpu().numpy().view(np.uint64)))
        from oracle import spmv as ospmv

        p = self.dm.to_host()
        want = ospmv.hybrid(self.perm.cpu().numpy(), (p.row_ptr, p.col_idx, p.values), 0, self.x_host)
        return bool(np.array_equal(self.y.cpu().numpy().view(np.uint64), want.view(np.uint64)))

    def e2e_setup(self):
        from paper_1303_2171_b200.datasets import csr_arrays
        from paper_1303_2171_b200.kernels_irregular import CsrMatrix, SpmvPrep, SpmvWorkload, spmv_preprocess
        from paper_1303_2171_b200.platform import Platform
        from paper_1303_2171_b200.rng import mix_seed, uniform_floats
        from paper_1303_2171_b200.worksharing import WorkShare

        rows = self.CONFIG
        if self.rows == rows:
            p = self.dm.to_host()
            perm = self.perm.cpu().numpy().astype(np.int64)
        else:  # the config matrix for the N>1 e2e leg (host generator: the API's numpy input)
            ptr, col, val = csr_arrays(rows, rows, self.seed, 1.6e-5)
            pr = spmv_preprocess(CsrMatrix(rows, rows, ptr, col, val), Platform.build(1.0, 3.0), WorkShare.manual(0.0))
            p, perm = pr.permuted, pr.perm
        self.e2e_arrays = (p.row_ptr, p.col_idx, p.values, perm)
        hm = CsrMatrix(p.rows, p.cols, pinned_copy(p.row_ptr), pinned_copy(p.col_idx), pinned_copy(p.values))
        self.hx = pinned_copy(2.0 * uniform_floats(mix_seed(self.seed, 0xDEC0), rows) - 1.0)
        self.platform = host_platform()
        wl = SpmvWorkload(SpmvPrep(hm, perm, 0), self.hx)
        self.share = e2e_share(ARGS, wl, self.platform, self.world)
        split = wl.partition(self.share.fraction_a)[0][1]  # the nnz rule of SpmvWorkload.partition
        self.hprep = SpmvPrep(hm, perm, split, self.platform.device_a.worker_count)
        self.e2e_units = 2 * int(p.row_ptr[-1])

    def e2e_pageable(self):
        from paper_1303_2171_b200.kernels_irregular import CsrMatrix, SpmvPrep, SpmvWorkload

        p = self.hprep.permuted
        hm = CsrMatrix(p.rows, p.cols, np.array(p.row_ptr), np.array(p.col_idx), np.array(p.values))
        perm = np.array(self.hprep.perm)
        self.hx = np.array(self.hx)
        # calibrated on the pageable buffers themselves (see HistBench.e2e_pageable)
        wl = SpmvWorkload(SpmvPrep(hm, perm, 0), self.hx)
        self.share = e2e_share(ARGS, wl, self.platform, self.world)
        split = wl.partition(self.share.fraction_a)[0][1]
        self.hprep = SpmvPrep(hm, perm, split, self.platform.device_a.worker_count)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_irregular import spmv_hybrid

        with self.group():
            return spmv_hybrid(self.hprep, self.hx)

    def e2e_verify(self, y):
        from oracle import spmv as ospmv

        ptr, col, val, perm = self.e2e_arrays
        want = ospmv.hybrid(perm, (ptr, col, val), 0, self.hx)
        return bool(np.array_equal(np.asarray(y).view(np.uint64), want.view(np.uint64)))

    def e2e_bytes(self):
        ptr = self.hprep.permuted.row_ptr
        s = self.hprep.split_row
        nz = int(ptr[-1] - ptr[s])
        rows = self.hprep.permuted.rows
        return (8 * (rows - s + 1) + 16 * nz) // self.world + 8 * rows, 8 * (rows - s) // self.world

    def cpu_sample(self):
        import bench_reference as br

        ptr, col, val, perm = self.e2e_arrays
        # the reference's own spmv_preprocess re-sorts the (already sorted) rows: same split rule
        return br.spmv_leg(self.CONFIG, 1.6e-5, arrays=(ptr, col, val), x=np.asarray(self.hx))


class BilatBench(Bench):
    """BASELINE configs[3]: bilateral filter, 16384 x 16384 image (uint8
    intensities from gen_image — the reference's integer-intensity
    semantics), r=5, sigma_s=2.5, sigma_r=40 (BilatRunner defaults); fp64
    arithmetic bit-identical to the reference, fp32 output image."""

    name, unit, kernel = "bilat", "Mpix/s", "bilateral_tma_kernel"
    compute_bound = "fp64 issue (2 DMUL + 2 DADD per tap)"
    CONFIG, LARGEST = 16384, 32768

    def __init__(self, radius: int = 5, seed: int = 42):
        self.radius, self.seed = radius, seed

    def setup(self, rank, world):
        import torch

        from paper_1303_2171_b200 import _lib
        from paper_1303_2171_b200.rng import device_splitmix

        self.configure(rank, world)
        self.side = self.LARGEST if ARGS.shape == "largest" else self.CONFIG
        self.height = self.side * world if self.mode == "weak" else self.side
        self.img = torch.empty((self.height, self.side), dtype=torch.uint8, device="cuda")
        device_splitmix(self.img, self.seed, _lib.HB_GEN_LOW8)
        self.make_filter()
        self.out = torch.empty((self.height, self.side), dtype=torch.float32, device="cuda")

    def make_filter(self):
        from paper_1303_2171_b200.kernels_regular import build_bilateral_lut

        self.lut = build_bilateral_lut(self.radius, max(self.radius / 2.0, 0.5), 40.0)

    def rows_fn(self, a, b, out=None, arithmetic="fp64"):
        from paper_1303_2171_b200.kernels_regular import gpu_bilateral_rows

        return gpu_bilateral_rows(self.img, self.lut, a, b, out=out, out_dtype=np.float32, asynchronous=True,
                                  arithmetic=arithmetic)

    def extra(self, args):
        """The fp32-arithmetic mode (north_star: filter outputs within 1e-5
        relative), device-resident, N=1: value + agreement with the fp64 kernel."""
        import torch

        if self.world > 1:
            return {}
        for _ in range(3):
            self.rows_fn(0, self.height, out=self.out, arithmetic="fp32")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            self.rows_fn(0, self.height, out=self.out, arithmetic="fp32")
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
        ref = self.rows_fn(0, self.height)  # fp64 taps
        torch.cuda.synchronize()
        err = float(((self.out.double() - ref.double()).abs() / ref.double().abs().clamp_min(1e-30)).max())
        return {"fp32": {"value": self.units_per_step() / (ms / 1e3) / 1e6, "ms_per_step": ms,
                         "max_rel_err_vs_fp64": err, "parity": err <= 1e-5}}

    def config(self):
        return {"workload": f"{self.name}: {self.height}x{self.side} image, {2 * self.radius + 1}x{2 * self.radius + 1}"
                            f" taps fp64, fp32 out ({self.mode}, row strips + all-gather)",
                "n_global": self.height * self.side, "l2": "input + output > L2"}

    def step(self):
        if self.world == 1:
            self.rows_fn(0, self.height, out=self.out)
            return 1
        from paper_1303_2171_b200 import sharding

        with self.group():  # the strip split + all-gather of BilateralApplyWorkload.run_part(DeviceB)
            self.out = sharding.run_sharded_rows(0, self.height, self.rows_fn)
        return 1

    def units_per_step(self):
        return self.height * self.side

    def bytes_per_launch(self):
        return self.height * self.side * (1 + 4) // self.world

    def flops_per_launch(self):
        return self.height * self.side * (2 * self.radius + 1) ** 2 * 4 // self.world

    def roofline_extra(self, ms):
        ach = self.flops_per_launch() / (ms / 1e3) / 1e9
        return {"compute": {"bound": self.compute_bound, "achieved_gflops": ach, "peak_gflops": FP64_PEAK_GFLOPS,
                            "frac": ach / FP64_PEAK_GFLOPS}}

    def _oracle_rows(self, host, a, b):
        from oracle import bilateral as obil

        sp, rg = obil.lut(self.radius, max(self.radius / 2.0, 0.5), 40.0)
        return obil.rows(host, sp, rg, self.radius, a, b)

    def verify(self):
        if self.world > 1:
            import torch

            one = self.rows_fn(0, self.height)
            return bool(torch.equal(one, self.out))
        host = self.img.cpu().numpy()
        ok = True
        for a, b in [(0, 8), (8000, 8008), (self.height - 8, self.height)]:
            ok &= np.array_equal(self.out[a:b].cpu().numpy(), self._oracle_rows(host, a, b).astype(np.float32))
        return bool(ok)

    def e2e_setup(self):
        from paper_1303_2171_b200.kernels_regular import Image

        self.e2e_side = self.CONFIG
        self.host = pinned_copy(self.img[: self.e2e_side, : self.e2e_side].contiguous().cpu().numpy())
        self.image = Image(self.host)
        self.platform = host_platform()
        self.share = e2e_share(ARGS, self.e2e_workload(), self.platform, self.world)
        self.e2e_units = self.e2e_side * self.e2e_side

    def e2e_pageable(self):
        from paper_1303_2171_b200.kernels_regular import Image

        self.host = np.array(self.host)
        self.image = Image(self.host)

    def e2e_workload(self):
        from paper_1303_2171_b200.kernels_regular import BilateralApplyWorkload

        return BilateralApplyWorkload(self.image, self.lut)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_regular import hybrid_bilateral

        with self.group():
            return hybrid_bilateral(self.image, self.lut, self.platform, self.share)

    def e2e_verify(self, img):
        out = np.asarray(img.pixels)
        s = self.e2e_side
        split = int(math.floor(self.share.fraction_a * s))
        rows = {(0, 4), (max(0, split - 2), min(s, split + 2)), (8000, 8004), (s - 4, s)}
        return bool(all(np.array_equal(out[a:b].view(np.uint64), self._oracle_rows(self.host, a, b).view(np.uint64))
                        for a, b in rows if b > a))

    def e2e_bytes(self):
        gpu_rows = self.e2e_side - int(math.floor(self.share.fraction_a * self.e2e_side))
        return gpu_rows * self.e2e_side // self.world, gpu_rows * self.e2e_side * 8

    def cpu_sample(self):
        import bench_reference as br

        return br.filter_leg(self.name, self.e2e_side, self.radius, img=self.host[: 64 + self.radius])


class ConvBench(BilatBench):
    """Convolution (not a BASELINE config): 16384 x 16384 uint8
    image, 15 x 15 Gaussian (FilterKernel.gaussian(7)), fp64 arithmetic
    bit-identical to the reference, fp32 output image."""

    name, kernel = "conv", "conv_rows_kernel"
    compute_bound = "fp64 issue (1 DMUL + 1 DADD per tap)"

    def __init__(self, radius: int = 7, seed: int = 42):
        super().__init__(radius, seed)

    def make_filter(self):
        from paper_1303_2171_b200.kernels_regular import FilterKernel

        self.fk = FilterKernel.gaussian(self.radius)

    def rows_fn(self, a, b, out=None, arithmetic="fp64"):
        from paper_1303_2171_b200.kernels_regular import gpu_convolve_rows

        return gpu_convolve_rows(self.img, self.fk, a, b, out=out, out_dtype=np.float32, asynchronous=True,
                                 arithmetic=arithmetic)

    def flops_per_launch(self):
        return self.height * self.side * (2 * self.radius + 1) ** 2 * 2 // self.world

    def _oracle_rows(self, host, a, b):
        from oracle import conv as oconv

        return oconv.rows(host, self.fk.weights, a, b)

    def e2e_workload(self):
        from paper_1303_2171_b200.kernels_regular import ConvolutionWorkload

        return ConvolutionWorkload(self.image, self.fk)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_regular import hybrid_convolve

        with self.group():
            return hybrid_convolve(self.image, self.fk, self.platform, self.share)


class SortBench(Bench):
    """BASELINE configs[2]: LSD radix sort of 2^28 uint32 keys + uint32
    payload (gen_sort_data keys, payload = global index) per GPU; at N>1 the
    sample-merge exchange (local sort, splitters, all-to-all, G-way merge)."""

    name, unit, kernel = "sort", "Mkeys/s", "onesweep_rfk_kernel"
    CONFIG, LARGEST = 1 << 28, 1 << 29
    per_rank_input = True

    def __init__(self, seed: int = 42):
        self.seed = seed

    def setup(self, rank, world):
        import torch

        self.configure(rank, world)
        base = self.LARGEST if ARGS.shape == "largest" else self.CONFIG
        self.n = base * world if self.mode == "weak" else base
        from paper_1303_2171_b200.sharding import shard_range

        self.lo, self.hi = shard_range(self.n, rank, world)  # this rank's slice of the global keys
        m = self.hi - self.lo
        self.keys = torch.empty(m, dtype=torch.int32, device="cuda")
        self.vals = torch.empty(m, dtype=torch.int32, device="cuda")
        self.prepare_step()

    def prepare_step(self):
        import torch

        from paper_1303_2171_b200 import _lib
        from paper_1303_2171_b200.rng import device_splitmix

        device_splitmix(self.keys, self.seed, _lib.HB_GEN_HI32, k0=self.lo)
        torch.arange(self.lo, self.hi, dtype=torch.int32, out=self.vals)

    def config(self):
        return {"workload": f"sort: LSD radix 2^{self.n.bit_length() - 1} uint32 keys + payload global"
                            f" ({self.mode}; N>1 sample-merge)",
                "n_global": self.n, "l2": "keys+payload > L2; regenerated before every step (untimed)",
                "algorithmic_bytes": "68 B/key: 4 (digit histogram) + 4 passes x 16"}

    def step(self):
        if self.world == 1:
            from paper_1303_2171_b200 import _lib
            from paper_1303_2171_b200.gpu import current_stream_handle, vp

            _lib.call("hb_sort", vp(self.keys.data_ptr()), vp(self.keys.data_ptr()), _lib.DTYPE_CODES["u4"],
                      vp(self.vals.data_ptr()), vp(self.vals.data_ptr()), self.keys.numel(), None,
                      _lib.HB_DEVICE_PTRS | _lib.HB_ASYNC, current_stream_handle(self.keys))
            return 1 + 4
        import torch

        from paper_1303_2171_b200.sort_exchange import exchange_sort

        self.out_k, self.out_v = exchange_sort(self.keys.view(torch.uint32), self.vals, self.g)
        return 5 + 1 + max(1, math.ceil(math.log2(self.world)))

    def units_per_step(self):
        return self.n

    def bytes_per_launch(self):
        return (self.hi - self.lo) * 68

    def verify(self):
        import torch

        from oracle import sort as osort
        from oracle.rng import draws

        if self.world == 1:
            k = self.keys.cpu().numpy().view(np.uint32)
            v = self.vals.cpu().numpy()
            torch.cuda.synchronize()
            self.prepare_step()
            keys_in = self.keys.cpu().numpy().view(np.uint32)
            return bool(np.array_equal(k, np.sort(keys_in)) and osort.check_stable_payload(keys_in, k, v))
        # distributed output: every rank's interval sorted by (key, index),
        # intervals in rank order, nothing lost, payload = the key's index
        from paper_1303_2171_b200.sharding import all_gather_small

        k = self.out_k.view(torch.int32).cpu().numpy().view(np.uint32).astype(np.int64)
        v = self.out_v.cpu().numpy().astype(np.int64)
        ok = bool(np.all((k[1:] > k[:-1]) | ((k[1:] == k[:-1]) & (v[1:] > v[:-1]))))
        pick = np.unique(np.linspace(0, max(k.size - 1, 0), 4096).astype(np.int64)) if k.size else np.zeros(0, np.int64)
        want = np.array([int(draws(self.seed, 1, int(i) + 1)[0] >> np.uint64(32)) for i in v[pick]], dtype=np.int64)
        ok &= np.array_equal(k[pick], want)
        edge = torch.tensor([k[0] if k.size else -1, k[-1] if k.size else -1, k.size, int(v.sum())],
                            dtype=torch.int64, device="cuda")
        allp = all_gather_small(edge, self.g).cpu().numpy()
        firsts, lasts, counts = allp[:, 0], allp[:, 1], allp[:, 2]
        ok &= int(counts.sum()) == self.n and int(allp[:, 3].sum()) == self.n * (self.n - 1) // 2
        nz = counts > 0
        ok &= bool(np.all(lasts[nz][:-1] <= firsts[nz][1:]))
        return bool(ok)

    def e2e_setup(self):
        m = self.CONFIG
        from paper_1303_2171_b200.datasets import device_gen_sort_data

        self.host_np = pinned_copy(device_gen_sort_data(m, self.seed).cpu().numpy().view(np.uint32))
        self.platform = host_platform()
        from paper_1303_2171_b200.worksharing import WorkShare

        self.share = WorkShare.manual(0.0)
        self.e2e_units = m

    def e2e_pageable(self):
        self.host_np = np.array(self.host_np)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_regular import sample_sort_hybrid

        with self.group():
            return sample_sort_hybrid(self.host_np, self.platform, share=self.share)

    def e2e_verify(self, res):
        """Sorted, same multiset as the input (count, sum, xor) — O(n)."""
        k = np.asarray(res[0]).view(np.uint32)
        src = self.host_np
        ok = k.size == src.size and bool(np.all(k[1:] >= k[:-1]))
        ok = ok and int(k.sum(dtype=np.uint64)) == int(src.sum(dtype=np.uint64))
        return bool(ok and int(np.bitwise_xor.reduce(k)) == int(np.bitwise_xor.reduce(src)))

    def e2e_bytes(self):
        return 4 * self.e2e_units, 4 * self.e2e_units

    def cpu_sample(self):
        import bench_reference as br

        return br.sort_leg(self.CONFIG, keys=self.host_np)


class LrBench(Bench):
    """BASELINE configs[4]: list ranking of a 2^28-node random linked list
    (gen_list(2^28, 42), generated on the device bit-identically), succ int32,
    ranks int64; N>1: the sharded sublist ranking (strong scaling)."""

    name, unit, kernel = "lr", "Mnodes/s", "lr_walk_log_kernel"
    CONFIG, LARGEST = 1 << 28, 1 << 29
    always_strong = True

    def __init__(self, seed: int = 42):
        self.seed = seed

    def setup(self, rank, world):
        import torch

        from paper_1303_2171_b200.datasets import device_gen_list

        self.configure(rank, world)
        self.n = self.LARGEST if ARGS.shape == "largest" else self.CONFIG
        self.succ, self.head = device_gen_list(self.n, self.seed)  # the same list on every rank
        self.rank_out = torch.empty(self.n, dtype=torch.int64, device="cuda")

    def config(self):
        return {"workload": f"lr: list ranking, 2^{self.n.bit_length() - 1}-node random list"
                            f" (strong; N>1 sublists split over GPUs + summary all-gather)",
                "n_global": self.n, "l2": "succ + rank > L2",
                "algorithmic_bytes": "12 B/node (4 succ + 8 rank)"}

    def step(self):
        from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

        with self.group():
            gpu_list_rank(self.succ, self.head, out=self.rank_out)
        return 8

    def units_per_step(self):
        return self.n

    def bytes_per_launch(self):
        return 12 * self.n // self.world

    # log ~8.3 + node sort: 2 digit passes x 16 over ~1.03 n log slots (the walk counts the digit
    # histograms; the first pass reads the log itself) + the bucket finish 16 (8 read + 8 int64 rank)
    SEQ_BYTES_PER_NODE = 58

    def roofline_extra(self, ms):
        # t >= one dependent random successor read per node at the measured
        # rate + the sequential passes (log, pairs, node sort, widen) at HBM peak
        n = self.n // self.world
        peak, _ = hbm_peak()
        bound_ms = (n / RANDOM_READ_PEAK / 1e9 + n * self.SEQ_BYTES_PER_NODE / (peak * 1e9)) * 1e3
        return {"random_access": {"bound_ms": bound_ms, "frac": bound_ms / ms,
                                  "peak_read_g_per_s": RANDOM_READ_PEAK,
                                  "seq_bytes_per_node": self.SEQ_BYTES_PER_NODE}}

    def verify(self):
        if self.world > 1:
            import torch

            from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

            one = gpu_list_rank(self.succ, self.head)  # no group: the one-GPU ranking
            return bool(torch.equal(one, self.rank_out))
        s = self.succ.cpu().numpy().astype(np.int64)
        r = self.rank_out.cpu().numpy()
        inner = s >= 0
        ok = r[self.head] == 0 and np.array_equal(r[s[inner]], r[inner] + 1)
        return bool(ok and np.array_equal(np.bincount(r, minlength=self.n), np.ones(self.n, dtype=np.int64)))

    def e2e_setup(self):
        from paper_1303_2171_b200.kernels_irregular import LinkedListArr

        self.host = pinned_copy(self.succ.cpu().numpy().astype(np.int64))
        self.lst = LinkedListArr(self.host, self.head)
        self.platform = host_platform()
        self.share = None
        self.e2e_units = self.n

    def e2e_pageable(self):
        from paper_1303_2171_b200.kernels_irregular import LinkedListArr

        self.host = np.array(self.host)
        self.lst = LinkedListArr(self.host, self.head)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_irregular import list_rank_hybrid

        with self.group():
            return list_rank_hybrid(self.lst, self.platform, self.seed)

    def e2e_verify(self, rank):
        return bool(np.array_equal(np.asarray(rank), self.rank_out.cpu().numpy()))

    def e2e_bytes(self):
        return 8 * self.n, 8 * self.n

    def cpu_sample(self):
        import bench_reference as br

        return br.lr_leg(self.n)


WORKLOADS = {"hist": HistBench, "spmv": SpmvBench, "bilat": BilatBench, "conv": ConvBench, "sort": SortBench,
             "lr": LrBench}


# ---------------------------------------------------------------- drivers
def time_cpu(fn, reps: int, warm: int = 1):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return ts


def scale_of(unit: str) -> float:
    return 1e9 if unit.startswith("G") else 1e6


def run_reference(args, name: str) -> dict | None:
    """--impl reference: the unmodified reference (baseline/_ref) on the host
    cores, on this arm's config; rank 0 only (the other ranks exit 0)."""
    import bench_reference as br

    rank, world, _ = dist_env()
    if rank != 0:
        return None
    units_name = {"hist": "Gelem/s", "spmv": "GFLOP/s", "bilat": "Mpix/s", "conv": "Mpix/s", "sort": "Mkeys/s",
                  "lr": "Mnodes/s"}[name]
    if name == "hist":
        fn, units, sample, cores, kind, same = br.hist_leg(HistBench.CONFIG)
    elif name == "spmv":
        fn, units, sample, cores, kind, same = br.spmv_leg(SpmvBench.CONFIG, 1.6e-5)
    elif name == "sort":
        fn, units, sample, cores, kind, same = br.sort_leg(SortBench.CONFIG)
    elif name == "lr":
        fn, units, sample, cores, kind, same = br.lr_leg(LrBench.CONFIG)
    else:
        fn, units, sample, cores, kind, same = br.filter_leg(name, 16384, 5 if name == "bilat" else 7)
    ts = time_cpu(fn, args.steps, warm=args.warmup)
    t = statistics.median(ts)
    val = units / t / scale_of(units_name)
    return {
        "metric": METRIC, "impl": "reference", "value": val, "unit": units_name, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8" if name == "hist" else "f64", "data": "synthetic",
        "config": {"workload": {"hist": "hist: 256-bin histogram, 2^30 uint8 global"}.get(name, name),
                   "same_config": same},
        "cpu_baseline": {"value": val, "unit": units_name, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": val, "unit": units_name, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_package": "baseline/_ref/hybridbench" if kind == "reference" else "oracle port (baseline/_ref missing)",
    }


def measure(args, wl, rank, world, with_cpu: bool) -> dict:
    import torch

    wl.setup(rank, world)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    with ClockSampler(torch.cuda.current_device()) as clocks:
        for _ in range(args.warmup):
            if hasattr(wl, "prepare_step"):
                wl.prepare_step()
            wl.step()
        torch.cuda.synchronize()
        barrier(world)
        launches = 0
        prep = getattr(wl, "prepare_step", None)
        t0 = time.perf_counter()
        if prep is None:
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(stream)
            for _ in range(args.steps):
                launches += wl.step()
            end.record(stream)
            torch.cuda.synchronize()
            ms = start.elapsed_time(end) / args.steps
        else:
            # inputs consumed in place: regenerated (untimed) between timed steps
            pairs = []
            for _ in range(args.steps):
                prep()
                torch.cuda.synchronize()
                barrier(world)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                launches += wl.step()
                b.record(stream)
                pairs.append((a, b))
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in pairs) / args.steps
        t1 = time.perf_counter()
        clk = clocks.summary(t0, t1)
    ms = reduce_over_ranks(ms, world, "max")
    ok = reduce_over_ranks(float(wl.verify()), world, "min") == 1.0
    extra = wl.extra(args) if hasattr(wl, "extra") else {}

    # end to end through the public API (host buffers)
    wl.e2e_setup()
    for _ in range(args.warmup):  # untimed: device memory pools and pinned stages settle
        wl.e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    e_steps = max(1, min(args.steps, args.e2e_steps))
    e0 = time.perf_counter()
    last = None
    for _ in range(e_steps):
        last = None  # a caller drops the previous result first (its pinned block is reused)
        last = wl.e2e_step()
    torch.cuda.synchronize()
    e_s = (time.perf_counter() - e0) / e_steps
    barrier(world)
    e_s = reduce_over_ranks(e_s, world, "max")
    e_ok = reduce_over_ranks(float(wl.e2e_verify(last)), world, "min") == 1.0
    del last

    pinned_share = share_info(wl)
    h2d, d2h = wl.e2e_bytes()

    # the same API on what a plain caller holds: pageable numpy inputs, and
    # every result kept (no pinned block recycled between calls)
    wl.e2e_pageable()
    wl.e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    p_steps = max(1, min(3, e_steps))
    kept = []
    p0 = time.perf_counter()
    for _ in range(p_steps):
        kept.append(wl.e2e_step())
    torch.cuda.synchronize()
    p_s = (time.perf_counter() - p0) / p_steps
    barrier(world)
    p_s = reduce_over_ranks(p_s, world, "max")
    p_ok = reduce_over_ranks(float(wl.e2e_verify(kept[-1])), world, "min") == 1.0
    del kept

    scale = scale_of(wl.unit)
    value = wl.units_per_step() / (ms / 1e3) / scale
    peak, peak_src = hbm_peak()
    achieved = wl.bytes_per_launch() / (ms / 1e3) / 1e9
    res = {
        "value": value, "unit": wl.unit, "ms_per_step": ms, "parity": ok, "gpu_launches": launches,
        "scaling": wl.mode,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic_of(wl.kernel), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": wl.bytes_per_launch(), "kernel": wl.kernel,
                     **wl.roofline_extra(ms)},
        "e2e": {"value": wl.e2e_units / e_s / scale, "unit": wl.unit, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e_s * 1e3, "steps": e_steps,
                "share": pinned_share, "parity": e_ok, "units": wl.e2e_units,
                "api": "public drop-in entry point, host buffers" + (" under gpu_group" if world > 1 else ""),
                "inputs": "page-locked host arrays; each step's result dropped before the next call",
                "pageable": {"value": wl.e2e_units / p_s / scale, "ms_per_step": p_s * 1e3, "steps": p_steps,
                             "parity": p_ok, "share": share_info(wl),
                             "inputs": "pageable numpy arrays, every result kept (what a plain caller does)"}},
        "clocks": clk,
        "config": wl.config(),
        **extra,
    }
    if with_cpu and rank == 0:
        fn, units, sample, cores, kind, _ = wl.cpu_sample()
        ts = time_cpu(fn, 1, warm=0)
        res["cpu_baseline"] = {"value": units / min(ts) / scale, "unit": wl.unit, "cores": cores, "kind": kind,
                               "sample": sample}
    return res


def compact(res: dict) -> dict:
    """One workload in a few hundred bytes (the driver keeps ~3 KB of stdout)."""
    rl = res["roofline"]
    out = {"v": round(res["value"], 2), "u": res["unit"], "ms": round(res["ms_per_step"], 4),
           "hbm_frac": round(rl["frac"], 3), "e2e": round(res["e2e"]["value"], 2),
           "e2e_pageable": round(res["e2e"]["pageable"]["value"], 2),
           "e2e_share": res["e2e"]["share"], "ok": bool(res["parity"] and res["e2e"]["parity"] and res["e2e"]["pageable"]["parity"]),
           "n": res["config"]["n_global"]}
    if "compute" in rl:
        out["fp64_frac"] = round(rl["compute"]["frac"], 3)
    if "fp32" in res:
        out["v_fp32"] = round(res["fp32"]["value"], 1)
        out["ok"] = out["ok"] and bool(res["fp32"]["parity"])
    if "random_access" in rl:
        out["ra_frac"] = round(rl["random_access"]["frac"], 3)
    if "cpu_baseline" in res:
        out["cpu"] = float(f"{res['cpu_baseline']['value']:.4g}")
        out["cpu_kind"] = res["cpu_baseline"]["kind"]
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="all", choices=sorted(WORKLOADS) + ["all"])
    ap.add_argument("--e2e-steps", type=int, default=10, help="steps of the end-to-end (host buffer) leg")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--shape", default="config", choices=["config", "largest"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--e2e-share", default="auto", choices=["auto", "calibrated", "gpu"])
    args = ap.parse_args()
    global ARGS
    ARGS = args
    args.warmup = max(args.warmup, 3)

    rank, world, local = dist_env()
    headline = "hist" if args.workload == "all" else args.workload

    if args.impl == "reference":
        out = run_reference(args, headline)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch

    # HB_BENCH_BACKEND=gloo + more ranks than GPUs: a functional check of the
    # multi-rank paths on a 1-GPU box (ranks share the device; not a timing)
    backend = os.environ.get("HB_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_1303_2171_b200.gpu import require_gpu

    require_gpu()

    def fresh_memory():
        # each workload starts from the memory state of a standalone run
        import gc

        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        if hasattr(torch._C, "_host_emptyCache"):
            torch._C._host_emptyCache()

    with_cpu = world == 1 and not args.no_cpu
    results = {headline: measure(args, WORKLOADS[headline](), rank, world, with_cpu)}
    if args.workload == "all":
        for name, cls in WORKLOADS.items():
            if name != headline:
                fresh_memory()
                results[name] = measure(args, cls(), rank, world, with_cpu)
    if rank == 0:
        head = results[headline]
        rl = head["roofline"]
        line = {
            "metric": METRIC, "value": head["value"], "unit": head["unit"], "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": head["scaling"], "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (reference generator streams, seed 42, device-generated)",
            "config": {**head["config"], "parallelism": f"shard{world}", "backend": backend if world > 1 else None},
            "roofline": {k: rl[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
            "e2e": {**{k: head["e2e"][k] for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step",
                                                    "share", "parity")},
                    "pageable": round(head["e2e"]["pageable"]["value"], 3)},
            "gpu_launches": head["gpu_launches"],
            "clocks": {k: head["clocks"][k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "parity": head["parity"],
        }
        if "cpu_baseline" in head:
            line["cpu_baseline"] = head["cpu_baseline"]
        if len(results) > 1:
            line["workloads"] = {k: compact(v) for k, v in results.items() if k != headline}
        try:
            DETAIL_FILE.parent.mkdir(exist_ok=True)
            DETAIL_FILE.write_text(json.dumps({"argv": sys.argv, "world": world, "results": results}, indent=1))
        except OSError:
            pass
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
