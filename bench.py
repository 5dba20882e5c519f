"""Benchmark driver for the B200 work-partitioned hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload hist|…|all]
                    [--impl ours|reference]

Prints ONE JSON line (rank 0).  At N=1 the headline workload is BASELINE.json
configs[1] — 256-bin histogram over 2^30 uint8 elements — and every other
configured workload is measured in the same run under "workloads".  A step is
one pass of the hot path over one batch of synthetic input already resident
in HBM (`value`); `e2e` is the same metric through the public drop-in API
(`hybrid_histogram(...)` on pinned host buffers, H2D + D2H inside the timed
region).  Under torchrun (N>1) every rank holds its own shard (weak scaling)
and the per-step merge is the workload's real collective (NCCL).

`--impl reference` times the reference's own CPU algorithm (the numpy
restatement under oracle/, the reference being pure Python) on the host
cores, rank 0 only.
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

ARGS = argparse.Namespace(e2e_share="auto")  # set by main()

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
TRAFFIC_FILE = ROOT / "profiles" / "traffic.json"
def e2e_share_info(wl):
    sh = getattr(wl, "share", None)
    if sh is None:
        return None
    pf = getattr(wl, "platform", None)
    return {"fraction_a": sh.fraction_a, "origin": sh.origin.value,
            "host_workers": pf.device_a.worker_count if pf is not None else None,
            "note": "fraction_a of the input computed on the host cores (native hb_host_* threads), the rest on the B200"}


def host_platform():
    """Platform for the end-to-end legs: DeviceA = the box's host cores (all
    but one, which drives the GPU copies), DeviceB = the B200."""
    from paper_1303_2171_b200.platform import Platform

    return Platform.build(1.0, 3.0, workers_a=max(1, (os.cpu_count() or 2) - 1))


def e2e_share(args, workload, platform):
    """The split the e2e leg runs with: `--e2e-share gpu` → all on the GPU;
    `calibrated` → worksharing.calibrate_measured on this box (the paper's
    hybrid host+GPU split, measured, not modelled; untimed); `auto` (default)
    → calibrated at N=1, all on the GPU when several ranks share the host."""
    from paper_1303_2171_b200.worksharing import WorkShare, calibrate_measured

    import torch.distributed as dist

    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
    if args.e2e_share == "gpu" or workload is None or (args.e2e_share == "auto" and multi):
        # N > 1: the ranks share one host's cores, so the host share is off
        return WorkShare.manual(0.0)
    return calibrate_measured(workload, platform, max_refinements=6, repeats=2)


RANDOM_READ_PEAK = 51.5   # G random 4-B DRAM reads/s, scripts/micro/gather.cu
RANDOM_WRITE_PEAK = 24.8  # G random 8-B DRAM writes/s (read-fill + write), same micro
FP64_PEAK_GFLOPS = 18370.0  # non-FMA fp64 instructions/s, scripts/micro/fp64peak.cu
METRIC = "per-workload throughput (SpMV GFLOP/s, sort Mkeys/s) and HBM-roofline fraction"


# ---------------------------------------------------------------- utilities
def hbm_peak() -> tuple[float, str]:
    try:
        return float(json.loads(PEAKS_FILE.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_of(kernel: str):
    try:
        return json.loads(TRAFFIC_FILE.read_text()).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """Polls NVML (SM clock + clock-event reasons) on a thread; `window()`
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
        return {
            "sm_mhz": statistics.median(mhz) if mhz else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(reasons),
            "samples": len(mhz),
            "window": window,
        }


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def coll_device():
    """Device of bench-level collective tensors: the GPU under NCCL, the host under gloo."""
    import torch.distributed as dist

    return "cuda" if dist.get_backend() == "nccl" else "cpu"


# ---------------------------------------------------------------- workloads
class HistBench:
    """BASELINE configs[1]: 256-bin histogram over 2^30 uint8 (per GPU)."""

    name = "hist"
    unit = "Gelem/s"
    kernel = "hist_striped_kernel"

    def __init__(self, n: int = 1 << 30, bins: int = 256, seed: int = 42):
        self.n, self.bins, self.seed = n, bins, seed

    def config(self):
        return {"workload": f"hist: 256-bin histogram over 2^{self.n.bit_length() - 1} uint8 per GPU",
                "n_per_gpu": self.n, "bins": self.bins, "seed": self.seed,
                "input": "gen_hist_data(n, 42) low byte (splitmix64, device-generated)",
                "l2": "input (1 GiB) > L2 (126 MB): no flush needed"}

    def setup(self, rank, world):
        import torch

        from paper_1303_2171_b200 import _lib
        from paper_1303_2171_b200.rng import device_splitmix

        self.x = torch.empty(self.n, dtype=torch.uint8, device="cuda")
        device_splitmix(self.x, self.seed, _lib.HB_GEN_LOW8, k0=rank * self.n)
        self.out = torch.empty(self.bins, dtype=torch.int64, device="cuda")
        self.world = world

    def step(self):
        from paper_1303_2171_b200.kernels_regular import gpu_histogram

        gpu_histogram(self.x, self.bins, self.out, asynchronous=True)
        if self.world > 1:
            import torch.distributed as dist

            if coll_device() == "cuda":
                dist.all_reduce(self.out)
            else:
                t = self.out.cpu()
                dist.all_reduce(t)
                self.out.copy_(t)
        return 1  # libhb200 kernels launched

    def units_per_step(self):
        return self.n

    def bytes_per_launch(self):
        return self.n * 1 + self.bins * 8

    def verify(self):
        import torch

        from oracle import hist as ohist

        # sampled check on the host: the first 2^24 elements vs the oracle
        m = 1 << 24
        part = self.x[:m]
        got = torch.empty(self.bins, dtype=torch.int64, device="cuda")
        from paper_1303_2171_b200.kernels_regular import gpu_histogram

        gpu_histogram(part, self.bins, got)
        host = part.cpu().numpy()
        ok = np.array_equal(got.cpu().numpy(), ohist.side_counts(host, self.bins, 1))
        full = int(self.out.sum().item()) == self.n * self.world
        return bool(ok and full)

    # end-to-end through the public drop-in API, pinned host buffers
    def e2e_setup(self):
        import torch

        self.host = torch.empty(self.n, dtype=torch.uint8, pin_memory=True)
        self.host.copy_(self.x)
        self.host_np = self.host.numpy()
        from paper_1303_2171_b200.kernels_regular import HistogramWorkload

        self.platform = host_platform()
        self.share = e2e_share(ARGS, HistogramWorkload(self.host_np, self.bins), self.platform)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_regular import hybrid_histogram

        res = hybrid_histogram(self.host_np, self.bins, self.platform, self.share)
        if self.world > 1:
            import torch
            import torch.distributed as dist

            t = torch.from_numpy(res.bins).to(coll_device(), copy=True)  # the reduce must not alias res
            dist.all_reduce(t)
        return res

    def e2e_verify(self, res):
        """The e2e result (host+GPU split) equals the device histogram of the same data."""
        import torch

        from paper_1303_2171_b200.kernels_regular import gpu_histogram

        ref = torch.zeros(self.bins, dtype=torch.int64, device="cuda")
        gpu_histogram(self.x, self.bins, ref)
        return bool(np.array_equal(np.asarray(res.bins), ref.cpu().numpy()))

    def e2e_bytes(self):
        return self.n - int(math.floor(self.share.fraction_a * self.n)), self.bins * 8

    # CPU baseline: the reference algorithm (oracle port) on a bounded sample
    def cpu_sample(self, budget_s: float):
        from oracle import hist as ohist

        m = min(self.n, 1 << 28)
        host = self.x[:m].cpu().numpy()
        fn = lambda: ohist.hybrid(host, self.bins, 0.25)  # noqa: E731
        return fn, m, f"{m} uint8 elements of the same stream (2^{m.bit_length() - 1}), formula share 0.25, 2 sides x 4 workers"

    def cpu_cores(self):
        return 2


class SpmvBench:
    """BASELINE configs[0]: CSR SpMV, 1M x 1M, ~16 nnz/row, fp64 (gen_csr seed 42,
    density 1.6e-5), rows nnz-sorted by spmv_preprocess; one step = y = A x
    over all rows with the inverse permutation fused into the store."""

    name = "spmv"
    unit = "GFLOP/s"
    kernel = "spmv_lpr_kernel"

    def __init__(self, rows: int = 1_000_000, density: float = 1.6e-5, seed: int = 42):
        self.rows, self.density, self.seed = rows, density, seed

    def config(self):
        return {"workload": f"spmv: CSR {self.rows}x{self.rows}, density {self.density} (~16 nnz/row), fp64, bit-exact row sums",
                "rows": self.rows, "nnz": int(self.nnz), "seed": self.seed,
                "input": "gen_csr(rows, rows, 42, 1.6e-5) + x = 2*uniform_floats(mix_seed(42,0xDEC0))-1",
                "l2": "matrix (204 MB) > L2 (126 MB); x (8 MB) L2-resident by design"}

    def setup(self, rank, world):
        import torch

        from paper_1303_2171_b200.datasets import csr_arrays
        from paper_1303_2171_b200.kernels_irregular import CsrMatrix, spmv_preprocess
        from paper_1303_2171_b200.platform import Platform
        from paper_1303_2171_b200.rng import mix_seed, uniform_floats
        from paper_1303_2171_b200.worksharing import WorkShare

        ptr, col, val = csr_arrays(self.rows, self.rows, self.seed, self.density)
        self.m = CsrMatrix(self.rows, self.rows, ptr, col, val)
        self.nnz = self.m.nnz
        self.x_host = 2.0 * uniform_floats(mix_seed(self.seed, 0xDEC0), self.rows) - 1.0
        self.platform = Platform.build(1.0, 3.0)
        self.prep = spmv_preprocess(self.m, self.platform, WorkShare.manual(0.0))
        self.dm = self.prep.permuted.to_device(np.int32)
        self.x = torch.from_numpy(self.x_host).cuda()
        self.perm = torch.from_numpy(np.asarray(self.prep.perm, dtype=np.int32)).cuda()
        self.y = torch.empty(self.rows, dtype=torch.float64, device="cuda")
        self.world = world

    def step(self):
        from paper_1303_2171_b200.kernels_irregular import gpu_spmv

        gpu_spmv(self.dm, self.x, 0, self.rows, y=self.y, perm=self.perm, asynchronous=True)
        return 1

    def units_per_step(self):
        return 2 * self.nnz  # flops

    def bytes_per_launch(self):
        r = self.rows
        return 12 * self.nnz + 4 * (r + 1) + 8 * r + 8 * r + 4 * r  # val+col, row_ptr, x, y, perm

    def verify(self):
        from oracle import spmv as ospmv

        p = self.prep.permuted
        want = ospmv.hybrid(self.prep.perm, (p.row_ptr, p.col_idx, p.values), 0, self.x_host)
        return bool(np.array_equal(self.y.cpu().numpy().view(np.uint64), want.view(np.uint64)))

    def e2e_setup(self):
        import torch

        from paper_1303_2171_b200.kernels_irregular import CsrMatrix, SpmvPrep

        def pinned(a):
            t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
            t.numpy()[...] = a
            return t.numpy()

        from paper_1303_2171_b200.kernels_irregular import SpmvWorkload

        p = self.prep.permuted
        hm = CsrMatrix(p.rows, p.cols, pinned(p.row_ptr), pinned(p.col_idx), pinned(p.values))
        self.hx = pinned(self.x_host)
        self.platform = host_platform()
        wl = SpmvWorkload(SpmvPrep(hm, self.prep.perm, 0), self.hx)
        self.share = e2e_share(ARGS, wl, self.platform)
        split = wl.partition(self.share.fraction_a)[0][1]  # the nnz rule of SpmvWorkload.partition
        self.hprep = SpmvPrep(hm, self.prep.perm, split, self.platform.device_a.worker_count)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_irregular import spmv_hybrid

        return spmv_hybrid(self.hprep, self.hx)

    def e2e_verify(self, y):
        """Bit-exact against the oracle (original row order)."""
        from oracle import spmv as ospmv

        p = self.prep.permuted
        want = ospmv.hybrid(self.prep.perm, (p.row_ptr, p.col_idx, p.values), 0, self.x_host)
        return bool(np.array_equal(np.asarray(y).view(np.uint64), want.view(np.uint64)))

    def e2e_bytes(self):
        p = self.prep.permuted
        s = self.hprep.split_row
        nz = int(p.row_ptr[-1] - p.row_ptr[s])
        per_nz = p.col_idx.dtype.itemsize + p.values.dtype.itemsize
        return (p.row_ptr.dtype.itemsize * (p.rows - s + 1) + per_nz * nz + self.x_host.nbytes), 8 * (p.rows - s)

    def cpu_sample(self, budget_s: float):
        from oracle import spmv as ospmv

        perm, permuted, _ = ospmv.preprocess(self.m.row_ptr, self.m.col_idx, self.m.values, 1.0, 3.0, None)
        split = ospmv.workload_split(permuted[0], 0.25)
        fn = lambda: ospmv.hybrid(perm, permuted, split, self.x_host)  # noqa: E731
        return fn, 2 * self.nnz, "full 1M-row matrix, one SpMV (prep excluded), formula share 0.25, 2 threads"

    def cpu_cores(self):
        return 2


class BilatBench:
    """BASELINE configs[3]: bilateral filter, 16384 x 16384 image (uint8
    intensities from gen_image, the reference's integer-intensity semantics),
    r=5, sigma_s=2.5, sigma_r=40 (BilatRunner defaults); fp64 arithmetic
    bit-identical to the reference, fp32 output image."""

    name = "bilat"
    unit = "Mpix/s"
    kernel = "bilateral_tma_kernel"

    def __init__(self, side: int = 16384, radius: int = 5, seed: int = 42):
        self.side, self.radius, self.seed = side, radius, seed

    def config(self):
        return {"workload": f"bilat: {self.side}x{self.side} image, r={self.radius}, sigma_s=2.5, sigma_r=40, fp64 taps, fp32 out",
                "side": self.side, "radius": self.radius, "seed": self.seed,
                "input": "gen_image(16384, 42) (splitmix64 low byte, device-generated)",
                "l2": "input 256 MiB + output 1 GiB > L2"}

    def setup(self, rank, world):
        import torch

        from paper_1303_2171_b200 import _lib
        from paper_1303_2171_b200.kernels_regular import build_bilateral_lut
        from paper_1303_2171_b200.rng import device_splitmix

        self.img = torch.empty((self.side, self.side), dtype=torch.uint8, device="cuda")
        device_splitmix(self.img, self.seed, _lib.HB_GEN_LOW8, k0=rank * self.side * self.side)
        self.lut = build_bilateral_lut(self.radius, max(self.radius / 2.0, 0.5), 40.0)
        self.out = torch.empty((self.side, self.side), dtype=torch.float32, device="cuda")
        self.world = world

    def step(self):
        from paper_1303_2171_b200.kernels_regular import gpu_bilateral_rows

        gpu_bilateral_rows(self.img, self.lut, 0, self.side, out=self.out, out_dtype=np.float32, asynchronous=True)
        return 1

    def units_per_step(self):
        return self.side * self.side

    def bytes_per_launch(self):
        return self.side * self.side * (1 + 4)

    def flops_per_launch(self):
        return self.side * self.side * (2 * self.radius + 1) ** 2 * 4

    def verify(self):
        from oracle import bilateral as obil

        sp, rg = obil.lut(self.radius, max(self.radius / 2.0, 0.5), 40.0)
        rows = [(0, 8), (8000, 8008), (self.side - 8, self.side)]
        host = self.img.cpu().numpy()
        ok = True
        for a, b in rows:
            want = obil.rows(host, sp, rg, self.radius, a, b).astype(np.float32)
            ok &= np.array_equal(self.out[a:b].cpu().numpy(), want)
        return bool(ok)

    def e2e_setup(self):
        import torch

        from paper_1303_2171_b200.kernels_regular import Image
        from paper_1303_2171_b200.platform import Platform
        from paper_1303_2171_b200.worksharing import WorkShare

        self.host = torch.empty((self.side, self.side), dtype=torch.uint8, pin_memory=True)
        self.host.copy_(self.img)
        self.image = Image(self.host.numpy())
        self.platform = host_platform()
        self.share = e2e_share(ARGS, self.e2e_workload(), self.platform)

    def e2e_workload(self):
        from paper_1303_2171_b200.kernels_regular import BilateralApplyWorkload

        return BilateralApplyWorkload(self.image, self.lut)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_regular import hybrid_bilateral

        return hybrid_bilateral(self.image, self.lut, self.platform, self.share)

    def _oracle_rows(self, host, a, b):
        from oracle import bilateral as obil

        sp, rg = obil.lut(self.radius, max(self.radius / 2.0, 0.5), 40.0)
        return obil.rows(host, sp, rg, self.radius, a, b)

    def e2e_verify(self, img):
        """Sampled rows of the f64 result image (both sides' strips) vs the oracle, bit-exact."""
        host = self.host.numpy()
        out = np.asarray(img.pixels)
        split = int(math.floor(self.share.fraction_a * self.side))
        rows = {(0, 4), (max(0, split - 2), min(self.side, split + 2)), (8000, 8004), (self.side - 4, self.side)}
        return bool(all(np.array_equal(out[a:b].view(np.uint64), self._oracle_rows(host, a, b).view(np.uint64))
                        for a, b in rows if b > a))

    def e2e_bytes(self):
        gpu_rows = self.side - int(math.floor(self.share.fraction_a * self.side))
        return gpu_rows * self.side, gpu_rows * self.side * 8

    def cpu_sample(self, budget_s: float):
        from oracle import bilateral as obil

        rows = 256
        host = self.img[: rows + self.radius].cpu().numpy()
        sp, rg = obil.lut(self.radius, max(self.radius / 2.0, 0.5), 40.0)
        fn = lambda: obil.hybrid(host[:rows], sp, rg, self.radius, 0.25)  # noqa: E731
        return fn, rows * self.side, f"{rows} x {self.side} strip of the same image, formula share 0.25, 2 threads"

    def cpu_cores(self):
        return 2


class ConvBench(BilatBench):
    """Convolution (not a BASELINE config): 16384 x 16384 uint8
    image, 15 x 15 Gaussian (the paper's figure kernel, FilterKernel.gaussian(7)),
    fp64 arithmetic bit-identical to the reference, fp32 output image."""

    name = "conv"
    kernel = "conv_rows_kernel"
    compute_bound = "fp64 issue (1 DMUL + 1 DADD per tap)"

    def __init__(self, side: int = 16384, radius: int = 7, seed: int = 42):
        super().__init__(side, radius, seed)

    def config(self):
        return {"workload": f"conv: {self.side}x{self.side} image, {2 * self.radius + 1}x{2 * self.radius + 1} Gaussian, fp64 taps, fp32 out",
                "side": self.side, "radius": self.radius, "seed": self.seed,
                "input": "gen_image(16384, 42) (splitmix64 low byte, device-generated)",
                "l2": "input 256 MiB + output 1 GiB > L2"}

    def setup(self, rank, world):
        super().setup(rank, world)
        from paper_1303_2171_b200.kernels_regular import FilterKernel

        self.fk = FilterKernel.gaussian(self.radius)

    def step(self):
        from paper_1303_2171_b200.kernels_regular import gpu_convolve_rows

        gpu_convolve_rows(self.img, self.fk, 0, self.side, out=self.out, out_dtype=np.float32, asynchronous=True)
        return 1

    def flops_per_launch(self):
        return self.side * self.side * (2 * self.radius + 1) ** 2 * 2

    def verify(self):
        from oracle import conv as oconv

        host = self.img.cpu().numpy()
        ok = True
        for a, b in [(0, 8), (8000, 8008), (self.side - 8, self.side)]:
            want = oconv.rows(host, self.fk.weights, a, b).astype(np.float32)
            ok &= np.array_equal(self.out[a:b].cpu().numpy(), want)
        return bool(ok)

    def e2e_workload(self):
        from paper_1303_2171_b200.kernels_regular import ConvolutionWorkload

        return ConvolutionWorkload(self.image, self.fk)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_regular import hybrid_convolve

        return hybrid_convolve(self.image, self.fk, self.platform, self.share)

    def _oracle_rows(self, host, a, b):
        from oracle import conv as oconv

        return oconv.rows(host, self.fk.weights, a, b)

    def cpu_sample(self, budget_s: float):
        from oracle import conv as oconv

        rows = 128
        host = self.img[: rows + self.radius].cpu().numpy()
        fn = lambda: oconv.hybrid(host[:rows], self.fk.weights, 0.25)  # noqa: E731
        return fn, rows * self.side, f"{rows} x {self.side} strip of the same image, formula share 0.25, 2 threads"


class SortBench:
    """BASELINE configs[2]: LSD radix sort of 2^28 uint32 keys + uint32
    payload (gen_sort_data keys, payload = global index), per GPU;
    multi-GPU runs add the sample-merge exchange (NCCL all-to-all)."""

    name = "sort"
    unit = "Mkeys/s"
    kernel = "onesweep_rfk_kernel"

    def __init__(self, n: int = 1 << 28, seed: int = 42):
        self.n, self.seed = n, seed

    def config(self):
        return {"workload": f"sort: LSD radix sort of 2^{self.n.bit_length() - 1} uint32 keys + uint32 payload per GPU",
                "n_per_gpu": self.n, "seed": self.seed,
                "input": "gen_sort_data(n, 42) (splitmix64 >> 32, device-generated), payload = global index",
                "l2": "2 GiB of keys+payload > L2; keys regenerated before every step (untimed)",
                "algorithmic_bytes": "68 B/key: 4 (digit histogram) + 4 passes x 16 (read+write key+payload)"}

    def setup(self, rank, world):
        import torch

        self.rank, self.world = rank, world
        self.keys = torch.empty(self.n, dtype=torch.int32, device="cuda")
        self.vals = torch.empty(self.n, dtype=torch.int32, device="cuda")
        self.prepare_step()

    def prepare_step(self):
        import torch

        from paper_1303_2171_b200 import _lib
        from paper_1303_2171_b200.rng import device_splitmix

        device_splitmix(self.keys, self.seed, _lib.HB_GEN_HI32, k0=self.rank * self.n)
        torch.arange(self.rank * self.n, (self.rank + 1) * self.n, dtype=torch.int32, out=self.vals)

    def step(self):
        from paper_1303_2171_b200 import _lib
        from paper_1303_2171_b200.gpu import current_stream_handle, vp

        _lib.call("hb_sort", vp(self.keys.data_ptr()), vp(self.keys.data_ptr()), _lib.DTYPE_CODES["u4"],
                  vp(self.vals.data_ptr()), vp(self.vals.data_ptr()), self.n, None, _lib.HB_DEVICE_PTRS,
                  current_stream_handle(self.keys))
        if self.world > 1:
            import torch

            from paper_1303_2171_b200.sharding import group_from_default
            from paper_1303_2171_b200.sort_exchange import exchange_sort

            # the keys are u32 (int32 storage): the exchange must order them unsigned
            self.out_k, self.out_v = exchange_sort(self.keys.view(torch.uint32), self.vals, group_from_default(),
                                                   local_sort=_presorted_then_gpu())
            return 1 + 4 + 1 + 1 + 4
        return 1 + 4  # digit histogram + 4 onesweep passes

    def units_per_step(self):
        return self.n

    def bytes_per_launch(self):
        return self.n * 68

    def verify(self):
        import torch

        from oracle import sort as osort

        if self.world > 1:
            k = self.out_k.view(torch.int32).cpu().numpy().view(np.uint32)
            return bool(np.all(np.diff(k.astype(np.int64)) >= 0))
        k = self.keys.cpu().numpy().view(np.uint32)
        v = self.vals.cpu().numpy()
        torch.cuda.synchronize()
        self.prepare_step()
        keys_in = self.keys.cpu().numpy().view(np.uint32)
        ok = np.array_equal(k, np.sort(keys_in))
        return bool(ok and osort.check_stable_payload(keys_in, k, v))

    def e2e_setup(self):
        import torch

        from paper_1303_2171_b200.platform import Platform
        from paper_1303_2171_b200.worksharing import WorkShare

        self.host = torch.empty(self.n, dtype=torch.int32, pin_memory=True)
        self.host.copy_(self.keys)
        self.host_np = self.host.numpy().view(np.uint32)
        self.platform = Platform.build(1.0, 3.0)
        self.share = WorkShare.manual(0.0)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_regular import sample_sort_hybrid

        return sample_sort_hybrid(self.host_np, self.platform, share=self.share)

    def e2e_verify(self, res):
        """Sorted, same multiset as the input (count, sum, xor of the keys) — O(n)."""
        k = np.asarray(res[0]).view(np.uint32)
        if self.world > 1:  # the sample-merge returns the group's keys: order only
            return bool(np.all(k[1:] >= k[:-1]))
        src = self.host_np
        ok = k.size == src.size and bool(np.all(k[1:] >= k[:-1]))
        ok = ok and int(k.sum(dtype=np.uint64)) == int(src.sum(dtype=np.uint64))
        return bool(ok and int(np.bitwise_xor.reduce(k)) == int(np.bitwise_xor.reduce(src)))

    def e2e_bytes(self):
        return 4 * self.n, 4 * self.n

    def cpu_sample(self, budget_s: float):
        from oracle import sort as osort

        m = 1 << 22
        host = self.keys[:m].cpu().numpy().view(np.uint32).astype(np.int64)
        fn = lambda: osort.sample_sort_hybrid(host, 0.25)  # noqa: E731
        return fn, m, "2^22 keys of the same stream through the reference's sample_sort_hybrid (formula share 0.25, 2 threads)"

    def cpu_cores(self):
        return 2


def _presorted_then_gpu():
    """exchange_sort's first local sort is already the timed hb_sort call;
    the second (of the received runs) is a GPU sort."""
    state = {"first": True}

    def fn(k, v):
        if state["first"]:
            state["first"] = False
            return k, v
        from paper_1303_2171_b200.sort_exchange import gpu_local_sort

        return gpu_local_sort(k, v)

    return fn


class LrBench:
    """BASELINE configs[4]: list ranking of a 2^28-node random linked list
    (gen_list(2^28, 42), generated on the device bit-identically), succ int32
    on the device, ranks int64."""

    name = "lr"
    unit = "Mnodes/s"
    kernel = "lr_walk_kernel"

    def __init__(self, n: int = 1 << 28, seed: int = 42):
        self.n, self.seed = n, seed

    def config(self):
        return {"workload": f"lr: list ranking of a 2^{self.n.bit_length() - 1}-node random list (sparse ruling set + Wyllie)",
                "n_per_gpu": self.n, "seed": self.seed,
                "input": "gen_list(n, 42): stable argsort of splitmix64 draws (device-generated, bit-identical)",
                "l2": "succ 1 GiB + rank 2 GiB > L2",
                "algorithmic_bytes": "12 B/node (4 succ + 8 rank); random 4-B reads move 32-B sectors"}

    def setup(self, rank, world):
        import torch

        from paper_1303_2171_b200.datasets import device_gen_list

        self.world = world
        self.succ, self.head = device_gen_list(self.n, self.seed + rank)
        self.rank = torch.empty(self.n, dtype=torch.int64, device="cuda")

    def step(self):
        from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

        gpu_list_rank(self.succ, self.head, out=self.rank)
        return 8  # check + 3 walks + top + 3 expands

    def units_per_step(self):
        return self.n

    def random_accesses_per_launch(self):
        # level-1 walk: one random succ read + one random (sublist, offset) write per node;
        # the recursion levels touch 1/64 as many nodes, the expansion is coalesced
        return self.n, self.n

    def bytes_per_launch(self):
        return 12 * self.n

    def verify(self):
        s = self.succ.cpu().numpy().astype(np.int64)
        r = self.rank.cpu().numpy()
        inner = s >= 0
        ok = r[self.head] == 0 and np.array_equal(r[s[inner]], r[inner] + 1)
        ok = ok and np.array_equal(np.bincount(r, minlength=self.n), np.ones(self.n, dtype=np.int64))
        return bool(ok)

    def e2e_setup(self):
        import torch

        from paper_1303_2171_b200.kernels_irregular import LinkedListArr
        from paper_1303_2171_b200.platform import Platform

        host = torch.empty(self.n, dtype=torch.int64, pin_memory=True)
        host.copy_(self.succ)
        self.host = host
        self.lst = LinkedListArr(host.numpy(), self.head)
        self.platform = Platform.build(1.0, 3.0)

    def e2e_step(self):
        from paper_1303_2171_b200.kernels_irregular import list_rank_hybrid

        return list_rank_hybrid(self.lst, self.platform, self.seed)

    def e2e_verify(self, rank):
        """Identical to the device-resident ranks (themselves checked in verify())."""
        return bool(np.array_equal(np.asarray(rank), self.rank.cpu().numpy()))

    def e2e_bytes(self):
        return 8 * self.n, 8 * self.n

    def cpu_sample(self, budget_s: float):
        from oracle import datasets as ods
        from oracle import listrank as olr

        m = 1 << 22
        succ, head = ods.linked_list(m, self.seed)
        fn = lambda: olr.list_rank_with_stats(succ, head, self.seed)  # noqa: E731
        return fn, m, "gen_list(2^22, 42) through the reference's list_rank_with_stats (validate + FIS + sublists), 1 thread"

    def cpu_cores(self):
        return 1


WORKLOADS = {"hist": HistBench, "spmv": SpmvBench, "bilat": BilatBench, "conv": ConvBench, "sort": SortBench, "lr": LrBench}


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


def run_reference(args, wl) -> dict:
    """--impl reference: the reference CPU algorithm on the host cores."""
    import torch

    rank, world, local = dist_env()
    if rank != 0:
        return {}
    if torch.cuda.is_available():
        torch.cuda.set_device(local % torch.cuda.device_count())
    wl.setup(0, 1)
    fn, units, sample = wl.cpu_sample(30.0)
    ts = time_cpu(fn, args.steps, warm=args.warmup)
    t = statistics.median(ts)
    val = units / t / (1e9 if wl.unit.startswith("G") else 1e6)
    return {
        "metric": METRIC,
        "impl": "reference",
        "value": val,
        "unit": wl.unit,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "config": wl.config(),
        "cpu_baseline": {"value": val, "unit": wl.unit, "cores": wl.cpu_cores(), "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": wl.unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def measure(args, wl, rank, world, with_cpu: bool) -> dict:
    import torch

    wl.setup(rank, world)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    with ClockSampler(torch.cuda.current_device()) as clocks:
        for _ in range(args.warmup):
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
            # inputs consumed in place: regenerate them (untimed) between timed steps
            pairs = []
            for _ in range(args.steps):
                prep()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                launches += wl.step()
                b.record(stream)
                pairs.append((a, b))
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in pairs) / args.steps
        t1 = time.perf_counter()
        clk = clocks.summary(t0, t1)
    ms = max_over_ranks(ms, world)
    ok = wl.verify()

    # end-to-end through the public API (host pinned buffers)
    wl.e2e_setup()
    for _ in range(1):
        wl.e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    e_steps = max(1, min(args.steps, args.e2e_steps))
    e0 = time.perf_counter()
    last = None
    for _ in range(e_steps):
        last = None  # drop the previous result first, as a caller would (its pinned block is reused)
        last = wl.e2e_step()
    torch.cuda.synchronize()
    e_s = (time.perf_counter() - e0) / e_steps
    barrier(world)
    e_s = max_over_ranks(e_s, world)

    scale = 1e9 if wl.unit.startswith("G") else 1e6
    value = wl.units_per_step() * world / (ms / 1e3) / scale
    peak, peak_src = hbm_peak()
    achieved = wl.bytes_per_launch() / (ms / 1e3) / 1e9
    h2d, d2h = wl.e2e_bytes()
    res = {
        "value": value,
        "unit": wl.unit,
        "ms_per_step": ms,
        "parity": ok,
        "gpu_launches": launches,
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic_of(wl.kernel),
            "peak_source": peak_src,
            "algorithmic_bytes_per_launch": wl.bytes_per_launch(),
            "kernel": wl.kernel,
        },
        "e2e": {
            "value": wl.units_per_step() * world / e_s / scale,
            "unit": wl.unit,
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "ms_per_step": e_s * 1e3,
            "steps": e_steps,
            "api": getattr(wl, "e2e_api", "public drop-in entry point on pinned host buffers"),
            "share": e2e_share_info(wl),
            "parity": wl.e2e_verify(last) if hasattr(wl, "e2e_verify") else None,
        },
        "clocks": clk,
        "config": wl.config(),
    }
    if hasattr(wl, "random_accesses_per_launch"):
        # random-access-bound kernel: DRAM row activations, not bytes, are the bound;
        # a random 8-B write costs a sector read-fill + a write (micro: 24.8 G/s)
        reads, writes = wl.random_accesses_per_launch()
        bound_ms = (reads / RANDOM_READ_PEAK + writes / RANDOM_WRITE_PEAK) / 1e9 * 1e3
        res["roofline"]["random_access"] = {
            "bound": "DRAM random accesses: t >= reads/R + writes/W",
            "reads_per_launch": reads,
            "writes_per_launch": writes,
            "peak_read_g_per_s": RANDOM_READ_PEAK,
            "peak_write_g_per_s": RANDOM_WRITE_PEAK,
            "bound_ms": bound_ms,
            "frac": bound_ms / ms,
            "peak_source": "measured: scripts/micro/gather.cu — 2^26 random 4-B loads from 1 GiB (51.5 G/s; "
                           "dependent chase 50 G/s; L2 fetch granularity 32/64 B: no change), 2^26 random 8-B "
                           "stores (24.8 G/s, ncu: 32 B read-fill + 32 B write per store)",
        }
    if hasattr(wl, "flops_per_launch"):
        # compute-bound kernel: fp64 issue is the bound, HBM fraction is low by design
        ach = wl.flops_per_launch() / (ms / 1e3) / 1e9
        res["roofline"]["compute"] = {
            "bound": getattr(wl, "compute_bound", "fp64 issue (2 DMUL + 2 DADD per tap)"),
            "achieved_gflops": ach,
            "peak_gflops": FP64_PEAK_GFLOPS,
            "frac": ach / FP64_PEAK_GFLOPS,
            "peak_source": "measured: scripts/micro/fp64peak.cu, DADD/DMUL 18.37 T instr/s on B200 (1 flop each, no FMA)",
            "flops_per_launch": wl.flops_per_launch(),
        }
    if with_cpu and rank == 0:
        fn, units, sample = wl.cpu_sample(20.0)
        ts = time_cpu(fn, 1, warm=0)
        cv = units / min(ts) / scale
        res["cpu_baseline"] = {"value": cv, "unit": wl.unit, "cores": wl.cpu_cores(), "kind": "port", "sample": sample}
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="all", choices=sorted(WORKLOADS) + ["all"])
    ap.add_argument("--e2e-steps", type=int, default=10, help="steps of the end-to-end (host buffer) leg")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--e2e-share", default="auto", choices=["auto", "calibrated", "gpu"],
                    help="e2e leg split: measured host+GPU calibration, all on the GPU, or auto "
                         "(calibrated at N=1, GPU-only when ranks share the host)")
    args = ap.parse_args()
    global ARGS
    ARGS = args
    args.warmup = max(args.warmup, 3)

    rank, world, local = dist_env()
    headline = "hist" if args.workload == "all" else args.workload

    if args.impl == "reference":
        out = run_reference(args, WORKLOADS[headline]())
        if rank == 0:
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
        # each workload starts from the memory state of a standalone run: the
        # previous one's device blocks and cached pinned host blocks (GiBs of
        # e2e inputs/results) are released first
        import gc

        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        if hasattr(torch._C, "_host_emptyCache"):
            torch._C._host_emptyCache()

    head = measure(args, WORKLOADS[headline](), rank, world, with_cpu=(world == 1 and not args.no_cpu))
    others = {}
    if args.workload == "all":
        for name, cls in WORKLOADS.items():
            if name != headline:
                fresh_memory()
                others[name] = measure(args, cls(), rank, world, with_cpu=(world == 1 and not args.no_cpu))
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": head["value"],
            "unit": head["unit"],
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": head["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic (splitmix64 streams of the reference generators, seed 42)",
            "config": dict(head["config"], parallelism=f"shard{world}"),
            "roofline": head["roofline"],
            "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
            "parity": head["parity"],
        }
        if "cpu_baseline" in head:
            line["cpu_baseline"] = head["cpu_baseline"]
        if others:
            line["workloads"] = others
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
