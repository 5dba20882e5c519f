"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
implementation (hybridbench, imported from /root/reference/pkg/src in the dev
container).  The GPU box has no /root/reference; the tests read only the
committed .npz files.  Re-run with:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main(only: str | None = None) -> None:
    sys.path.insert(0, str(REF))
    if only == "conv":
        conv()
        return
    if only == "formats":
        formats()
        return
    from hybridbench import datasets, rng
    from hybridbench.kernels_irregular import (
        CsrMatrix,
        LinkedListArr,
        list_rank_with_stats,
        spmv_hybrid,
        spmv_preprocess,
    )
    from hybridbench.kernels_regular import (
        Image,
        bilateral_rows,
        build_bilateral_lut,
        hybrid_bilateral,
        hybrid_histogram,
        sample_sort_hybrid,
    )
    from hybridbench.platform import Platform
    from hybridbench.worksharing import WorkShare

    p13 = Platform.build(1.0, 3.0)
    shares = [i / 10 for i in range(11)]

    # ------------------------------------------------------------- rng
    g = {}
    for seed in (0, 42, 12345, 0xDEADBEEF):
        g[f"splitmix_{seed}"] = rng.splitmix64_array(seed, 64)
    g["mix_seed"] = np.array([rng.mix_seed(s, t) for s in (0, 1, 42) for t in (0, 1, 2, 3, 0x5EED, 0xDEC0)], dtype=np.uint64)
    g["uniform_floats_7"] = rng.uniform_floats(7, 32)
    g["uniform_ints_9"] = rng.uniform_ints(9, 32, 1000)
    np.savez_compressed(OUT / "rng.npz", **g)

    # ------------------------------------------------------------- hist
    h = {}
    for i, (n, seed, bins) in enumerate([(20_000, 11, 256), (3000, 3, 32), (4096, 5, 64), (1_000_000, 42, 256)]):
        data = datasets.gen_hist_data(n, seed, bins)
        h[f"data_{i}"] = data.astype(np.uint8) if bins <= 256 else data
        h[f"meta_{i}"] = np.array([n, seed, bins])
        h[f"bins_{i}"] = np.stack([hybrid_histogram(data, bins, p13, WorkShare.manual(s)).bins for s in shares])
    np.savez_compressed(OUT / "hist.npz", **h)

    # ------------------------------------------------------------- sort
    s = {}
    cases = [
        ("uar50k", datasets.gen_sort_data(50_000, 1)),
        ("dups", datasets.gen_sort_data(30_000, 42) % 5000),
        ("rev", np.arange(3000)[::-1].copy()),
        ("tiny", datasets.gen_sort_data(1500, 2)),
        ("const", np.full(5000, 9, dtype=np.int64)),
    ]
    for name, data in cases:
        s[f"{name}_data"] = data
        rows = []
        for sh in (0.0, 0.25, 0.5, 1.0):
            out, wa, wb = sample_sort_hybrid(data, p13, share=WorkShare.manual(sh))
            assert np.array_equal(out, np.sort(data))
            rows.append([sh, wa, wb])
        _, wa, wb = sample_sort_hybrid(data, p13)  # formula share 0.25
        rows.append([-1.0, wa, wb])
        s[f"{name}_work"] = np.array(rows)
    np.savez_compressed(OUT / "sort.npz", **s)

    # ------------------------------------------------------------- spmv
    m = {}
    for i, (rows_, density, seed) in enumerate([(50, 0.1, 3), (30, 0.15, 5), (2000, 0.004, 42), (36, 0.12, 80)]):
        mat = datasets.gen_csr(rows_, rows_, seed, density)
        x = 2.0 * rng.uniform_floats(rng.mix_seed(seed, 0xDEC0), rows_) - 1.0
        m[f"ptr_{i}"], m[f"col_{i}"], m[f"val_{i}"], m[f"x_{i}"] = mat.row_ptr, mat.col_idx, mat.values, x
        prep = spmv_preprocess(mat, p13)
        m[f"perm_{i}"] = prep.perm
        m[f"split_{i}"] = np.array([prep.split_row] + [spmv_preprocess(mat, p13, WorkShare.manual(sh)).split_row for sh in shares])
        m[f"y_{i}"] = spmv_hybrid(prep, x)
    ident = CsrMatrix.identity(100)
    m["identity100_split"] = np.array([spmv_preprocess(ident, p13).split_row])
    np.savez_compressed(OUT / "spmv.npz", **m)

    # ------------------------------------------------------------- bilateral
    b = {}
    for i, (side, seed, radius, ss, sr) in enumerate([(24, 8, 2, 2.0, 30.0), (64, 4, 3, 2.5, 35.0), (40, 42, 5, 2.5, 40.0), (33, 7, 7, 3.5, 40.0)]):
        img = datasets.gen_image(side, seed)
        lut = build_bilateral_lut(radius, ss, sr)
        b[f"img_{i}"] = img.pixels
        b[f"meta_{i}"] = np.array([side, seed, radius, ss, sr])
        b[f"spatial_{i}"], b[f"range_{i}"] = lut.spatial_weights, lut.range_weights
        b[f"out_{i}"] = hybrid_bilateral(img, lut, p13).pixels
        b[f"strip_{i}"] = bilateral_rows(img.pixels, lut, side // 3, side // 3 + 5)
    rect = Image(datasets.gen_image(48, 3).pixels[:20, :].copy())
    lut = build_bilateral_lut(3, 2.0, 25.0)
    b["rect_img"], b["rect_out"] = rect.pixels, hybrid_bilateral(rect, lut, p13).pixels
    np.savez_compressed(OUT / "bilateral.npz", **b)

    # ------------------------------------------------------------- list ranking
    lr = {}
    for i, (n, seed, rseed) in enumerate([(10_000, 42, 7), (500, 0, 0), (1000, 3, 3), (4097, 11, 5), (2, 1, 1), (1, 1, 1)]):
        if n == 1:
            lst = LinkedListArr(np.array([-1]), 0)
        else:
            lst = datasets.gen_list(n, seed)
        ranks, st = list_rank_with_stats(lst, p13, rseed)
        lr[f"succ_{i}"], lr[f"head_{i}"], lr[f"seed_{i}"] = lst.succ, np.array([lst.head]), np.array([rseed])
        lr[f"rank_{i}"] = ranks
        lr[f"stats_{i}"] = np.array([st.fis_rounds, st.reduced_size, st.removed_total, st.sublist_count])
        lr[f"sizes_{i}"] = np.array(st.round_sizes, dtype=np.int64)
    np.savez_compressed(OUT / "listrank.npz", **lr)
    conv()
    formats()
    print("golden fixtures written to", OUT)


def conv() -> None:
    """Convolution fixtures (kernels_regular.py:327-414): hybrid_convolve at
    several shares, uint8 and float64 images, kernels with zero taps."""
    from hybridbench import datasets, rng
    from hybridbench.kernels_regular import ConvolutionWorkload, FilterKernel, Image, convolve_rows, hybrid_convolve
    from hybridbench.platform import Platform
    from hybridbench.worksharing import WorkShare

    p13 = Platform.build(1.0, 3.0)
    c = {}
    rand5 = rng.uniform_floats(123, 25).reshape(5, 5) * 2 - 1
    rand5[1, 3] = 0.0
    rand5[4, 0] = 0.0
    sparse7 = np.zeros((15, 15))
    sparse7[::3, ::2] = rng.uniform_floats(77, 40).reshape(5, 8) - 0.5
    cases = [(24, 9, rand5), (64, 4, FilterKernel.gaussian(3).weights), (40, 42, FilterKernel.delta(2).weights),
             (37, 7, sparse7), (50, 1, FilterKernel.gaussian(7).weights), (30, 5, FilterKernel.gaussian(10).weights)]
    for i, (side, seed, w) in enumerate(cases):
        img = datasets.gen_image(side, seed)
        k = FilterKernel(np.asarray(w, dtype=np.float64))
        c[f"img_{i}"], c[f"w_{i}"] = img.pixels, k.weights
        c[f"out_{i}"] = np.stack([hybrid_convolve(img, k, p13, WorkShare.manual(s)).pixels for s in (0.0, 0.3, 1.0)])
        c[f"strip_{i}"] = convolve_rows(img.pixels, k, side // 3, side // 3 + 5)
    # float64 image (linearity test input of test_kernels_regular.py:159-168)
    a = datasets.gen_image(16, 1).pixels.astype(np.float64)
    b = datasets.gen_image(16, 2).pixels.astype(np.float64)
    f = 0.7 * a - 1.3 * b
    k = FilterKernel.gaussian(2)
    c["f64_img"], c["f64_w"], c["f64_out"] = f, k.weights, hybrid_convolve(Image(f), k, p13).pixels
    # rectangular image, criterion-7 partition
    rect = datasets.gen_image(48, 3).pixels[:20, :].copy()
    c["rect_img"], c["rect_out"] = rect, hybrid_convolve(Image(rect), FilterKernel.gaussian(2), p13).pixels
    wl = ConvolutionWorkload(Image(np.zeros((3600, 3600), dtype=np.uint8)), FilterKernel.delta(7))
    c["part_18"] = np.array(wl.partition(0.18))
    np.savez_compressed(OUT / "conv.npz", **c)


def formats() -> None:
    """On-disk formats (datasets.py:133-163, kernels_regular.py:48-110,
    kernels_irregular.py:101-146): files written by the reference and what
    the reference reads back from hand-written inputs (comments, symmetric,
    duplicates)."""
    from hybridbench import datasets
    from hybridbench.kernels_irregular import load_matrix_market
    from hybridbench.kernels_regular import read_pgm, write_pgm

    d = OUT / "formats"
    d.mkdir(exist_ok=True)
    datasets.write_dataset("spmv", datasets.gen_csr(60, 60, 5, 0.05), d / "ref_spmv.mtx")
    datasets.write_dataset("bilat", datasets.gen_image(21, 6), d / "ref_img.pgm")
    write_pgm(datasets.gen_image(9, 2), d / "ref_img_p2.pgm", binary=False)
    datasets.write_dataset("sort", datasets.gen_sort_data(777, 8), d / "ref_sort.u32")
    (d / "in_sym.mtx").write_text(
        "%%MatrixMarket matrix coordinate real symmetric\n% a comment\n%another\n4 4 6\n"
        "1 1 2.5\n2 1 -1.0\n3 2 0.125\n4 4 1e-3\n3 1 7\n2 1 0.5\n"
    )
    (d / "in_comment.pgm").write_bytes(b"P2\n# made by hand\n3 2 # width height\n200\n0 1 2\n200 7 9\n")
    m = load_matrix_market(d / "in_sym.mtx")
    img = read_pgm(d / "in_comment.pgm")
    np.savez_compressed(d / "parsed.npz", sym_ptr=m.row_ptr, sym_col=m.col_idx, sym_val=m.values, comment_pix=img.pixels)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
