"""On-disk formats and typed generators: files written
here are byte-identical to the reference's (tests/golden/formats/, written
by hybridbench), and hand-written inputs parse to what the reference parsed.
CPU only."""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1303_2171_b200 import datasets as d
from paper_1303_2171_b200.errors import ConfigError, DataIOError
from paper_1303_2171_b200.kernels_irregular import CsrMatrix, LinkedListArr, load_matrix_market, save_matrix_market
from paper_1303_2171_b200.kernels_regular import Image, read_pgm, write_pgm

F = GOLDEN / "formats"


def test_writers_byte_identical_to_reference(tmp_path):
    d.write_dataset("spmv", d.gen_csr(60, 60, 5, 0.05), tmp_path / "a.mtx")
    assert (tmp_path / "a.mtx").read_bytes() == (F / "ref_spmv.mtx").read_bytes()
    d.write_dataset("bilat", d.gen_image(21, 6), tmp_path / "a.pgm")
    assert (tmp_path / "a.pgm").read_bytes() == (F / "ref_img.pgm").read_bytes()
    write_pgm(d.gen_image(9, 2), tmp_path / "b.pgm", binary=False)
    assert (tmp_path / "b.pgm").read_bytes() == (F / "ref_img_p2.pgm").read_bytes()
    d.write_dataset("sort", d.gen_sort_data(777, 8), tmp_path / "k.u32")
    assert (tmp_path / "k.u32").read_bytes() == (F / "ref_sort.u32").read_bytes()


def test_readers_match_reference():
    want = np.load(F / "parsed.npz")
    m = load_matrix_market(F / "in_sym.mtx")
    assert np.array_equal(m.row_ptr, want["sym_ptr"]) and np.array_equal(m.col_idx, want["sym_col"])
    assert np.array_equal(m.values, want["sym_val"])
    assert np.array_equal(read_pgm(F / "in_comment.pgm").pixels, want["comment_pix"])
    m = load_matrix_market(F / "ref_spmv.mtx")
    g = d.gen_csr(60, 60, 5, 0.05)
    assert np.array_equal(m.values, g.values) and np.array_equal(m.col_idx, g.col_idx)
    assert np.array_equal(read_pgm(F / "ref_img.pgm").pixels, d.gen_image(21, 6).pixels)
    assert np.array_equal(d.read_raw_u32(F / "ref_sort.u32"), d.gen_sort_data(777, 8))


def test_round_trips(tmp_path):
    m = d.gen_csr(500, 400, 9, 0.01)
    save_matrix_market(m, tmp_path / "m.mtx")
    back = load_matrix_market(tmp_path / "m.mtx")
    assert np.array_equal(back.row_ptr, m.row_ptr) and np.array_equal(back.values, m.values)
    img = Image(np.linspace(-20, 300, 64).reshape(8, 8))  # float pixels: rounded + clamped
    write_pgm(img, tmp_path / "f.pgm")
    assert np.array_equal(read_pgm(tmp_path / "f.pgm").pixels, np.clip(np.rint(img.pixels), 0, 255).astype(np.uint8))


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n",
])
def test_matrix_market_errors(tmp_path, text):
    (tmp_path / "bad.mtx").write_text(text)
    with pytest.raises(DataIOError):
        load_matrix_market(tmp_path / "bad.mtx")


def test_matrix_market_row_out_of_range_like_reference(tmp_path):
    # the reference's from_coo fails inside numpy (ValueError, not wrapped)
    (tmp_path / "bad.mtx").write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n")
    with pytest.raises(ValueError):
        load_matrix_market(tmp_path / "bad.mtx")


def test_pgm_and_raw_errors(tmp_path):
    for raw in (b"P6\n1 1\n255\n\x00", b"P5\n2 2\n300\n\x00\x00\x00\x00", b"P2\n2 2\n255\n1 2 3\n"):
        (tmp_path / "bad.pgm").write_bytes(raw)
        with pytest.raises(DataIOError):
            read_pgm(tmp_path / "bad.pgm")
    with pytest.raises(DataIOError):
        read_pgm(tmp_path / "missing.pgm")
    (tmp_path / "empty.u32").write_bytes(b"")
    with pytest.raises(DataIOError):
        d.read_raw_u32(tmp_path / "empty.u32")


def test_generate_uar_types_and_errors():
    assert isinstance(d.generate_uar("spmv", 50, 1, density=0.1), CsrMatrix)
    assert isinstance(d.generate_uar("lr", 50, 1), LinkedListArr)
    assert isinstance(d.generate_uar("conv", 16, 1), Image)
    assert d.generate_uar("hist", 100, 1, bins=16).max() < 16
    with pytest.raises(ConfigError):
        d.generate_uar("sort", 0, 1)
    with pytest.raises(ConfigError):
        d.generate_uar("cc", 10, 1)
    with pytest.raises(ConfigError):
        d.write_dataset("lr", d.gen_list(5, 1), "x")
