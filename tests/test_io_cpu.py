"""Matrix files (include/oocnmf/io.hpp, §8(f) rank 3) — host side, no GPU.

PDN1 and Matrix Market written by the compiled reference must read back identically through
the library's C++ host core and vice versa; the f32 dtype (the B200 extension in the byte the
reference reserves) round-trips at f32 precision and is refused by the reference as an unknown
dtype."""
import numpy as np
import pytest

import oracle
import paper_2202_09518_b200 as nmf

needs_ref = pytest.mark.skipif(not oracle.ref.available, reason="needs oracle/_ref")


def _csr(seed, m=40, n=30, density=0.2):
    d = np.random.default_rng(seed).random((m, n))
    d[d > density] = 0.0
    return nmf.CsrMatrix.from_dense(d)


@needs_ref
def test_pdn1_reference_written_files_read_back(tmp_path):
    a = np.random.default_rng(1).random((17, 9))
    oracle.ref.write_pdn1(tmp_path / "d.pdn1", a)
    assert np.array_equal(nmf.read_pdn1(tmp_path / "d.pdn1"), a)
    c = _csr(2)
    oracle.ref.write_pdn1(tmp_path / "c.pdn1", (c.row_ptr, c.col_idx, c.values, c.shape))
    got = nmf.read_pdn1(tmp_path / "c.pdn1")
    assert np.array_equal(got.row_ptr, c.row_ptr) and np.array_equal(got.col_idx, c.col_idx)
    assert np.array_equal(got.values, c.values)
    # our files are byte-identical to the reference's for f64
    nmf.write_pdn1(tmp_path / "d2.pdn1", a)
    nmf.write_pdn1(tmp_path / "c2.pdn1", c)
    assert (tmp_path / "d.pdn1").read_bytes() == (tmp_path / "d2.pdn1").read_bytes()
    assert (tmp_path / "c.pdn1").read_bytes() == (tmp_path / "c2.pdn1").read_bytes()


@needs_ref
def test_mtx_round_trips_with_the_reference(tmp_path):
    a = np.random.default_rng(3).random((6, 4))
    oracle.ref.write_mtx(tmp_path / "a.mtx", a)
    assert np.array_equal(nmf.read_matrix(tmp_path / "a.mtx"), a)
    nmf.write_mtx(tmp_path / "b.mtx", a)
    assert np.array_equal(oracle.ref.read_matrix(tmp_path / "b.mtx"), a)
    assert (tmp_path / "a.mtx").read_text() == (tmp_path / "b.mtx").read_text()
    c = _csr(4)
    nmf.write_mtx(tmp_path / "c.mtx", c)
    rp, ci, v, shape = oracle.ref.read_matrix(tmp_path / "c.mtx")
    assert shape == c.shape and np.array_equal(rp, c.row_ptr) and np.array_equal(ci, c.col_idx)
    assert np.array_equal(v, c.values)


@needs_ref
def test_mtx_unsorted_and_repeated_coordinates_like_the_reference(tmp_path):
    p = tmp_path / "u.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n% comment\n3 4 5\n"
                 "3 2 1.5\n1 4 2.0\n1 1 0.25\n3 2 7.0\n2 3 1e-3\n")
    ours = nmf.read_mtx(p)
    rp, ci, v, shape = oracle.ref.read_matrix(p)
    assert np.array_equal(ours.row_ptr, rp) and np.array_equal(ours.col_idx, ci) and np.array_equal(ours.values, v)
    assert ours.to_dense()[2, 1] == 7.0  # the later duplicate wins


def test_pdn1_f32_extension(tmp_path):
    a = np.random.default_rng(5).random((20, 12))
    nmf.write_pdn1(tmp_path / "a32.pdn1", a, dtype="f32")
    f = nmf.Pdn1File(tmp_path / "a32.pdn1")
    assert (f.dtype, f.rows, f.cols) == (1, 20, 12)
    assert (tmp_path / "a32.pdn1").stat().st_size == 26 + 20 * 12 * 4
    np.testing.assert_array_equal(f.read_dense_window(3, 9, 2, 7, np.float32), a.astype(np.float32)[3:9, 2:7])
    np.testing.assert_array_equal(nmf.read_pdn1(tmp_path / "a32.pdn1"), a.astype(np.float32).astype(np.float64))
    c = _csr(6)
    nmf.write_pdn1(tmp_path / "c32.pdn1", c, dtype="f32")
    r = nmf.Pdn1File(tmp_path / "c32.pdn1").read_csr_rows(5, 25)
    w = c.row_window(5, 25)
    assert np.array_equal(r.row_ptr, w.row_ptr) and np.array_equal(r.col_idx, w.col_idx)
    np.testing.assert_array_equal(r.values, w.values.astype(np.float32).astype(np.float64))
    if oracle.ref.available:
        with pytest.raises(OSError, match="dtype"):
            oracle.ref.read_matrix(tmp_path / "a32.pdn1")


def test_io_errors(tmp_path):
    with pytest.raises(nmf.IoError, match="cannot open"):
        nmf.read_pdn1(tmp_path / "missing.pdn1")
    (tmp_path / "bad.pdn1").write_bytes(b"NOTPDN1" + bytes(30))
    with pytest.raises(nmf.IoError, match="magic"):
        nmf.read_pdn1(tmp_path / "bad.pdn1")
    nmf.write_pdn1(tmp_path / "d.pdn1", np.ones((4, 4)))
    with pytest.raises(nmf.ShapeError, match="out of bounds"):
        nmf.Pdn1File(tmp_path / "d.pdn1").read_dense_window(0, 5, 0, 4)
    with pytest.raises(nmf.IoError, match="CSR row read on dense"):
        nmf.Pdn1File(tmp_path / "d.pdn1").read_csr_rows(0, 2)
    (tmp_path / "t.pdn1").write_bytes((tmp_path / "d.pdn1").read_bytes()[:-9])
    with pytest.raises(nmf.IoError, match="truncated"):
        nmf.read_pdn1(tmp_path / "t.pdn1")
    (tmp_path / "x.mtx").write_text("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n")
    with pytest.raises(nmf.IoError, match="unsupported"):
        nmf.read_mtx(tmp_path / "x.mtx")
