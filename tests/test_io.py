"""MatrixMarket / .tlcsr ingestion (src/io.py behaviour).

Same inputs and expectations as the reference's ingestion contract
(T/test_io.py): symmetric mirroring, banner / size / entry rejections that
name path:line, zero off-diagonal dropping, exact write/read round trips,
the binary cache's magic / version / truncation checks, format sniffing.
Plus a larger file through the native scanner and an end-to-end solve of a
loaded matrix.  CPU only (the scanner is host code in libhbmc_b200.so).
"""

import numpy as np
import pytest

import paper_1908_00741_b200 as P
import workloads as problems

BANNER_SYM = "%%MatrixMarket matrix coordinate real symmetric"
BANNER_GEN = "%%MatrixMarket matrix coordinate real general"


def write(tmp_path, text, name="m.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def expect_error(path, *frags):
    with pytest.raises(P.IngestionError) as e:
        P.read_matrix_market(path)
    for f in frags:
        assert f in str(e.value), str(e.value)
    return e.value


def test_symmetric_file_is_mirrored(tmp_path):
    text = f"{BANNER_SYM}\n3 3 4\n1 1 2.0\n2 2 2.0\n3 3 2.0\n3 1 -1.0\n"
    a = P.coo_to_csr(P.read_matrix_market(write(tmp_path, text)))
    d = a.to_dense()
    assert d[2, 0] == d[0, 2] == -1.0 and a.nnz == 5
    assert np.array_equal(d, d.T)


def test_general_file_not_mirrored(tmp_path):
    text = f"{BANNER_GEN}\n2 2 3\n1 1 4.0\n1 2 -1.0\n2 2 4.0\n"
    d = P.coo_to_csr(P.read_matrix_market(write(tmp_path, text))).to_dense()
    assert d[0, 1] == -1.0 and d[1, 0] == 0.0


def test_line_numbers_count_comments_and_blanks(tmp_path):
    text = f"{BANNER_GEN}\n% c\n\n2 2 2\n1 1 1.0\n% c2\n2 99 1.0\n"
    expect_error(write(tmp_path, text), ":7:", "outside")


@pytest.mark.parametrize("banner,frag", [
    ("%%MatrixMarket matrix array real general", "coordinate"),
    ("%%MatrixMarket matrix coordinate complex general", "non-real"),
    ("%%MatrixMarket matrix coordinate pattern symmetric", "non-real"),
    ("%%MatrixMarket matrix coordinate real hermitian", "symmetry"),
    ("%%MatrixMarket vector coordinate real general", "object"),
    ("%%NotMatrixMarket", "banner"),
])
def test_banner_rejected_on_line_1(tmp_path, banner, frag):
    expect_error(write(tmp_path, banner + "\n1 1 0\n"), ":1:", frag)


def test_banner_is_case_insensitive(tmp_path):
    text = "%%MATRIXMARKET Matrix COORDINATE real Symmetric\n2 2 2\n1 1 1.0\n2 2 1.0\n"
    assert P.read_matrix_market(write(tmp_path, text)).n == 2


def test_size_line_errors(tmp_path):
    expect_error(write(tmp_path, f"{BANNER_GEN}\n2 3 1\n1 1 1.0\n"), ":2:", "square")
    expect_error(write(tmp_path, f"{BANNER_GEN}\n2 2\n1 1 1.0\n"), ":2:", "rows cols nnz")
    expect_error(write(tmp_path, f"{BANNER_GEN}\n2 2 x\n"), ":2:", "three integers")
    expect_error(write(tmp_path, f"{BANNER_GEN}\n% only a comment\n"), "missing size line")


def test_entry_count_mismatch(tmp_path):
    expect_error(write(tmp_path, f"{BANNER_GEN}\n2 2 3\n1 1 1.0\n"),
                 "expected 3 entries, found 1", ":2:")
    expect_error(write(tmp_path, f"{BANNER_GEN}\n2 2 1\n1 1 1.0\n2 2 1.0\n"),
                 "expected 1 entries, found 2", ":4:")


@pytest.mark.parametrize("bad,frag", [("2 2\n", "row col value"), ("2 x 1.0\n", "bad index"),
                                      ("2 2 abc\n", "non-real value 'abc'"),
                                      ("2 1.5 1.0\n", "bad index"),
                                      ("2 2 1.0 7\n", "row col value")])
def test_malformed_entry_names_its_line(tmp_path, bad, frag):
    expect_error(write(tmp_path, f"{BANNER_GEN}\n2 2 2\n1 1 1.0\n" + bad), ":4:", frag)


def test_integral_real_indices(tmp_path):
    # accepted when every entry line is numeric (the reference's fast path) ...
    ok = f"{BANNER_GEN}\n2 2 2\n1.0 1 1.0\n2 2.0 1.0\n"
    a = P.coo_to_csr(P.read_matrix_market(write(tmp_path, ok)))
    assert a.to_dense().tolist() == [[1.0, 0.0], [0.0, 1.0]]
    # ... and named as a bad index once another line fails (its slow path)
    bad = f"{BANNER_GEN}\n2 2 2\n1.0 1 1.0\n2 2 zz\n"
    expect_error(write(tmp_path, bad), ":3:", "bad index")


def test_upper_triangle_rejected_in_symmetric(tmp_path):
    text = f"{BANNER_SYM}\n2 2 3\n1 1 1.0\n1 2 -1.0\n2 2 1.0\n"
    expect_error(write(tmp_path, text), ":4:", "above the diagonal")


def test_duplicate_reports_second_occurrence(tmp_path):
    text = f"{BANNER_GEN}\n2 2 3\n1 1 1.0\n2 2 1.0\n1 1 5.0\n"
    expect_error(write(tmp_path, text), ":5:", "duplicate entry (1 1)")


def test_zero_offdiagonals_dropped_diagonal_kept(tmp_path):
    text = f"{BANNER_SYM}\n3 3 5\n1 1 0.0\n2 2 2.0\n3 3 2.0\n2 1 0.0\n3 1 -1.0\n"
    coo = P.read_matrix_market(write(tmp_path, text))
    assert coo.dropped_zeros == 1
    a = P.coo_to_csr(coo)
    assert a.diagonal()[0] == 0.0 and a.to_dense()[1, 0] == 0.0


def test_crlf_and_leading_whitespace(tmp_path):
    text = f"{BANNER_GEN}\r\n  2 2 2\r\n\t1 1 1.5\r\n 2 2 -2.5e-1 \r\n"
    d = P.coo_to_csr(P.read_matrix_market(write(tmp_path, text))).to_dense()
    assert d.tolist() == [[1.5, 0.0], [0.0, -0.25]]


def test_round_trip_exact(tmp_path):
    a = P.gen_random_spd(40, density=0.08, seed=9)
    p = str(tmp_path / "rt.mtx")
    P.write_matrix_market(p, a, comment="round trip\nsecond line")
    back = P.coo_to_csr(P.read_matrix_market(p))
    for f in ("row_ptr", "col_idx", "vals"):
        assert np.array_equal(getattr(back, f), getattr(a, f))


def test_writer_emits_lower_triangle(tmp_path):
    a, _ = P.gen_laplacian_5pt(4, 3)
    p = str(tmp_path / "lo.mtx")
    P.write_matrix_market(p, a)
    body = [ln for ln in open(p).read().splitlines() if ln and not ln.startswith("%")]
    assert int(body[0].split()[2]) == len(body) - 1
    assert all(int(ln.split()[0]) >= int(ln.split()[1]) for ln in body[1:])


def test_cache_round_trip_and_rejections(tmp_path):
    a = P.gen_random_spd(50, density=0.05, seed=4)
    p = tmp_path / "a.tlcsr"
    P.write_csr_cache(str(p), a)
    back = P.read_csr_cache(str(p))
    for f in ("row_ptr", "col_idx", "vals"):
        assert np.array_equal(getattr(back, f), getattr(a, f))
    assert all(back.col_idx[back.diag_ptr[i]] == i for i in range(a.n))
    raw = p.read_bytes()
    p.write_bytes(raw[:-8])
    with pytest.raises(P.IngestionError, match="truncated"):
        P.read_csr_cache(str(p))
    v = bytearray(raw)
    v[6:10] = (7).to_bytes(4, "little")
    p.write_bytes(bytes(v))
    with pytest.raises(P.IngestionError, match="version"):
        P.read_csr_cache(str(p))
    p.write_bytes(b"NOTCSR" + raw[6:])
    with pytest.raises(P.IngestionError, match="magic"):
        P.read_csr_cache(str(p))


def test_load_matrix_sniffs_and_writes_sibling_cache(tmp_path):
    a, _ = P.gen_laplacian_5pt(5, 4)
    mtx = str(tmp_path / "g.mtx")
    P.write_matrix_market(mtx, a)
    m1 = P.load_matrix(mtx, write_cache=True)
    assert np.array_equal(m1.vals, a.vals)
    m2 = P.load_matrix(mtx + ".tlcsr")
    assert np.array_equal(m2.vals, a.vals) and np.array_equal(m2.col_idx, a.col_idx)
    with pytest.raises((P.IngestionError, OSError)):
        P.load_matrix(str(tmp_path / "absent.mtx"))


def test_large_file_through_native_scanner(tmp_path):
    """A BASELINE-family matrix (7-point 24^3, 13,824 rows) survives
    write -> native read bit for bit, and its HBMC ordering matches the one
    of the in-memory matrix."""
    a = problems.varcoef7(24, seed=0)
    p = str(tmp_path / "v.mtx")
    P.write_matrix_market(p, a)
    b = P.load_matrix(p)
    for f in ("row_ptr", "col_idx", "vals"):
        assert np.array_equal(getattr(b, f), getattr(a, f))
    ha = P.build_hbmc(P.color_blocks(a, P.build_blocks(a, 8)), 32)
    hb = P.build_hbmc(P.color_blocks(b, P.build_blocks(b, 8)), 32)
    assert np.array_equal(ha.composed_perm.new_of_old, hb.composed_perm.new_of_old)
