"""File formats on the path's boundary:
Matrix Market coordinate complex (matrix_market.hpp:22-106) and CFDB block
vectors (block_vector.hpp:182-229), against the reference's own readers and
writers run from oracle/_ref, and the reference's KATs (test_matrix.cpp:84-131).
Bit-exact: CRS arrays, file bytes, vector bit patterns."""
import numpy as np
import pytest

import oracle as orc
import paper_1803_02156_b200 as cf

needs_ref = pytest.mark.skipif(orc.REF is None, reason="oracle/_ref not built")


def same_crs(A, B):
    return (A.n == B.n and np.array_equal(A.row_ptr.astype(np.uint64), B.row_ptr.astype(np.uint64))
            and np.array_equal(A.col_idx, B.col_idx)
            and np.array_equal(A.values.view(np.uint64), B.values.view(np.uint64)))


def test_matrix_market_round_trip(tmp_path):
    """test_matrix.cpp:84-96."""
    H = cf.topi_generate(cf.LatticeSpec(2, 2, 2))
    p = tmp_path / "rt.mtx"
    cf.matrix_market_write(p, H)
    H2 = cf.matrix_market_read(p)
    assert same_crs(H, H2) and H2.symmetry == cf.Symmetry.hermitian


def test_matrix_market_reports_the_offending_line(tmp_path):
    """test_matrix.cpp:98-114."""
    p = tmp_path / "bad.mtx"
    p.write_text("%%MatrixMarket matrix coordinate complex general\n3 3 2\n1 1 1.0 0.0\n4 1 1.0 0.0\n")
    with pytest.raises(cf.MatrixMarketError) as e:
        cf.matrix_market_read(p)
    assert e.value.line_number == 4 and "line 4" in str(e.value)


def test_hermitian_lower_triangle_expands():
    """test_matrix.cpp:116-131."""
    import tempfile
    from pathlib import Path
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "h.mtx"
        p.write_text("%%MatrixMarket matrix coordinate complex hermitian\n2 2 3\n1 1 2.0 0.0\n2 1 1.0 -0.5\n"
                     "2 2 3.0 0.0\n")
        H = cf.matrix_market_read(p)
    E = cf.build_from_triplets(2, [cf.Triplet(0, 0, 2.0), cf.Triplet(1, 0, 1.0 - 0.5j), cf.Triplet(0, 1, 1.0 + 0.5j),
                                   cf.Triplet(1, 1, 3.0)])
    assert same_crs(H, E)


def _random_mm(rng, n, nnz, herm, comments=True):
    lines = [f"%%MatrixMarket matrix coordinate complex {'hermitian' if herm else 'general'}"]
    if comments:
        lines += ["% a comment", ""]
    lines.append(f"{n} {n} {nnz}")
    for k in range(nnz):
        i = int(rng.integers(1, n + 1))
        j = int(rng.integers(1, i + 1)) if herm else int(rng.integers(1, n + 1))
        re, im = rng.normal(), (0.0 if herm and i == j else rng.normal())
        if comments and k % 7 == 3:
            lines.append("%")
        lines.append(f"{i} {j} {re!r} {im!r}")
    return "\n".join(lines) + "\n"


@needs_ref
@pytest.mark.parametrize("herm", [True, False])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_matrix_market_read_equals_reference(tmp_path, herm, seed):
    """Random files with duplicates (summed in file order), comments, blank lines."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    p = tmp_path / "r.mtx"
    p.write_text(_random_mm(rng, n, int(rng.integers(1, 4 * n + 2)), herm))
    H = cf.matrix_market_read(p)
    R, sym = orc.ref_mm_read(p)
    assert same_crs(H, R) and (sym == 0) == (H.symmetry == cf.Symmetry.hermitian)


@needs_ref
@pytest.mark.parametrize("lattice", [(2, 2, 2), (3, 2, 5), (4, 4, 4)])
def test_matrix_market_write_is_byte_identical(tmp_path, lattice):
    H = cf.topi_generate(cf.LatticeSpec(*lattice))
    cf.matrix_market_write(tmp_path / "ours.mtx", H)
    orc.ref_mm_write(orc.Crs(H.n, H.row_ptr, H.col_idx, H.values), tmp_path / "ref.mtx")
    assert (tmp_path / "ours.mtx").read_bytes() == (tmp_path / "ref.mtx").read_bytes()
    G = cf.from_dense(np.array([[1.0, 2.0 - 1j], [-0.0, 3.5j]]), cf.Symmetry.general)
    cf.matrix_market_write(tmp_path / "g.mtx", G)
    assert same_crs(cf.matrix_market_read(tmp_path / "g.mtx"), orc.ref_mm_read(tmp_path / "g.mtx")[0])


BAD = {
    "empty": "",
    "banner": "%%MatrixMarket matrix array complex general\n1 1 1\n1 1 1 0\n",
    "field": "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1 0\n",
    "symmetry": "%%MatrixMarket matrix coordinate complex symmetric\n1 1 1\n1 1 1 0\n",
    "size": "%%MatrixMarket matrix coordinate complex general\n% c\n3 x 2\n",
    "square": "%%MatrixMarket matrix coordinate complex general\n3 4 1\n1 1 1 0\n",
    "entry": "%%MatrixMarket matrix coordinate complex general\n2 2 2\n1 1 1 0\n2 2 abc 0\n",
    "range0": "%%MatrixMarket matrix coordinate complex general\n2 2 1\n\n0 1 1 0\n",
    "eof": "%%MatrixMarket matrix coordinate complex general\n2 2 3\n1 1 1 0\n2 2 1 0\n",
    "nonfinite": "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 nan 0\n",
}


@needs_ref
@pytest.mark.parametrize("case", list(BAD))
def test_matrix_market_errors_match_reference(tmp_path, case):
    p = tmp_path / f"{case}.mtx"
    p.write_text(BAD[case])
    with pytest.raises(RuntimeError) as ref_err:
        orc.ref_mm_read(p)
    with pytest.raises(RuntimeError) as ours:
        cf.matrix_market_read(p)
    assert getattr(ours.value, "line_number", 0) == ref_err.value.line_number
    assert str(ours.value) == str(ref_err.value)


@needs_ref
@pytest.mark.parametrize("shape", [(7, 4, 2), (33, 6, 6), (1, 1, 1)])
def test_cfdb_interoperates_with_reference(tmp_path, shape):
    n, ns, nb = shape
    orc.REF.ref_bv_write(str(tmp_path / "ref.cfdb").encode(), n, ns, nb, 9)
    X = cf.block_vector_read(tmp_path / "ref.cfdb", device="cpu")
    assert (X.rows(), X.cols(), X.block_width()) == shape
    expect = cf.seeded_random_host(n, ns, nb, 9)
    assert np.array_equal(X.panels_numpy().view(np.uint64), expect.view(np.uint64))
    cf.block_vector_write(tmp_path / "ours.cfdb", X)
    assert (tmp_path / "ours.cfdb").read_bytes() == (tmp_path / "ref.cfdb").read_bytes()
    assert np.array_equal(orc.ref_bv_read(tmp_path / "ours.cfdb").view(np.uint64), expect.view(np.uint64))


def test_cfdb_rejects_corrupt_files(tmp_path):
    X = cf.BlockVector(5, 4, 2, cf.InitSeededRandom(3), device="cpu")
    p = tmp_path / "x.cfdb"
    cf.block_vector_write(p, X)
    raw = p.read_bytes()
    for name, data in {"magic": b"CFDX" + raw[4:], "version": raw[:4] + b"\x02" + raw[5:],
                       "layout": raw[:32] + b"\x01" + raw[33:], "truncated": raw[:-5]}.items():
        q = tmp_path / f"{name}.cfdb"
        q.write_bytes(data)
        with pytest.raises(RuntimeError):
            cf.block_vector_read(q, device="cpu")
