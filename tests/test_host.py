"""Host half of the product (libchebfd_b200.so, no GPU needed) against the
reference fixtures and the oracle: bit-exact generator, bounds, coefficients,
RNG, partition / halo lists, shard plans, SELL-C-sigma/B4 permutation."""
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as orc
import paper_1803_02156_b200 as cf
from golden_io import bits, load, topi_cases
from paper_1803_02156_b200 import _lib


def test_library_exports_every_declared_symbol():
    hdr = (Path(__file__).resolve().parents[1] / "include" / "chebfd_b200.h").read_text()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(cf_\w+)\s*\(", hdr, flags=re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert declared == set(_lib.EXPORTED)


@pytest.mark.parametrize("case", range(len(topi_cases())))
def test_topi_generate_bit_identical(case):
    c = topi_cases()[case]
    nx, ny, nz, m, t, op = c["spec"]
    H = cf.topi_generate(cf.LatticeSpec(nx, ny, nz, m, t, cf.Boundary.open if op else cf.Boundary.periodic))
    assert np.array_equal(H.row_ptr, c["row_ptr"])
    assert np.array_equal(H.col_idx, c["col_idx"])
    assert np.array_equal(bits(H.values), bits(c["values"]))
    assert np.array_equal(bits(np.array(cf.gershgorin_bounds(H))), bits(c["bounds"]))


def test_topi_generate_matches_oracle_at_cfg1():
    H = cf.topi_generate(cf.LatticeSpec(64, 64, 40))
    O = orc.topi(64, 64, 40)
    assert np.array_equal(H.row_ptr, O.row_ptr) and np.array_equal(H.col_idx, O.col_idx)
    assert np.array_equal(bits(H.values), bits(O.values))


def test_topi_rejects_bad_extents():
    with pytest.raises(ValueError):
        cf.topi_generate(cf.LatticeSpec(0, 1, 1))


def test_coefficients_and_map_bit_identical():
    d = load("coeffs")
    k = 0
    while f"case{k}_in" in d:
        wlo, whi, lo, hi, margin, np_, damp = d[f"case{k}_in"]
        s = cf.spectral_map(lo, hi, margin)
        assert np.array_equal(bits(np.array([s.alpha, s.beta])), bits(d[f"case{k}_map"]))
        fc = cf.filter_coefficients(wlo, whi, s, int(np_), cf.Damping(int(damp)))
        assert np.array_equal(bits(fc.c), bits(d[f"case{k}_c"]))
        assert np.array_equal(bits(fc.g), bits(d[f"case{k}_g"]))
        k += 1


def test_coefficient_errors():  # test_filter.cpp:47-63
    with pytest.raises(ValueError):
        cf.spectral_map(1.0, 1.0)
    with pytest.raises(ValueError):
        cf.spectral_map(0.0, 1.0, -0.1)
    ident = cf.ShiftScale(1.0, 0.0)
    for args in [(-1.2, 0.0, ident, 20), (0.3, 0.1, ident, 20), (-0.1, 0.1, ident, 1)]:
        with pytest.raises(ValueError):
            cf.filter_coefficients(*args)


def test_rng_bit_identical():
    d = load("rng")
    for k in range(4):
        n, ns, nb, seed, off = (int(x) for x in d[f"case{k}_in"])
        x = cf.seeded_random_host(n, ns, nb, seed, off)
        assert np.array_equal(bits(x), bits(d[f"case{k}_x"].view(np.complex128)))


def _partition(H, w):
    import ctypes as C
    ln = C.c_size_t()
    _lib.check(_lib.lib.cf_partition_rows(H.n, H.row_ptr.ctypes.data, H.col_idx.ctypes.data, w, None, None,
                                          C.byref(ln)))
    ranges = np.empty(2 * w, np.uint64)
    halo = np.empty(max(ln.value, 1), np.uint64)
    _lib.check(_lib.lib.cf_partition_rows(H.n, H.row_ptr.ctypes.data, H.col_idx.ctypes.data, w,
                                          ranges.ctypes.data, halo.ctypes.data, C.byref(ln)))
    return ranges, halo[:ln.value]


def test_partition_and_halo_lists_bit_exact():
    from paper_1803_02156_b200.dist import partition_rows, shard_plan
    d = load("partition")
    k = 0
    while f"case{k}_in" in d:
        nx, ny, nz, w = (int(x) for x in d[f"case{k}_in"])
        H = cf.topi_generate(cf.LatticeSpec(nx, ny, nz))
        ranges, halo = _partition(H, w)
        assert np.array_equal(ranges, d[f"case{k}_ranges"])
        assert np.array_equal(halo, d[f"case{k}_halo"])
        plan = partition_rows(H, w)
        assert [list(r) for r in plan.row_ranges] == d[f"case{k}_ranges"].reshape(-1, 2).tolist()
        for s in range(w):
            sh = shard_plan(H, plan, s)
            ln, hn, nnz = (int(x) for x in d[f"case{k}_shard{s}_sizes"])
            assert (sh.local_n, sh.halo_n, sh.local.nnz()) == (ln, hn, nnz)
            assert np.array_equal(sh.local.row_ptr, d[f"case{k}_shard{s}_row_ptr"])
            assert np.array_equal(sh.local.col_idx, d[f"case{k}_shard{s}_col_idx"])
            assert np.array_equal(sh.halo_global, d[f"case{k}_shard{s}_halo_global"])
            assert sh.send_flat().tolist() == d[f"case{k}_shard{s}_send"].tolist()
            assert sh.recv_flat().tolist() == d[f"case{k}_shard{s}_recv"].tolist()
        k += 1


def test_partition_errors():  # test_matrix.cpp:195-199
    from paper_1803_02156_b200.dist import partition_rows
    H = cf.diagonal_matrix([1.0, 2.0, 3.0])
    with pytest.raises(ValueError):
        partition_rows(H, 4)
    with pytest.raises(ValueError):
        partition_rows(H, 0)


def _random_sparse(n, density, seed, ncols=None):
    rng = np.random.default_rng(seed)
    ncols = ncols or n
    rows, cols, vals = [], [], []
    for i in range(n):
        k = max(1, rng.binomial(ncols, density))
        cs = np.sort(rng.choice(ncols, size=min(k, ncols), replace=False))
        rows += [i] * len(cs)
        cols += list(cs)
        vals += list(rng.normal(size=len(cs)) + 1j * rng.normal(size=len(cs)))
    rp = np.zeros(n + 1, np.uint64)
    np.add.at(rp, np.array(rows) + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    return cf.SparseMatrixCRS(n, rp, np.array(cols, np.int32), np.array(vals), ncols=ncols)


@pytest.mark.parametrize("seed,n,C,sigma", [(1, 97, 8, 8), (2, 200, 8, 32), (3, 61, 4, 16), (4, 333, 16, 64)])
def test_sell_permutation_matches_checker(seed, n, C, sigma):
    H = _random_sparse(n, 0.05, seed)
    O = orc.Crs(H.n, H.row_ptr, H.col_idx, H.values)
    assert np.array_equal(cf.sell_permutation(H, None, C, sigma), orc.sell_permutation(O, None, C, sigma))
    order = np.random.default_rng(seed).permutation((n + 3) // 4).astype(np.int32)
    assert np.array_equal(cf.sell_permutation(H, order, C, sigma), orc.sell_permutation(O, order, C, sigma))


def test_sell_permutation_topi_lattice_order():
    H = cf.topi_generate(cf.LatticeSpec(8, 6, 5, boundary=cf.Boundary.open))
    O = orc.Crs(H.n, H.row_ptr, H.col_idx, H.values)
    order = np.empty(8 * 6 * 5, np.int32)
    _lib.check(_lib.lib.cf_lattice_order(8, 6, 5, 3, 4, order.ctypes.data))
    assert sorted(order.tolist()) == list(range(240))
    for sigma in (8, 32, 256):
        assert np.array_equal(cf.sell_permutation(H, order, 8, sigma), orc.sell_permutation(O, order, 8, sigma))


def test_sell_rejects_bad_parameters():
    H = cf.diagonal_matrix(np.arange(10.0))
    for C, sigma in [(6, 12), (8, 12), (0, 8), (128, 128)]:
        with pytest.raises(ValueError):
            cf.sell_permutation(H, None, C, sigma)
    with pytest.raises(ValueError):
        cf.sell_permutation(H, np.array([0, 0, 1], np.int32))


@pytest.mark.parametrize("spec,workers", [((4, 4, 4), 2), ((4, 4, 4), 3), ((4, 4, 4), 4), ((3, 3, 3), 2),
                                          ((5, 3, 8), 4), ((4, 4, 6), 6), ((2, 3, 5), 3)])
def test_topi_shard_closed_form_matches_global_sharding(spec, workers):
    from paper_1803_02156_b200.dist import partition_rows, shard_plan, topi_shard_plan
    ls = cf.LatticeSpec(*spec)
    H = cf.topi_generate(ls)
    plan = partition_rows(H, workers)
    for w in range(workers):
        a = shard_plan(H, plan, w)
        b = topi_shard_plan(ls, workers, w)
        assert (a.row_begin, a.local_n, a.halo_n) == (b.row_begin, b.local_n, b.halo_n)
        assert np.array_equal(a.local.row_ptr, b.local.row_ptr)
        assert np.array_equal(a.local.col_idx, b.local.col_idx)
        assert np.array_equal(bits(a.local.values), bits(b.local.values))
        assert np.array_equal(a.halo_global, b.halo_global)
        assert a.send_flat().tolist() == b.send_flat().tolist()
        assert a.recv_flat().tolist() == b.recv_flat().tolist()


def test_halo_plan_runs_are_contiguous_and_mirrored():
    from paper_1803_02156_b200.dist import HaloPlan, topi_shard_plan
    ls = cf.LatticeSpec(4, 4, 8)
    for workers in (2, 4):
        plans = [HaloPlan(topi_shard_plan(ls, workers, w)) for w in range(workers)]
        for p in plans:
            for peer, start, cnt in p.sends:
                # the receiver expects a run of the same length from this sender, in the same order
                lens_in = [c for (src, _, c) in plans[peer].recvs if src == p.id]
                lens_out = [c for (dst, _, c) in p.sends if dst == peer]
                assert lens_in == lens_out
        # z-slab topology: every run is a whole lattice plane of 4*nx*ny rows
        assert all(c == 4 * 4 * 4 for p in plans for (_, _, c) in p.sends + p.recvs)


def test_sell_permutation_unsorted_rows_and_duplicates():
    H = _random_sparse(90, 0.08, 7)
    rng = np.random.default_rng(1)
    rp = H.row_ptr.astype(np.int64)
    ci = H.col_idx.copy()
    for i in range(H.n):
        ci[rp[i]:rp[i + 1]] = rng.permutation(ci[rp[i]:rp[i + 1]])
    S = cf.SparseMatrixCRS(H.n, H.row_ptr, ci, H.values)
    O = orc.Crs(S.n, S.row_ptr, S.col_idx, S.values)
    assert np.array_equal(cf.sell_permutation(S, None, 8, 32), orc.sell_permutation(O, None, 8, 32))
    assert np.array_equal(cf.sell_permutation(S, None, 8, 32), cf.sell_permutation(H, None, 8, 32))


def test_sell_layout_signature_chunks_and_staging_plans():
    """Host-side build (csrc/host.cpp build_sell): a periodic Topi lattice in the
    locality order is all signature chunks (the Wilson-Dirac block-row) with a
    staging plan per chunk: 42 block columns in at most 7 runs for 8 x-sites."""
    H = cf.topi_generate(cf.LatticeSpec(32, 16, 8))
    st = cf.sparse.sell_layout_stats(H)
    assert st["chunks"] == H.n // 32 and st["pieces"] == st["chunks"]
    assert st["staged"] == 1 and st["signature_chunks"] == st["chunks"]
    assert st["max_staged"] == 42 and 5 <= st["max_runs"] <= 7
    # open boundaries: fewer blocks at the faces -> not every chunk has the signature
    Ho = cf.topi_generate(cf.LatticeSpec(32, 8, 8, boundary=cf.Boundary.open))
    so = cf.sparse.sell_layout_stats(Ho)
    assert so["staged"] == 1 and 0 < so["signature_chunks"] < so["chunks"]


def test_sell_layout_falls_back_without_plans_for_wide_chunks():
    """A chunk touching more than 44 block columns has no staging plan: the
    matrix then runs the register-gather kernel."""
    rng = np.random.default_rng(0)
    a = rng.normal(size=(400, 400)) + 1j * rng.normal(size=(400, 400))
    st = cf.sparse.sell_layout_stats(cf.from_dense(a))
    assert st["staged"] == 0 and st["signature_chunks"] == 0
    band = np.triu(np.tril(a[:200, :200], 6), -6)  # 13 diagonals: each chunk reads a narrow column band
    small = cf.sparse.sell_layout_stats(cf.from_dense(band))
    assert small["staged"] == 1 and small["max_runs"] == 1 and small["max_staged"] <= 12


@pytest.mark.parametrize("dims,tile", [((8, 6, 5), (3, 4)), ((16, 16, 4), (16, 16)), ((4, 4, 3), (2, 2))])
def test_lattice_order_boundary_first(dims, tile):
    """A slab shard's order (cf_lattice_order_boundary_first): the planes z = 0 and
    z = nz - 1 come first, each in the same tile order as the plain schedule's,
    then the interior planes in the plain schedule's order; a permutation."""
    nx, ny, nz = dims
    n = nx * ny * nz
    plain = np.empty(n, np.int32)
    bf = np.empty(n, np.int32)
    _lib.check(_lib.lib.cf_lattice_order(nx, ny, nz, *tile, plain.ctypes.data))
    _lib.check(_lib.lib.cf_lattice_order_boundary_first(nx, ny, nz, *tile, bf.ctypes.data))
    assert sorted(bf.tolist()) == list(range(n))
    plane = nx * ny
    z = bf // plane
    assert set(z[:plane]) == {0} and set(z[plane:2 * plane]) == {nz - 1} and set(z[2 * plane:]) <= set(range(1, nz - 1))
    assert np.array_equal(bf[2 * plane:], plain[(plain // plane > 0) & (plain // plane < nz - 1)])
    assert np.array_equal(bf[:plane], plain[plain // plane == 0])


def test_topi_shard_plan_declares_boundary_planes():
    """topi_shard_plan with neighbours: the local matrix keeps the lattice schedule
    with its two boundary planes first and declares them as the boundary rows."""
    from paper_1803_02156_b200 import dist as cfd
    spec = cf.LatticeSpec(4, 4, 8)
    sp = cfd.topi_shard_plan(spec, 2, 1)
    plane_rows = 4 * 4 * 4
    assert sp.local.boundary_rows == (plane_rows, plane_rows)
    order = sp.local.locality_order()
    z = order // 16
    assert set(z[:16]) == {0} and set(z[16:32]) == {3}
    assert cfd.topi_shard_plan(spec, 1, 0).local.boundary_rows is None


def test_work_units_tail_split():
    """Work units (host.cpp build_sell): at least 16 chunks, at most 32, and the last
    ~two per worker CTA half as long so the kernel's tail is short.  configs[0]
    lattice: 20,480 chunks -> 1,132 units of 16 + 296 of 8 = 1,428."""
    H = cf.topi_generate(cf.LatticeSpec(64, 64, 40))
    from paper_1803_02156_b200.sparse import sell_layout_stats
    st = sell_layout_stats(H)
    assert st["chunks"] == 20480 and st["staged"] == 1
    assert st["units"] == 18112 // 16 + (20480 - 18112) // 8
