"""Analytic eigenvectors of the periodic Topi (Wilson-Dirac) operator -- a
size-independent answer key for the full filter (TEST INFRASTRUCTURE ONLY).

SURVEY.md App. A.2: the periodic generator (reference sparse_matrix.hpp:181-228)
is translation invariant, so a plane wave times a spinor,
    v(s, r) = exp(i k . x_s) phi_r,   k_d = 2 pi j_d / N_d,
is an eigenvector when phi is an eigenvector of the 4x4 Bloch matrix
    H(k) = sum_delta h_delta exp(i k . delta),
h_delta = the 4x4 block coupling a site to its neighbour at offset delta
(0, +-x, +-y, +-z).  The blocks are read off the library's own generator on a
4x4x4 lattice (bit-identical to the reference, tests/test_host.py), not typed
in, so the key follows the matrix under test.

The filtered vector is then exact in closed form:
    apply_filter(v) = f(lambda) v,   f(lambda) = sum_p g_p c_p T_p(alpha lambda + beta)
(filter.hpp:76-93), and the moments of the degree-p step (kernels.hpp:189-193)
are eta_p = T_p(x) T_{p-1}(x) |v|^2, mu_p = T_{p-1}(x)^2 |v|^2, with
x = alpha lambda + beta and |v|^2 = number of sites.
"""
from __future__ import annotations

import numpy as np

OFFSETS = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]


def site_blocks(mass=1.0, hop=1.0):
    """h_delta for delta in OFFSETS, from the generator's rows of one site of a
    periodic 4x4x4 lattice (extents >= 3: no wrap-summed duplicates)."""
    import paper_1803_02156_b200 as cf
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4, mass, hop))
    nx = ny = nz = 4
    s0 = (1 * ny + 1) * nx + 1  # site (1, 1, 1)
    blocks = {d: np.zeros((4, 4), np.complex128) for d in OFFSETS}
    for r in range(4):
        row = 4 * s0 + r
        for k in range(int(H.row_ptr[row]), int(H.row_ptr[row + 1])):
            col = int(H.col_idx[k])
            s1, r1 = divmod(col, 4)
            x1, y1, z1 = s1 % nx, (s1 // nx) % ny, s1 // (nx * ny)
            d = tuple(((c - 1 + 2) % 4) - 2 for c in (x1, y1, z1))  # offset from (1,1,1) in -2..1
            blocks[d][r, r1] += H.values[k]
    return blocks


def bloch_matrix(blocks, k):
    h = np.zeros((4, 4), np.complex128)
    for d, b in blocks.items():
        h += b * np.exp(1j * (k[0] * d[0] + k[1] * d[1] + k[2] * d[2]))
    return h


def pick_modes(blocks, dims, count_in, count_out, window, seed=0):
    """count_in modes with |lambda| inside the window and count_out outside it:
    (j, band, lambda, phi) with integer wave numbers j = (jx, jy, jz)."""
    rng = np.random.default_rng(seed)
    lo, hi = window
    inside, outside, seen = [], [], set()
    # near the zero level (k ~ (pi, pi, 0) and permutations) for the in-window modes
    centres = [(dims[0] // 2, dims[1] // 2, 0), (dims[0] // 2, 0, dims[2] // 2), (0, dims[1] // 2, dims[2] // 2)]
    tries = 0
    while (len(inside) < count_in or len(outside) < count_out) and tries < 200000:
        tries += 1
        if len(inside) < count_in and tries % 2:
            c = centres[rng.integers(3)]
            j = tuple(int((c[d] + rng.integers(-6, 7)) % dims[d]) for d in range(3))
        else:
            j = tuple(int(rng.integers(dims[d])) for d in range(3))
        k = [2 * np.pi * j[d] / dims[d] for d in range(3)]
        w, v = np.linalg.eigh(bloch_matrix(blocks, k))
        band = int(rng.integers(4))
        key = (j, band)
        if key in seen:
            continue
        seen.add(key)
        lam = float(w[band])
        if lo < lam < hi and len(inside) < count_in:
            inside.append((j, band, lam, v[:, band].copy()))
        elif (lam < lo - 0.2 or lam > hi + 0.2) and len(outside) < count_out:
            outside.append((j, band, lam, v[:, band].copy()))
    return inside + outside


def filter_value(fc, lam):
    """f(lambda) = sum_p g_p c_p T_p(alpha lambda + beta) (scalar recurrence)."""
    x = fc.map.alpha * lam + fc.map.beta
    tm, t = 1.0, x
    acc = fc.g[0] * fc.c[0] + fc.g[1] * fc.c[1] * t
    for p in range(2, fc.np + 1):
        tn = 2.0 * x * t - tm
        acc += fc.g[p] * fc.c[p] * tn
        tm, t = t, tn
    return acc


def moments_key(fc, lam, sites):
    """eta_p, mu_p for p = 3..n_p of one mode column (degree-major)."""
    x = fc.map.alpha * lam + fc.map.beta
    T = [1.0, x]
    for p in range(2, fc.np + 1):
        T.append(2.0 * x * T[-1] - T[-2])
    eta = np.array([T[p] * T[p - 1] for p in range(3, fc.np + 1)]) * sites
    mu = np.array([T[p - 1] ** 2 for p in range(3, fc.np + 1)]) * sites
    return eta, mu


def modes_rows(modes, dims, row0, row1, device):
    """Rows [row0, row1) of the mode panel (rows x len(modes), complex128) on
    `device` (torch): exp(i k.x_s) phi_r, phases reduced exactly (integer mod)."""
    import torch
    nx, ny, nz = dims
    rows = torch.arange(row0, row1, device=device, dtype=torch.int64)
    s, r = rows // 4, rows % 4
    x, y, z = s % nx, (s // nx) % ny, s // (nx * ny)
    out = torch.empty((row1 - row0, len(modes)), dtype=torch.complex128, device=device)
    for c, (j, _band, _lam, phi) in enumerate(modes):
        # phase / 2 pi = (jx x / nx + jy y / ny + jz z / nz) mod 1, exact in integers
        L = nx * ny * nz
        num = (j[0] * x * (L // nx) + j[1] * y * (L // ny) + j[2] * z * (L // nz)) % L
        ph = num.to(torch.float64) * (2.0 * np.pi / L)
        spin = torch.as_tensor(phi, device=device)[r]
        out[:, c] = torch.polar(torch.ones_like(ph), ph) * spin
    return out
