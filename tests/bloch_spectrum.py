"""Full analytic spectrum of a periodic Topi lattice from its 4x4 Bloch matrices
(TEST INFRASTRUCTURE ONLY; tests/bloch.py): eigenvalues of H(k) over all
k = 2 pi j / N, one z-layer of wave numbers at a time."""
from __future__ import annotations

import numpy as np

import bloch


def spectrum(dims, mass=1.0, hop=1.0) -> np.ndarray:
    blocks = bloch.site_blocks(mass, hop)
    nx, ny, nz = dims
    kx, ky = np.meshgrid(2 * np.pi * np.arange(nx) / nx, 2 * np.pi * np.arange(ny) / ny, indexing="ij")
    out = []
    for jz in range(nz):
        ks = np.stack([kx.ravel(), ky.ravel(), np.full(nx * ny, 2 * np.pi * jz / nz)], -1)
        hk = sum(b[None] * np.exp(1j * (ks @ np.array(d, float)))[:, None, None] for d, b in blocks.items())
        out.append(np.linalg.eigvalsh(hk).ravel())
    return np.sort(np.concatenate(out))
