"""Block vectors in the reference's panel layout, resident in GPU memory.

Mirrors proj/include/chebfilter/block_vector.hpp: an n x n_s complex block
vector is n_s/n_b panels, each row-major n x n_b (element (i, j) in panel j//n_b
at offset i*n_b + j%n_b, :49-52, 81-94); panels are individually owned so
swap_blocks is a handle exchange (:138-142).  Each panel is one contiguous
complex128 torch tensor on the device (128-bit aligned rows of n_b*16 bytes).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import check, lib, ptr


@dataclass
class InitZero:
    pass


@dataclass
class InitConstant:
    value: complex


@dataclass
class InitSeededRandom:
    seed: int
    row_offset: int = 0


def seeded_random_host(n: int, ns: int, nb: int, seed: int, row_offset: int = 0) -> np.ndarray:
    """InitSeededRandom on the host (block_vector.hpp:17-35, 68-73), panel-concatenated
    (n_s/n_b, n, n_b) complex128; bit-identical to the reference."""
    out = np.empty((ns // nb, n, nb), np.complex128)
    check(lib.cf_blockvec_random(n, ns, nb, seed, row_offset, ptr(out)))
    return out


def random_fill_device(X: "BlockVector", seed: int, row_offset: int = 0, first_col: int = 0) -> None:
    """InitSeededRandom{seed, row_offset} generated on the device (columns >= first_col):
    for vectors too large for the host; values within 1-2 ulp of the host generator."""
    from .kernels import _stream
    panels = (C.c_void_p * X.panel_count())(*[X.panel(b).data_ptr() for b in range(X.panel_count())])
    check(lib.cf_blockvec_random_device(X.rows(), X.cols(), X.block_width(), seed, row_offset, panels, first_col,
                                        _stream()))


def _default_device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")


class BlockVector:
    def __init__(self, n: int, n_s: int, n_b: int, init=None, device=None):
        if n < 1:
            raise ValueError("n must be >= 1")
        if n_b == 0 or n_s == 0 or n_s % n_b != 0:
            raise ValueError("n_b must divide n_s")
        self._n, self._ns, self._nb = int(n), int(n_s), int(n_b)
        self.device = torch.device(device) if device is not None else _default_device()
        init = InitZero() if init is None else init
        npan = n_s // n_b
        if isinstance(init, InitSeededRandom):
            host = torch.from_numpy(seeded_random_host(n, n_s, n_b, init.seed, init.row_offset))
            self._panels = [host[b].to(self.device) for b in range(npan)]
        else:
            fill = complex(init.value) if isinstance(init, InitConstant) else 0j
            self._panels = [torch.full((n, n_b), fill, dtype=torch.complex128, device=self.device)
                            for _ in range(npan)]

    # shape -----------------------------------------------------------------
    def rows(self) -> int:
        return self._n

    def cols(self) -> int:
        return self._ns

    def block_width(self) -> int:
        return self._nb

    def panel_count(self) -> int:
        return len(self._panels)

    def panel(self, b: int) -> torch.Tensor:
        if not 0 <= b < len(self._panels):
            raise ValueError("panel index out of range")
        return self._panels[b]

    def panel_view(self, b: int) -> "BlockVector":
        """A one-panel BlockVector (n x n_b) sharing panel b's memory."""
        v = BlockVector.__new__(BlockVector)
        v._n, v._ns, v._nb, v.device = self._n, self._nb, self._nb, self.device
        v._panels = [self.panel(b)]
        return v

    def set_panel(self, b: int, t: torch.Tensor) -> None:
        self.panel(b).copy_(t)

    def linear_offset(self, i: int, j: int) -> int:
        self._check(i, j)
        return (j // self._nb) * self._n * self._nb + i * self._nb + j % self._nb

    def __getitem__(self, ij):
        i, j = ij
        self._check(i, j)
        return complex(self._panels[j // self._nb][i, j % self._nb].item())

    def __setitem__(self, ij, value):
        i, j = ij
        self._check(i, j)
        self._panels[j // self._nb][i, j % self._nb] = complex(value)

    def _check(self, i, j):
        if not (0 <= i < self._n and 0 <= j < self._ns):
            raise IndexError("block vector index out of range")

    # host conversion ---------------------------------------------------------
    def to_numpy(self) -> np.ndarray:
        """(n, n_s) complex128 in column order j."""
        return torch.cat([p.cpu() for p in self._panels], dim=1).numpy()

    def panels_numpy(self) -> np.ndarray:
        """Panel-concatenated (n_s/n_b, n, n_b) array (CFDB / reference linear order)."""
        return torch.stack([p.cpu() for p in self._panels]).numpy()

    @classmethod
    def from_numpy(cls, a: np.ndarray, n_b: int, device=None) -> "BlockVector":
        a = np.asarray(a, np.complex128)
        X = cls(a.shape[0], a.shape[1], n_b, device=device)
        for b in range(X.panel_count()):
            X._panels[b].copy_(torch.from_numpy(np.ascontiguousarray(a[:, b * n_b:(b + 1) * n_b])))
        return X


class SubblockView:
    """Non-owning handle to one panel (block_vector.hpp:116-151)."""

    def __init__(self, parent: BlockVector, b: int):
        if not 0 <= b < parent.panel_count():
            raise ValueError("panel index out of range")
        self.parent, self.b = parent, b

    def rows(self) -> int:
        return self.parent.rows()

    def width(self) -> int:
        return self.parent.block_width()

    def panel_index(self) -> int:
        return self.b

    def data(self) -> torch.Tensor:
        return self.parent._panels[self.b]

    def __getitem__(self, ij):
        i, j = ij
        if not (0 <= i < self.rows() and 0 <= j < self.width()):
            raise IndexError("subblock index out of range")
        return complex(self.data()[i, j].item())


def swap_blocks(a: SubblockView, b: SubblockView) -> None:
    """O(1) buffer exchange (block_vector.hpp:138-142)."""
    if a.rows() != b.rows() or a.width() != b.width():
        raise ValueError("swap_blocks: shape mismatch")
    pa, pb = a.parent._panels, b.parent._panels
    pa[a.b], pb[b.b] = pb[b.b], pa[a.b]


# ------------------------------------------------------ CFDB files ---
def block_vector_write(path, X: BlockVector) -> None:
    """block_vector.hpp:182-204: CFDB v1, panel row-major layout tag."""
    host = np.ascontiguousarray(X.panels_numpy())
    check(lib.cf_blockvec_write(os.fsencode(str(path)), X.rows(), X.cols(), X.block_width(), ptr(host)))


def block_vector_read(path, device=None) -> BlockVector:
    """block_vector.hpp:206-229."""
    p = os.fsencode(str(path))
    n, ns, nb = C.c_size_t(), C.c_size_t(), C.c_size_t()
    check(lib.cf_blockvec_read(p, C.byref(n), C.byref(ns), C.byref(nb), None))
    host = np.empty((ns.value // nb.value, n.value, nb.value), np.complex128)
    check(lib.cf_blockvec_read(p, C.byref(n), C.byref(ns), C.byref(nb), ptr(host)))
    X = BlockVector(n.value, ns.value, nb.value, device=device)
    for b in range(X.panel_count()):
        X._panels[b].copy_(torch.from_numpy(host[b]))
    return X
