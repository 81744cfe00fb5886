"""Loaders for the committed reference fixtures (tests/golden/*.npz)."""
from pathlib import Path

import numpy as np

G = Path(__file__).resolve().parent / "golden"


def load(name):
    return np.load(G / f"{name}.npz")


def topi_cases():
    d = load("topi")
    k = 0
    out = []
    while f"case{k}_spec" in d:
        nx, ny, nz, m, t, op = d[f"case{k}_spec"]
        out.append(dict(spec=(int(nx), int(ny), int(nz), float(m), float(t), bool(op)),
                        row_ptr=d[f"case{k}_row_ptr"], col_idx=d[f"case{k}_col_idx"],
                        values=d[f"case{k}_values"].view(np.complex128), bounds=d[f"case{k}_bounds"]))
        k += 1
    return out


def bits(a):
    """Exact bit pattern view (distinguishes -0.0 and +0.0)."""
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype in (np.float64, np.complex128) else a
