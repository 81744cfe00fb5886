"""Performance model of the filter step (proj/include/chebfilter/perf_model.hpp).

KernelGeometry :17-30, RooflinePoint :32-37, arithmetic_intensity :41-45,
roofline_limit :47-51, min_traffic_volume :56-62, flop_count :64-68,
slow_memory_amortization :73-78 (host arithmetic, same formulas), and
stream_bench :80-121 measured on the device (cf_stream_bench: HBM instead of
host DRAM).  bench.py derives roofline.achieved from these definitions.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

from ._lib import check, lib


@dataclass
class KernelGeometry:
    n: int = 1
    n_nzr: float = 13.0
    entry_bytes: int = 20      # 16-byte value + 4-byte index
    vec_elem_bytes: int = 16   # complex double
    flops_per_row_per_vec: float = 146.0
    n_b: int = 1

    def validate(self) -> None:
        if (self.n_nzr <= 0 or self.entry_bytes == 0 or self.vec_elem_bytes == 0 or self.flops_per_row_per_vec <= 0
                or self.n_b == 0):
            raise ValueError("kernel geometry fields must be positive")


@dataclass
class RooflinePoint:
    p_max: float = 0.0      # flop/s
    bandwidth: float = 0.0  # bytes/s
    intensity: float = 0.0  # flop/byte
    p_star: float = 0.0     # min(p_max, intensity * bandwidth)


def arithmetic_intensity(g: KernelGeometry) -> float:
    g.validate()
    return g.flops_per_row_per_vec / (g.n_nzr * g.entry_bytes / float(g.n_b) + 5.0 * g.vec_elem_bytes)


def roofline_limit(p_max: float, bandwidth: float, intensity: float) -> RooflinePoint:
    if p_max <= 0 or bandwidth <= 0 or intensity <= 0:
        raise ValueError("roofline inputs must be positive")
    return RooflinePoint(p_max, bandwidth, intensity, min(p_max, intensity * bandwidth))


def min_traffic_volume(g: KernelGeometry) -> tuple[float, float]:
    """(read, write) bytes of one iteration: the matrix + U, W, X read; W, X written."""
    g.validate()
    read = float(g.n) * g.n_nzr * g.entry_bytes + 3.0 * g.n * g.n_b * g.vec_elem_bytes
    write = 2.0 * g.n * g.n_b * g.vec_elem_bytes
    return read, write


def flop_count(g: KernelGeometry, iterations: int) -> float:
    g.validate()
    return g.flops_per_row_per_vec * float(g.n) * float(g.n_b) * float(iterations)


def slow_memory_amortization(working_set_bytes: float, slow_bw: float, n_p: int, t_iter_fast: float) -> float:
    if working_set_bytes <= 0 or slow_bw <= 0 or n_p == 0 or t_iter_fast <= 0:
        raise ValueError("amortization inputs must be positive")
    return 1.0 + (working_set_bytes / slow_bw) / (float(n_p) * t_iter_fast)


class StreamKind(enum.Enum):
    copy = 0
    scale = 1
    add = 2
    triad = 3


def stream_bytes_per_element(kind: StreamKind) -> float:
    return 16.0 if kind in (StreamKind.copy, StreamKind.scale) else 24.0


def stream_bench(array_elems: int, kind: StreamKind, repetitions: int = 10, device: int = 0) -> float:
    """Best bytes/s of the STREAM kernel on the device (HBM)."""
    if array_elems == 0 or repetitions == 0:
        raise ValueError("stream_bench inputs must be positive")
    out = C.c_double()
    check(lib.cf_stream_bench(device, array_elems, kind.value, repetitions, C.byref(out)))
    return out.value
