"""Row-block distribution: partition plan, shard plans, halo exchange and the
distributed filter (Alg. 3 vector mode / Alg. 4 subspace pipelining).

Mirrors proj/include/chebfilter/partition.hpp:13-60 (PartitionPlan,
partition_rows) and dist.hpp:19-98 (WorkerShard, shard_and_distribute),
:102-144 (ProtocolError, halo_exchange), :227-359 (filter_distributed).  The
plans (row ranges, halo_in/halo_out, halo slot order, send/recv rows, local
column remap) come from the library's host code and are bit-exact with the
reference (tests/test_host.py).  The data path differs by design: the halo
rows of a panel travel device-to-device -- NCCL send/recv between ranks
(one process per GPU, torch.distributed) or peer copies between shards of one
process -- and contiguous halo runs move without packing.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import ProtocolError, check, lib, ptr
from .blockvec import BlockVector, SubblockView, swap_blocks
from .filter import FilterCoefficients
from .kernels import MomentSeries, TrafficCounter, cheb_init, chebfd_op, spmmv_shifted, spmmv_shifted_two_minus
from .sparse import SparseMatrixCRS


class CommMode(enum.Enum):
    vector = 0
    pipelined = 1


class ExchangePhase(enum.Enum):
    init = 0
    finalize = 1


@dataclass
class PartitionPlan:
    worker_count: int = 1
    row_ranges: list = field(default_factory=list)   # [(start, end)]
    halo_in: list = field(default_factory=list)      # [w] -> {v: [global rows]}
    halo_out: list = field(default_factory=list)

    def owner_of(self, row: int) -> int:
        for w, (lo, hi) in enumerate(self.row_ranges):
            if lo <= row < hi:
                return w
        raise IndexError("row not covered by partition")


def _flat_to_plan(workers, ranges, halo) -> PartitionPlan:
    plan = PartitionPlan(workers, [(int(ranges[2 * w]), int(ranges[2 * w + 1])) for w in range(workers)],
                         [dict() for _ in range(workers)], [dict() for _ in range(workers)])
    q = 0
    halo = halo.tolist()
    while q < len(halo):
        w, v, cnt = halo[q:q + 3]
        plan.halo_in[w][v] = halo[q + 3:q + 3 + cnt]
        q += 3 + cnt
    for w in range(workers):
        for v, rows in plan.halo_in[w].items():
            plan.halo_out[v][w] = list(rows)
    plan.halo_out = [dict(sorted(d.items())) for d in plan.halo_out]
    return plan


def partition_rows(H: SparseMatrixCRS, workers: int) -> PartitionPlan:
    """partition.hpp:28-60"""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    ln = C.c_size_t()
    check(lib.cf_partition_rows(H.n, ptr(H.row_ptr), ptr(H.col_idx), workers, None, None, C.byref(ln)))
    ranges = np.empty(2 * workers, np.uint64)
    halo = np.empty(max(ln.value, 1), np.uint64)
    check(lib.cf_partition_rows(H.n, ptr(H.row_ptr), ptr(H.col_idx), workers, ptr(ranges), ptr(halo),
                                C.byref(ln)))
    return _flat_to_plan(workers, ranges, halo[:ln.value])


@dataclass
class NeighborRows:
    neighbor: int
    rows: np.ndarray  # local row / halo slot indices, plan order

    def contiguous(self):
        """(start, stop) if rows form one ascending run, else None."""
        r = self.rows
        if r.size and np.all(np.diff(r.astype(np.int64)) == 1):
            return int(r[0]), int(r[-1]) + 1
        return None


@dataclass
class ShardPlan:
    """The index part of WorkerShard (dist.hpp:19-37)."""
    id: int
    row_begin: int
    row_end: int
    local_n: int
    halo_n: int
    local: SparseMatrixCRS
    halo_global: np.ndarray
    send_plan: list
    recv_plan: list

    def send_flat(self):
        return np.array([x for nr in self.send_plan for x in (nr.neighbor, nr.rows.size, *nr.rows.tolist())],
                        np.uint64)

    def recv_flat(self):
        return np.array([x for nr in self.recv_plan for x in (nr.neighbor, nr.rows.size, *nr.rows.tolist())],
                        np.uint64)


def _unflatten(flat):
    out, q = [], 0
    flat = flat.tolist()
    while q < len(flat):
        v, cnt = flat[q:q + 2]
        out.append(NeighborRows(int(v), np.array(flat[q + 2:q + 2 + cnt], np.int64)))
        q += 2 + cnt
    return out


def shard_plan(H: SparseMatrixCRS, plan: PartitionPlan, w: int) -> ShardPlan:
    """dist.hpp:39-98 for one worker (host arrays only)."""
    if plan.row_ranges[-1][1] != H.n:
        raise ValueError("partition plan does not match matrix")
    a = [C.c_size_t() for _ in range(4)]
    sl, rl = C.c_size_t(), C.c_size_t()
    check(lib.cf_shard(H.n, ptr(H.row_ptr), ptr(H.col_idx), ptr(H.values), plan.worker_count, w,
                       *[C.byref(x) for x in a], None, None, None, None, None, C.byref(sl), None, C.byref(rl)))
    rb, ln, hn, nnz = (x.value for x in a)
    rp = np.empty(ln + 1, np.uint64)
    ci = np.empty(nnz, np.int32)
    v = np.empty(nnz, np.complex128)
    hg = np.empty(max(hn, 1), np.uint64)
    sf = np.empty(max(sl.value, 1), np.uint64)
    rf = np.empty(max(rl.value, 1), np.uint64)
    check(lib.cf_shard(H.n, ptr(H.row_ptr), ptr(H.col_idx), ptr(H.values), plan.worker_count, w,
                       *[C.byref(x) for x in a], ptr(rp), ptr(ci), ptr(v), ptr(hg), ptr(sf), C.byref(sl), ptr(rf),
                       C.byref(rl)))
    local = SparseMatrixCRS(ln, rp, ci, v, H.symmetry, ncols=ln + hn)
    return ShardPlan(w, rb, rb + ln, ln, hn, local, hg[:hn], _unflatten(sf[:sl.value]), _unflatten(rf[:rl.value]))
