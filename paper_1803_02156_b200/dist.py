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
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import ProtocolError, check, lib, ptr
from .blockvec import BlockVector, SubblockView, swap_blocks
from .filter import FilterCoefficients
from .kernels import MomentSeries, TrafficCounter, chebfd_op, spmmv_shifted
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


def topi_shard_plan(spec, workers: int, w: int) -> ShardPlan:
    """shard_plan(topi_generate(spec), partition_rows(.., workers), w) in closed form:
    only worker w's rows are generated (cf_topi_shard); bit-identical plans."""
    from .sparse import Boundary
    op = 1 if spec.boundary == Boundary.open else 0
    a = [C.c_size_t() for _ in range(4)]
    sl, rl = C.c_size_t(), C.c_size_t()
    args = (spec.nx, spec.ny, spec.nz, spec.mass, spec.hop, op, workers, w)
    check(lib.cf_topi_shard(*args, *[C.byref(x) for x in a], None, None, None, None, None, C.byref(sl), None,
                            C.byref(rl)))
    rb, ln, hn, nnz = (x.value for x in a)
    rp = np.empty(ln + 1, np.uint64)
    ci = np.empty(nnz, np.int32)
    v = np.empty(nnz, np.complex128)
    hg = np.empty(max(hn, 1), np.uint64)
    sf = np.empty(max(sl.value, 1), np.uint64)
    rf = np.empty(max(rl.value, 1), np.uint64)
    check(lib.cf_topi_shard(*args, *[C.byref(x) for x in a], ptr(rp), ptr(ci), ptr(v), ptr(hg), ptr(sf),
                            C.byref(sl), ptr(rf), C.byref(rl)))
    lattice = None
    sites_per_plane = spec.nx * spec.ny
    slab = ln % (4 * sites_per_plane) == 0 and rb % (4 * sites_per_plane) == 0
    if slab:  # a z-slab: keep the locality schedule; with neighbours, its boundary planes first
        lattice = (spec.nx, spec.ny, ln // (4 * sites_per_plane), workers > 1)
    local = SparseMatrixCRS(ln, rp, ci, v, ncols=ln + hn, lattice=lattice)
    if slab and workers > 1 and ln >= 2 * 4 * sites_per_plane:
        local.boundary_rows = (4 * sites_per_plane, 4 * sites_per_plane)
    return ShardPlan(w, rb, rb + ln, ln, hn, local, hg[:hn], _unflatten(sf[:sl.value]), _unflatten(rf[:rl.value]))


def _runs(idx: np.ndarray):
    """Split an index list into maximal ascending runs of consecutive values -> [(pos, start, len)]."""
    out = []
    if idx.size == 0:
        return out
    brk = np.nonzero(np.diff(idx.astype(np.int64)) != 1)[0] + 1
    starts = np.concatenate([[0], brk])
    ends = np.concatenate([brk, [idx.size]])
    for s, e in zip(starts, ends):
        out.append((int(s), int(idx[s]), int(e - s)))
    return out


class HaloPlan:
    """Message schedule of one shard's halo exchange (dist.hpp:110-144).

    Each neighbour's rows travel as runs of consecutive global rows, so both
    sides agree on the cut points and every message is a contiguous slice of
    the panel on the sender (owned rows) and on the receiver (halo slots):
    no pack or unpack kernel, and NCCL send/recv move panel memory directly.
    """

    def __init__(self, sp: ShardPlan):
        self.id = sp.id
        self.sends = []  # (peer, local_row_start, nrows) in plan order
        self.recvs = []  # (peer, halo_row_start, nrows)
        for nr in sp.send_plan:
            for _, start, cnt in _runs(nr.rows):
                self.sends.append((nr.neighbor, start, cnt))
        pos = 0
        for nr in sp.recv_plan:
            glob = sp.halo_global[pos:pos + nr.rows.size]
            for off, _, cnt in _runs(glob):
                self.recvs.append((nr.neighbor, int(nr.rows[off]), cnt))
            pos += nr.rows.size

    def messages(self):
        return len(self.sends) + len(self.recvs)


class TorchDistExchange:
    """Halo exchange over torch.distributed point-to-point ops (NCCL on GPUs,
    gloo in the CPU tests): one batch of isend/irecv per panel exchange,
    posted on NCCL's stream; wait() orders the current stream after it."""

    def __init__(self, plan: HaloPlan, group=None):
        import torch.distributed as tdist
        self.tdist = tdist
        self.plan = plan
        self.group = group
        self._pending = {}

    def start(self, panel: torch.Tensor, key=0):
        if key in self._pending:
            raise ProtocolError("halo_exchange: exchange already outstanding on panel")
        ops = []
        P2P = self.tdist.P2POp
        for peer, start, cnt in self.plan.recvs:
            ops.append(P2P(self.tdist.irecv, panel[start:start + cnt], peer, self.group))
        for peer, start, cnt in self.plan.sends:
            ops.append(P2P(self.tdist.isend, panel[start:start + cnt], peer, self.group))
        self._pending[key] = self.tdist.batch_isend_irecv(ops) if ops else []

    def finish(self, key=0):
        if key not in self._pending:
            raise ProtocolError("halo_exchange: finalize without init")
        for r in self._pending.pop(key):
            r.wait()

    def exchange(self, panel: torch.Tensor, key=0):
        self.start(panel, key)
        self.finish(key)


class DeviceBuffer:
    """A cudaMalloc'd block (cf_dev_alloc) seen as a torch tensor through
    __cuda_array_interface__: its IPC handle addresses exactly this buffer."""

    def __init__(self, shape, device: torch.device):
        self.device = torch.device(device)
        nbytes = int(np.prod(shape)) * 16
        p = C.c_void_p()
        check(lib.cf_dev_alloc(self.device.index, nbytes, C.byref(p)))
        self.ptr = p.value
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<c16", "data": (self.ptr, False),
                                         "version": 3, "strides": None}
        with torch.cuda.device(self.device):
            self.tensor = torch.as_tensor(self, device=self.device)
        self.tensor.zero_()

    def ipc_handle(self) -> bytes:
        h = (C.c_char * 64)()
        check(lib.cf_ipc_get_handle(self.ptr, h))
        return bytes(h)

    def __del__(self):
        if getattr(self, "ptr", None):
            lib.cf_dev_free(self.ptr)
            self.ptr = None


def peer_block_vector(rows: int, ns: int, nb: int, device, init=None) -> tuple[BlockVector, list]:
    """BlockVector whose panels are DeviceBuffers (IPC-shareable); returns it and the buffers."""
    X = BlockVector(rows, ns, nb, device="cpu")
    bufs = [DeviceBuffer((rows, nb), device) for _ in range(ns // nb)]
    X.device = torch.device(device)
    X._panels = [bf.tensor for bf in bufs]
    X._buffers = bufs  # the panels view these allocations: keep them alive with the vector
    if init is not None:
        host = X.__class__(rows, ns, nb, init, device="cpu")
        for b in range(X.panel_count()):
            X._panels[b].copy_(host.panel(b))
    return X, bufs


class RankPeers:
    """Fused halo exchange for one process per GPU (torchrun): the neighbours'
    panels are opened through CUDA IPC, and every kernel writing a vector the
    neighbours hold as halo stores those rows straight into their halo slots
    (cf_mirror, peer stores over NVLink).  `barrier()` orders a rank's next step
    after every neighbour's mirrored stores landed and after every neighbour
    finished reading the panel it is about to overwrite: per-neighbour step flags
    in peer memory (default; cf_flag_signal / cf_flag_wait, stream memory
    operations, no SM held and no global collective, so a slow rank only holds
    up its two slab neighbours), or with flags=False a one-element all-reduce on
    the current stream (NCCL) / a host barrier (gloo).

    `tensors`: {tag: DeviceBuffer} of this rank; every rank registers the same
    tags (e.g. ("U", b), ("W", b), ("X", b)).  swap_blocks exchanges tensors, so
    `mirror(t)` looks up the tag of the tensor being written."""

    def __init__(self, plan: HaloPlan, buffers: dict, group=None, flags: bool = True):
        import torch.distributed as tdist
        self.tdist, self.group = tdist, group
        self.rank = tdist.get_rank(group)
        self.device = next(iter(buffers.values())).device
        self.tag_of = {bf.ptr: tag for tag, bf in buffers.items()}
        world = tdist.get_world_size(group)
        # per-neighbour step flags (cf_flag_signal / cf_flag_wait): slot v of a rank's
        # flag array holds the last step neighbour v completed
        self._flags = DeviceBuffer((world,), self.device) if flags else None
        fh = self._flags.ipc_handle() if flags else None
        torch.cuda.synchronize(self.device)  # flag slots zeroed before any neighbour can signal
        mine = (self.rank, plan.sends, plan.recvs, {tag: bf.ipc_handle() for tag, bf in buffers.items()}, fh)
        allinfo = [None] * world
        tdist.all_gather_object(allinfo, mine, group=group)
        plans = {r: info for r, *info in allinfo}
        self.pairs = {}
        self.remote = {}  # (peer, tag) -> device pointer
        self._opened = []
        for v in sorted({peer for peer, _, _ in plan.sends}):
            sends = [(st, cnt) for peer, st, cnt in plan.sends if peer == v]
            recvs = [(st, cnt) for peer, st, cnt in plans[v][1] if peer == self.rank]
            if [c for _, c in sends] != [c for _, c in recvs]:
                raise ProtocolError("halo plans of the two ranks disagree")
            self.pairs[v] = [(a, c, r) for (a, c), (r, _) in zip(sends, recvs)]
            for tag, h in plans[v][2].items():
                if v == self.rank:
                    self.remote[(v, tag)] = buffers[tag].ptr
                    continue
                self.remote[(v, tag)] = self._open(h)
        self.neighbours = sorted(({p for p, _, _ in plan.sends} | {p for p, _, _ in plan.recvs}) - {self.rank})
        self._remote_flag = {}
        if flags:
            for v in self.neighbours:
                self._remote_flag[v] = self._open(plans[v][3]) + 16 * self.rank
        self._k = 0
        self.early_steps = 0  # steps whose kernel raised the neighbours' flags itself
        self._flag = torch.zeros(1, device=self.device if tdist.get_backend(group) == "nccl" else "cpu")

    def _open(self, h):
        ptr_ = C.c_void_p()
        check(lib.cf_ipc_open_handle(self.device.index, (C.c_char * 64).from_buffer_copy(h), C.byref(ptr_)))
        self._opened.append(ptr_.value)
        return ptr_.value

    def _runs(self, out: torch.Tensor):
        tag = self.tag_of[out.data_ptr()]
        nb = out.shape[1]
        runs = []
        for v, pairs in self.pairs.items():
            base = self.remote[(v, tag)]
            for start, cnt, rstart in pairs:
                runs.append((start, start + cnt, base + rstart * nb * 16))
        return runs

    def mirror(self, out: torch.Tensor):
        """Mirror runs of `out` for the kernels' fused stores (cf_mirror), or None when
        the plan has more than the kernels' 4 runs: after_step() then copies them."""
        runs = self._runs(out)
        return runs if len(runs) <= 4 else None

    def _copy(self, panel: torch.Tensor):
        # on the caller's current stream: ordered after the kernel that wrote `panel`
        st = torch.cuda.current_stream(self.device).cuda_stream
        nb = panel.shape[1]
        for start, end, dst in self._runs(panel):
            check(lib.cf_memcpy_async(dst, panel[start:end].data_ptr(), (end - start) * nb * 16, st))

    def after_step(self, out: torch.Tensor):
        """Halo rows of `out` that no kernel mirrored (plans of more than 4 runs):
        copied into the neighbours' halo slots (peer copies on the current stream)."""
        if len(self._runs(out)) > 4:
            self._copy(out)

    def push(self, panel: torch.Tensor):
        """Owned rows of an input vector into the neighbours' halo slots (recurrence start)."""
        self._copy(panel)
        self.barrier()

    def step_signal(self):
        """(neighbour flag slots, k) for a step that raises its own "step k done"
        (cf_chebfd_step_signal: from inside the kernel once its boundary units are
        done); follow it with wait(k).  None without flags."""
        if self._flags is None:
            return None
        self._k += 1
        return [self._remote_flag[v] for v in self.neighbours], self._k

    def wait(self, k: int):
        """The current stream waits until every neighbour raised step k."""
        st = torch.cuda.current_stream(self.device).cuda_stream
        for v in self.neighbours:
            check(lib.cf_flag_wait(self._flags.ptr + 16 * v, k, st))

    def barrier(self):
        """Device-side ordering after a step: with flags, signal "step k done" into
        every neighbour's flag slot and make the stream wait for each neighbour's
        step k (nearest-neighbour lockstep, no global collective); without flags,
        a one-element all-reduce on the stream (NCCL) or a host barrier (gloo)."""
        if self._flags is not None:
            self._k += 1
            st = torch.cuda.current_stream(self.device).cuda_stream
            for v in self.neighbours:
                check(lib.cf_flag_signal(self._remote_flag[v], self._k, st))
            for v in self.neighbours:
                check(lib.cf_flag_wait(self._flags.ptr + 16 * v, self._k, st))
        elif self._flag.is_cuda:
            self.tdist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.synchronize(self.device)
            self.tdist.barrier(group=self.group)

    def close(self):
        for p in self._opened:
            lib.cf_ipc_close(p)
        self._opened = []


class FilterOps:
    """Device operators the distributed driver calls (the sm_100a kernels)."""

    def __init__(self, H: SparseMatrixCRS, s):
        self.H, self.s = H, s

    def spmmv(self, X, U, mirror=None):
        spmmv_shifted(self.H, self.s, X, U, mirror=mirror)

    def init_tail(self, X, U, W, g0c0, g1c1, g2c2, mirror=None):
        from .kernels import cheb_init_tail
        cheb_init_tail(self.H, self.s, X, U, W, g0c0, g1c1, g2c2, mirror=mirror)

    def step(self, U, W, X, p, gc, mom, col, mirror=None):
        chebfd_op(self.H, self.s, U, W, X, p, gc, mom, col, mirror=mirror)

    def grouped_step(self, U, W, X, d, mom, col, mirror=None, signal=None):
        """One step of apply_filter's grouped schedule (kernels.degree_schedule);
        signal: see kernels.chebfd_step."""
        from .kernels import chebfd_step
        return chebfd_step(self.H, self.s, U, W, X, d, mom, col, mirror=mirror, signal=signal)


@dataclass
class TimelineEvent:
    """dist.hpp:146-153, measured: kind "compute" (a degree step's kernels, halo
    stores included) or "comm" (the wait for the neighbours' step flags / the
    halo exchange), panel `block`, degree `degree`, start / end in ms from the
    first recorded event (CUDA events on the rank's stream)."""
    kind: str
    block: int
    degree: int
    start: float
    end: float


@dataclass
class Timeline:
    """dist.hpp:155-162."""
    events: list = field(default_factory=list)

    def makespan(self) -> float:
        return max((e.end for e in self.events), default=0.0)

    def totals(self) -> dict:
        out = {"compute": 0.0, "comm": 0.0}
        for e in self.events:
            out[e.kind] += e.end - e.start
        return out


class _EventLog:
    """CUDA events on the current stream, resolved into a Timeline after a sync."""

    def __init__(self, device):
        self.device, self.marks = device, []

    def mark(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream(self.device))
        return e

    def add(self, kind, block, degree, a, b):
        self.marks.append((kind, block, degree, a, b))

    def resolve(self, tl: Timeline):
        if not self.marks:
            return tl
        torch.cuda.synchronize(self.device)
        t0 = self.marks[0][3]
        for kind, block, degree, a, b in self.marks:
            tl.events.append(TimelineEvent(kind, block, degree, t0.elapsed_time(a), t0.elapsed_time(b)))
        return tl


def filter_rank(ops, X: BlockVector, U: BlockVector, W: BlockVector, fc: FilterCoefficients, mode: CommMode,
                exch, moments: MomentSeries) -> MomentSeries:
    """One worker's body of filter_distributed (dist.hpp:241-311) for one process:
    X, U, W hold local rows + halo slots; `exch` moves halo rows between ranks.
    The degree loop is apply_filter's grouped schedule (X updated once per three
    degrees); halo traffic and moments are per degree as in the reference."""
    from .kernels import degree_schedule
    sched = degree_schedule(fc)
    panels = X.panel_count()
    nb = X.block_width()
    g0c0, g1c1, g2c2 = fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2]
    for b in range(panels):  # recurrence start (:250-262)
        Xb, Ub, Wb = SubblockView(X, b), SubblockView(U, b), SubblockView(W, b)
        exch.exchange(X.panel(b), ("X", b))
        ops.spmmv(Xb, Ub)
        exch.exchange(U.panel(b), ("U", b))
        ops.init_tail(Xb, Ub, Wb, g0c0, g1c1, g2c2)
    if mode == CommMode.vector:  # Alg. 3 (:268-282)
        for b in range(panels):
            for d in sched:
                swap_blocks(SubblockView(W, b), SubblockView(U, b))
                exch.exchange(U.panel(b), ("U", b))
                ops.grouped_step(SubblockView(U, b), SubblockView(W, b), SubblockView(X, b), d, moments, b * nb)
    else:  # Alg. 4 (:283-311): panel b+1's halo travels while panel b computes
        for d in sched:
            for b in range(panels):
                swap_blocks(SubblockView(W, b), SubblockView(U, b))
            exch.exchange(U.panel(0), ("U", 0))
            for b in range(panels - 1):
                exch.start(U.panel(b + 1), ("U", b + 1))
                ops.grouped_step(SubblockView(U, b), SubblockView(W, b), SubblockView(X, b), d, moments, b * nb)
                exch.finish(("U", b + 1))
            last = panels - 1
            ops.grouped_step(SubblockView(U, last), SubblockView(W, last), SubblockView(X, last), d, moments,
                             last * nb)
    return moments


def filter_rank_peer(ops, X: BlockVector, U: BlockVector, W: BlockVector, fc: FilterCoefficients, mode: CommMode,
                     peers: RankPeers, moments: MomentSeries, timeline: Timeline | None = None) -> MomentSeries:
    """filter_rank with the halo exchange fused into the kernels (RankPeers): each
    step mirrors its boundary rows into the neighbours' next-U halo slots; one
    device-side barrier per step (vector mode) or per degree (pipelined mode)
    orders a rank's next reads after its neighbours' stores.  Degree loop: apply_filter's
    grouped schedule (X updated once per three degrees).  `timeline`: filled with
    the measured compute / comm intervals of every (panel, degree) of the degree
    loop (dist.hpp:216-219's timelines, from CUDA events instead of a model)."""
    from .kernels import degree_schedule
    sched = degree_schedule(fc)
    panels, nb = X.panel_count(), X.block_width()
    g0c0, g1c1, g2c2 = fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2]
    log = _EventLog(X.device) if timeline is not None else None
    for b in range(panels):  # recurrence start (dist.hpp:250-262)
        Xb, Ub, Wb = SubblockView(X, b), SubblockView(U, b), SubblockView(W, b)
        peers.push(X.panel(b))
        ops.spmmv(Xb, Ub, mirror=peers.mirror(U.panel(b)))
        peers.after_step(U.panel(b))
        peers.barrier()
        ops.init_tail(Xb, Ub, Wb, g0c0, g1c1, g2c2, mirror=peers.mirror(W.panel(b)))
        peers.after_step(W.panel(b))
        peers.barrier()

    def step(b, d, signal=False):
        """One degree step of panel b; signal: this step raises the neighbours' flags
        itself (early, from the kernel, when the plan's halo is fused into mirror
        runs); returns the step value to wait for, or None (then barrier())."""
        a = log.mark() if log else None
        swap_blocks(SubblockView(W, b), SubblockView(U, b))
        mir = peers.mirror(W.panel(b))
        sig = peers.step_signal() if (signal and mir is not None) else None
        if ops.grouped_step(SubblockView(U, b), SubblockView(W, b), SubblockView(X, b), d, moments, b * nb,
                            mirror=mir, signal=sig):
            peers.early_steps += 1
        peers.after_step(W.panel(b))
        if log:
            log.add("compute", b, d[0], a, log.mark())
        return None if sig is None else sig[1]

    def sync(b, d, k):
        a = log.mark() if log else None
        if k is None:
            peers.barrier()
        else:
            peers.wait(k)
        if log:
            log.add("comm", b, d[0], a, log.mark())

    if mode == CommMode.vector:
        for b in range(panels):
            for d in sched:
                sync(b, d, step(b, d, signal=True))
    else:
        for d in sched:
            for b in range(panels - 1):
                step(b, d)
            sync(panels - 1, d, step(panels - 1, d, signal=True))
    if log:
        log.resolve(timeline)
    return moments


def filter_rank_peer_staged(ops, X: BlockVector, U: BlockVector, W: BlockVector, slots, fc: FilterCoefficients,
                            peers: RankPeers, moments: MomentSeries) -> MomentSeries:
    """filter_rank_peer with X host-staged (configs[3]: a rank's X exceeds its
    GPU): X is a host BlockVector (pinned panels of local_n + halo_n rows, e.g.
    host_block_vector), `slots` two device panel tensors registered with `peers`
    (DeviceBuffers, so the neighbours' X halo pushes land in them), U and W
    one-panel peer vectors.  The paper's slow-memory scheme
    on Alg. 3 (dist.hpp:268-282): panel b+1's owned rows are copied in on one
    stream and panel b-1's copied out on another while panel b filters with the
    fused halo; the per-panel working set (U, W, one X slot) is reused n_p - 2
    times.  Halo slots of the X slots are written by the neighbours' pushes only."""
    from .kernels import degree_schedule
    if X.device.type != "cpu":
        raise ValueError("filter_rank_peer_staged: X must be a host block vector")
    if len(slots) != 2 or U.panel_count() != 1 or W.panel_count() != 1:
        raise ValueError("filter_rank_peer_staged: two X slots and one-panel U, W")
    sched = degree_schedule(fc)
    panels, nb = X.panel_count(), X.block_width()
    own = ops.H.n
    dev = slots[0].device
    g0c0, g1c1, g2c2 = fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2]
    st = torch.cuda.current_stream(dev)
    hs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    in_ev = [torch.cuda.Event() for _ in range(panels)]
    out_ev = [torch.cuda.Event() for _ in range(panels)]

    def copy_in(b):
        with torch.cuda.stream(hs):
            if b >= 2:
                hs.wait_event(out_ev[b - 2])  # the slot's previous panel is back on the host
            slots[b % 2][:own].copy_(X.panel(b)[:own], non_blocking=True)
            in_ev[b].record(hs)

    Ub, Wb = SubblockView(U, 0), SubblockView(W, 0)
    copy_in(0)
    for b in range(panels):
        st.wait_event(in_ev[b])
        if b + 1 < panels:
            copy_in(b + 1)
        xs = slots[b % 2]
        Xv = BlockVector.__new__(BlockVector)
        Xv._n, Xv._ns, Xv._nb, Xv.device, Xv._panels = xs.shape[0], nb, nb, dev, [xs]
        Xb = SubblockView(Xv, 0)
        peers.push(xs)  # recurrence start (dist.hpp:250-262)
        ops.spmmv(Xb, Ub, mirror=peers.mirror(U.panel(0)))
        peers.after_step(U.panel(0))
        peers.barrier()
        ops.init_tail(Xb, Ub, Wb, g0c0, g1c1, g2c2, mirror=peers.mirror(W.panel(0)))
        peers.after_step(W.panel(0))
        peers.barrier()
        for d in sched:
            swap_blocks(Wb, Ub)
            ops.grouped_step(Ub, Wb, Xb, d, moments, b * nb, mirror=peers.mirror(W.panel(0)))
            peers.after_step(W.panel(0))
            peers.barrier()
        done = torch.cuda.Event()
        done.record(st)
        ds.wait_event(done)
        with torch.cuda.stream(ds):
            X.panel(b)[:own].copy_(xs[:own], non_blocking=True)
            out_ev[b].record(ds)
    for e in out_ev[-2:]:
        st.wait_event(e)
    return moments


def reduce_moments_tree(parts):
    """Rank-ordered pairwise tree (dist.hpp:344-351) over a list of (eta, mu) tensors."""
    eta = [e.clone() for e, _ in parts]
    mu = [m.clone() for _, m in parts]
    workers = len(parts)
    stride = 1
    while stride < workers:
        for w in range(0, workers - stride, 2 * stride):
            eta[w] += eta[w + stride]
            mu[w] += mu[w + stride]
        stride *= 2
    return eta[0], mu[0]


def allreduce_moments_ordered(mom: MomentSeries, group=None):
    """Gather every rank's moments and apply the rank-ordered tree on all ranks
    (deterministic, identical on every rank)."""
    import torch.distributed as tdist
    ws = tdist.get_world_size(group)
    both = torch.stack([torch.view_as_real(mom.eta), torch.view_as_real(mom.mu)])
    bufs = [torch.empty_like(both) for _ in range(ws)]
    tdist.all_gather(bufs, both, group=group)
    eta, mu = reduce_moments_tree([(torch.view_as_complex(b[0].contiguous()), torch.view_as_complex(b[1].contiguous()))
                                   for b in bufs])
    mom.eta.copy_(eta)
    mom.mu.copy_(mu)
    return mom


# ------------------------------------------------ single-process drop-in ---
@dataclass
class WorkerShard:
    """dist.hpp:19-37: plan + local U, W, X panels (local_n + halo_n rows) on a device."""
    plan: ShardPlan
    U: BlockVector
    W: BlockVector
    X: BlockVector
    exchange_pending: list
    device: torch.device | None = None  # the shard's GPU (X may be host-staged)

    @property
    def dev(self) -> torch.device:
        return self.device if self.device is not None else self.X.device

    @property
    def host_staged(self) -> bool:
        return self.X.device.type == "cpu"

    @property
    def id(self):
        return self.plan.id

    @property
    def local_n(self):
        return self.plan.local_n

    @property
    def halo_n(self):
        return self.plan.halo_n

    @property
    def row_begin(self):
        return self.plan.row_begin

    @property
    def local(self):
        return self.plan.local


def shard_and_distribute(H: SparseMatrixCRS, Xglobal: BlockVector, plan: PartitionPlan, devices=None,
                         host_panels: bool = False):
    """dist.hpp:39-98; shard w lives on devices[w % len(devices)] (default: all on X's device).
    host_panels: the shards' X panels stay in pinned host memory (the paper's
    slow-memory scheme); filter_distributed_native then stages
    them through two device slots per shard (cf_filter_distributed_host)."""
    if plan.row_ranges[-1][1] != H.n:
        raise ValueError("partition plan does not match matrix")
    if Xglobal.rows() != H.n:
        raise ValueError("block vector does not match matrix")
    devices = devices or [Xglobal.device if Xglobal.device.type == "cuda" else torch.device("cuda", 0)]
    ns, nb = Xglobal.cols(), Xglobal.block_width()
    shards = []
    for w in range(plan.worker_count):
        sp = shard_plan(H, plan, w)
        dev = torch.device(devices[w % len(devices)])
        rows = sp.local_n + sp.halo_n
        if host_panels:
            U = W = None
            X = host_block_vector(rows, ns, nb)
        else:
            U, W, X = (BlockVector(rows, ns, nb, device=dev) for _ in range(3))
        for b in range(X.panel_count()):
            X.panel(b)[:sp.local_n].copy_(Xglobal.panel(b)[sp.row_begin:sp.row_end])
        shards.append(WorkerShard(sp, U, W, X, [0] * X.panel_count(), dev))
    return shards


def host_block_vector(rows: int, ns: int, nb: int) -> BlockVector:
    """A zero BlockVector whose panels live in pinned host memory (host-staged X)."""
    X = BlockVector.__new__(BlockVector)
    X._n, X._ns, X._nb, X.device = rows, ns, nb, torch.device("cpu")
    X._panels = [torch.zeros((rows, nb), dtype=torch.complex128).pin_memory() for _ in range(ns // nb)]
    return X


class LocalTransport:
    """In-process transport between shards of one process (QueueTransport,
    wire.hpp:101-134): init copies each owned run into the receiver's halo slots
    (device-to-device, peer copies across GPUs); contiguous runs, no frames."""

    def __init__(self, shards):
        self.shards = {sh.id: sh for sh in shards}
        self.plans = {sh.id: HaloPlan(sh.plan) for sh in shards}
        self.inbox = {}

    def send_runs(self, src_id, which, b, tag):
        sh = self.shards[src_id]
        panel = getattr(sh, which).panel(b)
        for peer, start, cnt in self.plans[src_id].sends:
            self.inbox.setdefault((peer, src_id, which, b), []).append((tag, panel[start:start + cnt].clone()))

    def recv_runs(self, dst_id, which, b, tag):
        sh = self.shards[dst_id]
        panel = getattr(sh, which).panel(b)
        for peer, start, cnt in self.plans[dst_id].recvs:
            q = self.inbox.get((dst_id, peer, which, b))
            if not q:
                raise ProtocolError("halo_exchange: missing frame")
            t, data = q.pop(0)
            if t != tag:
                raise ProtocolError("halo_exchange: frame tag mismatch")
            if data.shape[0] != cnt:
                raise ProtocolError("halo_exchange: frame size mismatch")
            panel[start:start + cnt].copy_(data, non_blocking=True)


def _run_pairs(plans, w, v):
    """Matching message runs of shard w's sends to v and v's receives from w (both
    cut at the same global-row breaks): [(w_row_start, count, v_halo_start)]."""
    sends = [(st, cnt) for peer, st, cnt in plans[w].sends if peer == v]
    recvs = [(st, cnt) for peer, st, cnt in plans[v].recvs if peer == w]
    if [c for _, c in sends] != [c for _, c in recvs]:
        raise ProtocolError("halo plans of the two shards disagree")
    return [(a, c, r) for (a, c), (r, _) in zip(sends, recvs)]


class PeerTransport:
    """Fused halo exchange for shards of one process: every kernel that writes a
    vector some neighbour holds as halo (U after the init SpMMV, W after the
    fused steps) ALSO stores those rows straight into the neighbour's halo slots
    (cf_mirror; peer memory over NVLink when the shards sit on different GPUs),
    so halo_exchange (dist.hpp:110-144) costs no separate copy, send or kernel:
    the transfer overlaps the step row by row.  Stream order on one device, or a
    device synchronize across devices, stands for the neighbour's receipt."""

    def __init__(self, shards):
        self.shards = {sh.id: sh for sh in shards}
        self.plans = {sh.id: HaloPlan(sh.plan) for sh in shards}
        devs = {sh.X.device for sh in shards}
        for a in devs:
            for b2 in devs:
                if a != b2:
                    check(lib.cf_enable_peer_access(a.index, b2.index))
        self.multi_device = len(devs) > 1
        self.pairs = {}
        for w in self.shards:
            for v in {peer for peer, _, _ in self.plans[w].sends}:
                self.pairs[(w, v)] = _run_pairs(self.plans, w, v)

    def mirror(self, w, which, b):
        """Mirror runs for shard w's output vector `which` (its current panel b)."""
        runs = []
        for (src, v), pairs in self.pairs.items():
            if src != w:
                continue
            dst = getattr(self.shards[v], which).panel(b)
            nb = dst.shape[1]
            for start, cnt, rstart in pairs:
                runs.append((start, start + cnt, dst.data_ptr() + rstart * nb * 16))
        if len(runs) > 4:
            raise ValueError("fused halo exchange supports at most 4 runs per shard")
        return runs

    def push(self, which, b):
        """Owned rows of an input vector into the neighbours' halo slots (recurrence start)."""
        for (w, v), pairs in self.pairs.items():
            src = getattr(self.shards[w], which).panel(b)
            dst = getattr(self.shards[v], which).panel(b)
            for start, cnt, rstart in pairs:
                dst[rstart:rstart + cnt].copy_(src[start:start + cnt], non_blocking=True)

    def fence(self):
        if self.multi_device:
            for dev in {sh.X.device for sh in self.shards.values()}:
                torch.cuda.synchronize(dev)


def halo_exchange(shard: WorkerShard, vec: BlockVector, b: int, phase: ExchangePhase, transport: LocalTransport,
                  degree_tag: int) -> None:
    """dist.hpp:110-144 (same protocol checks)."""
    if b >= len(shard.exchange_pending) or b < 0:
        raise ValueError("panel index out of range")
    which = "U" if vec is shard.U else "W" if vec is shard.W else "X"
    if phase == ExchangePhase.init:
        if shard.exchange_pending[b]:
            raise ProtocolError("halo_exchange: exchange already outstanding on panel")
        shard.exchange_pending[b] = 1
        transport.send_runs(shard.id, which, b, degree_tag)
    else:
        if not shard.exchange_pending[b]:
            raise ProtocolError("halo_exchange: finalize without init")
        transport.recv_runs(shard.id, which, b, degree_tag)
        shard.exchange_pending[b] = 0


@dataclass
class DistributedResult:
    X: BlockVector
    moments: MomentSeries
    traffic: TrafficCounter = field(default_factory=TrafficCounter)
    timelines: list = field(default_factory=list)  # per worker, degree loop only (dist.hpp:216-219), measured


def filter_distributed(shards, fc: FilterCoefficients, mode: CommMode, transport: LocalTransport,
                       costs=None) -> DistributedResult:
    """dist.hpp:227-359 for shards of one process (possibly spread over GPUs):
    the degree loop runs worker-interleaved on the host, the kernels and halo
    copies run asynchronously on the devices; moments are reduced in the
    reference's rank-ordered tree."""
    workers = len(shards)
    if workers == 0:
        raise ValueError("no shards")
    if any(sh.host_staged for sh in shards):
        return filter_distributed_native(shards, fc, mode)  # host-staged panels: the native staging loop
    ns, nb = shards[0].X.cols(), shards[0].X.block_width()
    panels = shards[0].X.panel_count()
    moms = [MomentSeries(fc.np, ns, device=sh.X.device) for sh in shards]
    ops = [FilterOps(sh.local, fc.map) for sh in shards]

    def exchange_all(which, b, tag):
        for sh in shards:
            halo_exchange(sh, getattr(sh, which), b, ExchangePhase.init, transport, tag)
        for sh in shards:
            halo_exchange(sh, getattr(sh, which), b, ExchangePhase.finalize, transport, tag)

    g0c0, g1c1, g2c2 = fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2]
    if isinstance(transport, PeerTransport):
        _filter_fused(shards, fc, mode, transport, ops, moms)
        return _gather_result(shards, fc, moms)
    for b in range(panels):
        exchange_all("X", b, 1)
        for sh, op in zip(shards, ops):
            op.spmmv(SubblockView(sh.X, b), SubblockView(sh.U, b))
        exchange_all("U", b, 2)
        for sh, op in zip(shards, ops):
            op.init_tail(SubblockView(sh.X, b), SubblockView(sh.U, b), SubblockView(sh.W, b), g0c0, g1c1, g2c2)
    order = ([(b, p) for b in range(panels) for p in range(3, fc.np + 1)] if mode == CommMode.vector
             else [(b, p) for p in range(3, fc.np + 1) for b in range(panels)])
    for b, p in order:
        for sh in shards:
            swap_blocks(SubblockView(sh.W, b), SubblockView(sh.U, b))
        exchange_all("U", b, p)
        for sh, op, mom in zip(shards, ops, moms):
            op.step(SubblockView(sh.U, b), SubblockView(sh.W, b), SubblockView(sh.X, b), p, fc.g[p] * fc.c[p], mom,
                    b * nb)
    return _gather_result(shards, fc, moms)


class _DistWorkerC(C.Structure):
    _fields_ = [("local", C.c_void_p), ("local_n", C.c_size_t), ("halo_n", C.c_size_t), ("X_panels", C.c_void_p),
                ("send_flat", C.c_void_p), ("send_len", C.c_size_t), ("recv_flat", C.c_void_p),
                ("recv_len", C.c_size_t)]


def filter_distributed_native(shards, fc: FilterCoefficients, mode: CommMode,
                              timeline: bool = False) -> DistributedResult:
    """filter_distributed (dist.hpp:227-359) in one native call, cf_filter_distributed:
    the host loop, the per-shard streams and the step-to-step ordering run in the
    library; halo rows move with the kernels' stores over peer memory (mirror
    runs) or a push kernel; moments come back summed in the rank-ordered tree.
    timeline: also return each worker's measured Timeline of the degree loop
    (cf_filter_distributed_timeline, CUDA events per (panel, degree) step)."""
    workers = len(shards)
    if workers == 0:
        raise ValueError("no shards")
    ns, nb = shards[0].X.cols(), shards[0].X.block_width()
    host = shards[0].host_staged
    if any(sh.host_staged != host for sh in shards):
        raise ValueError("filter_distributed: every shard's X on the device or every shard's X host-staged")
    if host and mode != CommMode.vector:
        raise ValueError("host-staged panels run the vector schedule (Alg. 3); pipelined needs every panel resident")
    keep = []
    arr = (_DistWorkerC * workers)()
    for w, sh in enumerate(shards):
        dm = sh.local.device_matrix(sh.dev.index)
        panels = (C.c_void_p * sh.X.panel_count())(*[sh.X.panel(b).data_ptr() for b in range(sh.X.panel_count())])
        sf, rf = np.ascontiguousarray(sh.plan.send_flat()), np.ascontiguousarray(sh.plan.recv_flat())
        keep += [panels, sf, rf]
        arr[w] = _DistWorkerC(dm.handle, sh.local_n, sh.halo_n, C.cast(panels, C.c_void_p), sf.ctypes.data, sf.size,
                              rf.ctypes.data, rf.size)
    rows = max(fc.np - 2, 0) * ns
    eta = np.zeros(rows, np.complex128)
    mu = np.zeros(rows, np.complex128)
    m = 0 if mode == CommMode.vector else 1
    tls = []
    if timeline:
        cap = workers * 2 * shards[0].X.panel_count() * max(fc.np - 2, 0)
        rows_tl = np.zeros((max(cap, 1), 6))
        cnt = C.c_size_t()
        check(lib.cf_filter_distributed_timeline(arr, workers, ns, nb, fc.np, ptr(fc.c), ptr(fc.g), fc.map.alpha,
                                                 fc.map.beta, m, 1 if host else 0, ptr(eta), ptr(mu),
                                                 ptr(rows_tl), cap, C.byref(cnt)))
        tls = [Timeline() for _ in range(workers)]
        for w, kind, b, p, t0, t1 in rows_tl[:min(cnt.value, cap)]:
            tls[int(w)].events.append(TimelineEvent("compute" if kind == 0 else "comm", int(b), int(p), t0, t1))
    else:
        entry = lib.cf_filter_distributed_host if host else lib.cf_filter_distributed
        check(entry(arr, workers, ns, nb, fc.np, ptr(fc.c), ptr(fc.g), fc.map.alpha, fc.map.beta, m, ptr(eta),
                    ptr(mu)))
    dev0 = shards[0].X.device
    moms = MomentSeries(fc.np, ns, device=dev0)
    moms.eta.copy_(torch.from_numpy(eta))
    moms.mu.copy_(torch.from_numpy(mu))
    res = _gather_result(shards, fc, [moms])
    res.timelines = tls
    return res


def _filter_fused(shards, fc, mode, tr: PeerTransport, ops, moms):
    """filter_distributed's schedule with the halo exchange fused into the kernels'
    stores (PeerTransport): no exchange step remains, so vector and pipelined
    mode coincide up to the panel order."""
    panels, nb = shards[0].X.panel_count(), shards[0].X.block_width()
    g0c0, g1c1, g2c2 = fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2]
    for b in range(panels):
        tr.push("X", b)
        tr.fence()
        for sh, op in zip(shards, ops):
            op.spmmv(SubblockView(sh.X, b), SubblockView(sh.U, b), mirror=tr.mirror(sh.id, "U", b))
        tr.fence()
        for sh, op in zip(shards, ops):
            op.init_tail(SubblockView(sh.X, b), SubblockView(sh.U, b), SubblockView(sh.W, b), g0c0, g1c1, g2c2,
                         mirror=tr.mirror(sh.id, "W", b))
        tr.fence()
    order = ([(b, p) for b in range(panels) for p in range(3, fc.np + 1)] if mode == CommMode.vector
             else [(b, p) for p in range(3, fc.np + 1) for b in range(panels)])
    for b, p in order:
        for sh in shards:
            swap_blocks(SubblockView(sh.W, b), SubblockView(sh.U, b))
        for sh, op, mom in zip(shards, ops, moms):
            op.step(SubblockView(sh.U, b), SubblockView(sh.W, b), SubblockView(sh.X, b), p, fc.g[p] * fc.c[p], mom,
                    b * nb, mirror=tr.mirror(sh.id, "W", b))
        tr.fence()


def _gather_result(shards, fc, moms):
    ns, nb = shards[0].X.cols(), shards[0].X.block_width()
    panels = shards[0].X.panel_count()
    n = sum(sh.local_n for sh in shards)
    dev0 = shards[0].X.device
    X = BlockVector(n, ns, nb, device=dev0)
    for sh in shards:
        for b in range(panels):
            X.panel(b)[sh.row_begin:sh.row_begin + sh.local_n].copy_(sh.X.panel(b)[:sh.local_n])
    eta, mu = reduce_moments_tree([(m.eta.to(dev0), m.mu.to(dev0)) for m in moms])
    out = MomentSeries(fc.np, ns, device=dev0)
    out.eta.copy_(eta)
    out.mu.copy_(mu)
    return DistributedResult(X, out)


class TopiSlab:
    """One rank's z-slab of a Topi lattice (weak-scaling benchmark)."""

    def __init__(self, spec_global, workers: int, rank: int):
        self.plan = topi_shard_plan(spec_global, workers, rank)
        self.row_begin = self.plan.row_begin
        self.local_n = self.plan.local_n
        self.halo_n = self.plan.halo_n

    def local_matrix(self) -> SparseMatrixCRS:
        return self.plan.local


class SlabExchange(TorchDistExchange):
    def __init__(self, slab: TopiSlab, nb: int, device, group=None):
        super().__init__(HaloPlan(slab.plan), group)


# ------------------------------------------------ distributed eigensolver ---
def _gram_rows(A: BlockVector, B: BlockVector, n: int, ka: int, kb: int, group):
    """S = A^H B over this rank's n owned rows, summed over the ranks (k x k, host)."""
    import torch.distributed as tdist
    from .kernels import _stream
    S = torch.zeros((ka, kb), dtype=torch.complex128, device=A.device)
    pa = (C.c_void_p * A.panel_count())(*[A.panel(b).data_ptr() for b in range(A.panel_count())])
    pb = (C.c_void_p * B.panel_count())(*[B.panel(b).data_ptr() for b in range(B.panel_count())])
    check(lib.cf_gram(n, pa, A.block_width(), ka, pb, B.block_width(), kb, S.data_ptr(), _stream()))
    if tdist.get_backend(group) != "nccl":
        S = S.cpu()
    tdist.all_reduce(S, group=group)
    return S.cpu().numpy()


def _rotate_rows(A: BlockVector, k: int, T: np.ndarray, Y: BlockVector, n: int):
    from .kernels import _stream
    T = np.ascontiguousarray(T, np.complex128)
    pa = (C.c_void_p * A.panel_count())(*[A.panel(b).data_ptr() for b in range(A.panel_count())])
    py = (C.c_void_p * Y.panel_count())(*[Y.panel(b).data_ptr() for b in range(Y.panel_count())])
    check(lib.cf_rotate(n, pa, A.block_width(), k, ptr(T), T.shape[1], py, Y.block_width(), _stream()))


def chebfd_solve_rank(plan: ShardPlan, window_lo: float, window_hi: float, opt=None, group=None, device=None):
    """chebfd_solve (filter.hpp:247-320) for one rank of a row-block partition,
    one process per GPU.  The filter runs with the halo fused into the kernels
    (RankPeers); SVQB and Rayleigh-Ritz Gram matrices are summed over ranks
    (torch.distributed all-reduce of k x k), the k x k Jacobi problems are solved
    identically on every rank, and the rotations act on each rank's own rows.
    Returns the SolveResult with the eigenvectors' local rows."""
    import torch.distributed as tdist
    from .filter import filter_coefficients, spectral_map
    from .kernels import ShiftScale, spmmv_shifted
    from .solve import RitzPair, SolveOptions, SolveResult, jacobi_hermitian_eig
    opt = SolveOptions() if opt is None else opt
    if opt.n_b == 0 or opt.n_s == 0 or opt.n_s % opt.n_b != 0:
        raise ValueError("n_b must divide n_s")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    H = plan.local
    n, rows, ns, nb = plan.local_n, plan.local_n + plan.halo_n, opt.n_s, opt.n_b
    if nb < 32 and ns % 32 == 0 and os.environ.get("CHEBFD_SOLVE_WIDE", "1") != "0":
        nb = 32  # the solver's own block: panel width free (block-width invariance), see cf_chebfd_solve
    if opt.spectral_bounds:
        lo, hi = opt.spectral_bounds
    else:  # Gershgorin over all ranks' rows (sparse_matrix.hpp:89-107)
        a, b = C.c_double(), C.c_double()
        check(lib.cf_gershgorin_bounds(n, ptr(H.row_ptr), ptr(H.col_idx), ptr(H.values), C.byref(a), C.byref(b)))
        t = torch.tensor([-a.value, b.value], dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX, group=group)
        lo, hi = -t[0].item(), t[1].item()
    if window_lo < lo or window_hi > hi:
        raise ValueError("search window outside spectral bounds")
    fc = filter_coefficients(window_lo, window_hi, spectral_map(lo, hi, opt.margin), opt.n_p, opt.damping)
    vecs = {name: peer_block_vector(rows, ns, nb, dev) for name in ("X", "U", "W", "Q", "Y")}
    bufs = {(name, b): bf for name, (_, bl) in vecs.items() for b, bf in enumerate(bl)}
    X, U, W, Q, Y = (vecs[k][0] for k in ("X", "U", "W", "Q", "Y"))
    HQ = BlockVector(rows, ns, nb, device=dev)
    peers = RankPeers(HaloPlan(plan), bufs, group)
    ops = FilterOps(H, fc.map)
    from .blockvec import random_fill_device
    big = n * ns > (1 << 27)  # device generation above 2 GB, as cf_chebfd_solve
    host = None if big else np.empty((ns // nb, n, nb), np.complex128)
    if big:
        random_fill_device(X, opt.seed, plan.row_begin)  # halo rows are overwritten by the first push
    else:
        check(lib.cf_blockvec_random(n, ns, nb, opt.seed, plan.row_begin, ptr(host)))
        for b in range(X.panel_count()):
            X.panel(b)[:n].copy_(torch.from_numpy(host[b]))
    res = SolveResult()
    empty_streak = 0

    def svqb_pass(A, k, out):
        S = _gram_rows(A, A, n, k, k, group)
        S = np.triu(S) + np.triu(S, 1).conj().T  # upper triangle as the reference builds it
        e = jacobi_hermitian_eig(S)
        lmax = e.values[-1] if len(e.values) else 0.0
        if not lmax > 0.0:
            raise RuntimeError("svqb: all columns numerically zero")
        keep = [j for j in range(k) if e.values[j] > opt.drop_tol * lmax]
        if not keep:
            raise RuntimeError("svqb: empty basis after dropping")
        T = e.vectors[:, keep] / np.sqrt(e.values[keep])
        _rotate_rows(A, k, T, out, n)
        return len(keep)

    def defect(A, k):
        G = _gram_rows(A, A, n, k, k, group)
        return float(np.abs(G - np.eye(k)).max())

    def apply_h(A, k, out):
        for b in range((k + nb - 1) // nb):
            peers.push(A.panel(b))
            spmmv_shifted(H, ShiftScale(1.0, 0.0), SubblockView(A, b), SubblockView(out, b))

    for restart in range(1, opt.max_restarts + 1):
        res.iterations = restart
        mom = MomentSeries(fc.np, ns, device=dev)
        filter_rank_peer(ops, X, U, W, fc, CommMode.pipelined, peers, mom)
        allreduce_moments_ordered(mom, group)
        res.moments.append(mom)
        # SVQB (filter.hpp:139-150): X -> Q, extra passes Q -> X -> Q ...
        rank = svqb_pass(X, ns, Q)
        cur, other = Q, X
        for _ in range(3):
            if defect(cur, rank) <= 1e-10:
                break
            rank = svqb_pass(cur, rank, other)
            cur, other = other, cur
        # Rayleigh-Ritz (filter.hpp:170-211) on cur; HQ then Y = cur V, H Y
        if defect(cur, rank) > 1e-8:
            raise ValueError("rayleigh_ritz: basis not orthonormal")
        apply_h(cur, rank, HQ)
        S = _gram_rows(cur, HQ, n, rank, rank, group)
        S = np.triu(S) + np.triu(S, 1).conj().T
        e = jacobi_hermitian_eig(S)
        Ybuf = Y if cur is not Y else other
        _rotate_rows(cur, rank, e.vectors, Ybuf, n)
        apply_h(Ybuf, rank, HQ)
        nd = np.zeros(2 * rank)
        py = (C.c_void_p * Ybuf.panel_count())(*[Ybuf.panel(b).data_ptr() for b in range(Ybuf.panel_count())])
        ph = (C.c_void_p * HQ.panel_count())(*[HQ.panel(b).data_ptr() for b in range(HQ.panel_count())])
        from .kernels import _stream
        check(lib.cf_residual_sums(n, py, nb, ph, nb, rank, ptr(np.ascontiguousarray(e.values)), ptr(nd), _stream()))
        t = torch.from_numpy(nd)
        tdist.all_reduce(t, group=group)
        nd = t.numpy()
        resid = np.sqrt(nd[0::2]) / np.sqrt(nd[1::2])
        res.all_pairs = [RitzPair(float(v), float(r), bool(window_lo < v < window_hi),
                                  bool(window_lo < v < window_hi and r <= opt.res_tol))
                         for v, r in zip(e.values, resid)]
        inside = sum(p.inside_window for p in res.all_pairs)
        conv = sum(p.converged for p in res.all_pairs)
        if inside == 0:
            empty_streak += 1
            if empty_streak >= 2:
                res.converged = True
                break
        else:
            empty_streak = 0
        if inside > 0 and conv == inside:
            res.converged = True
            sel = [i for i, p in enumerate(res.all_pairs) if p.converged]
            res.eigenvalues = np.array([res.all_pairs[i].value for i in sel])
            res.residuals = np.array([res.all_pairs[i].residual for i in sel])
            full = torch.cat([Ybuf.panel(b)[:n] for b in range(Ybuf.panel_count())], dim=1)
            Vloc = BlockVector(n, len(sel), len(sel), device=dev)
            Vloc._panels[0].copy_(full[:, sel])
            res.eigenvectors = Vloc
            break
        # restart basis: rotated Ritz vectors + fresh random columns (filter.hpp:313-318)
        for b in range(X.panel_count()):
            X.panel(b)[:n].copy_(Ybuf.panel(b)[:n])
        if rank < ns:
            if big:
                random_fill_device(X, opt.seed + restart, plan.row_begin, first_col=rank)
            else:
                check(lib.cf_blockvec_random(n, ns, nb, opt.seed + restart, plan.row_begin, ptr(host)))
                for b in range(X.panel_count()):
                    for jj in range(nb):
                        if b * nb + jj >= rank:
                            X.panel(b)[:n, jj] = torch.from_numpy(host[b][:, jj])
    else:
        res.converged = False
    if not res.converged or res.eigenvectors is None:
        conv_pairs = [p for p in res.all_pairs if p.converged]
        if not res.converged:
            res.eigenvalues = np.array([p.value for p in conv_pairs])
            res.residuals = np.array([p.residual for p in conv_pairs])
    torch.cuda.synchronize(dev)
    tdist.barrier(group=group)
    peers.close()
    return res
