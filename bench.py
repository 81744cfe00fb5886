"""Benchmark of the fused Chebyshev SpMMV hot path (BASELINE.json metric).

Workload (N=1): BASELINE configs[1] -- topological insulator 4x128x128x128
(n = 8,388,608), block width n_b = 32, Chebyshev degree n_p = 500, inputs as the
reference's bench-kernel (proj/tools/chebfilter.cpp:277-294): Gershgorin bounds,
spectral map margin 0.01, window [lo+0.45 span, lo+0.55 span], Jackson damping.
A step = one fused degree step (swap + chebfd_op) over the n x 32 panel,
device-resident; flops use the paper convention 146*n*n_b per step
(perf_model.hpp:64-68) and algorithmic bytes n*(13*20 + 5*16*n_b)
(perf_model.hpp:56-62).  The panel (4.3 GB) is far larger than L2, so no flush
is needed between steps.

N>1 (torchrun, one rank per GPU): weak scaling, each rank owns a z-slab of
4x128x128x128 sites of the lattice 4x128x128x(128N) with NCCL halo exchange of
the two boundary planes per degree step.

`--impl reference` times the reference's own CPU chebfd_op (oracle/_ref, the
reference headers compiled unchanged) on this host's cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fused Chebyshev SpMMV Gflop/s + HBM GB/s vs roofline at 1/2/4/8 B200; ChebFD time"
NNZ_ROW = 13


def step_bytes(n, nb):
    """perf_model.hpp:56-62 min_traffic_volume, read + write: n (13*20 + 5*16*n_b)
    (read n(13*20 + 3*16 n_b), write 2*16 n n_b).  Inline, so that the reference
    arm never imports the product package (and never maps its library)."""
    return n * (NNZ_ROW * 20 + 3 * 16 * nb) + 2 * 16 * n * nb


def filter_bytes(n, nb, np_):
    """Algorithmic bytes of apply_filter's own schedule on one panel (perf_model.hpp
    accounting: 260 B/row of matrix per sweep, 16 B per panel element read or
    written): cheb_init = an SpMMV (X read, U written) + the fused two-minus/axpby
    (U, X read; W, X written), then per degree step 3 panel passes (U, W read, W
    written) plus 2 (X read and written) on the steps that update X."""
    import paper_1803_02156_b200 as cfm
    from paper_1803_02156_b200.kernels import degree_schedule
    fc = cfm.filter_coefficients(-0.1, 0.1, cfm.spectral_map(-1.0, 1.0), np_)
    panel = 16 * n * nb
    total = (260 * n + 2 * panel) + (260 * n + 4 * panel)
    for _p, kind, *_ in degree_schedule(fc):
        total += 260 * n + (3 if kind == 1 else 5) * panel
    return int(total)
def step_flops(n, nb):
    """perf_model.hpp:64-68 flop_count for one iteration: 146 n n_b (inline, see step_bytes)."""
    return 146 * n * nb


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload_key(nx, ny, nz, nb, kernel="M_CHEB"):
    return f"topi_4x{nx}x{ny}x{nz}_nb{nb}_{kernel}"


def ncu_traffic(key):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, one
    `ncu --set full` capture) of the dominant kernel FOR THIS WORKLOAD, from
    profiles/ncu_traffic.json (keyed by workload_key); None when no capture of
    this exact workload was committed."""
    f = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(f.read_text())
    except Exception:
        return None, None
    e = d.get(key)
    if not e:
        return None, None
    return e.get("dram_bytes_per_launch"), f"profiles/ncu_traffic.json[{key}] <- {e.get('source')}"


class ClockSampler:
    """SM clocks, power and throttle reasons sampled every ~10 ms by an NVML thread
    (nvidia-smi's query fields through nvidia-ml-py; nvidia-smi -lms 20 as the
    fallback).  Sampling starts on __enter__ and the first sample is awaited, so
    the timed region (marked by start() / stop()) is covered even when it lasts
    only ~100 ms; the summary uses the samples inside the region (at least the
    two nearest ones)."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index):
        self.index, self.rows, self.t0, self.t1 = index, [], None, None
        self._stop = threading.Event()
        self._thr = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{getattr(pr, 'pci_domain_id', 0):08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _loop_nvml(self, nv, h):
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                self.rows.append((time.monotonic(), float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), float(mx),
                                  nv.nvmlDeviceGetPowerUsage(h) / 1000.0, int(get_reasons(h))))
            except Exception:
                pass
            self._stop.wait(0.01)

    def _loop_smi(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "20",
                                     "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                    text=True)
        except OSError:
            return
        bits = [0x8, 0x40, 0x20, 0x4]
        try:
            for line in proc.stdout:
                if self._stop.is_set():
                    break
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 7 and p[0].replace(".", "").isdigit():
                    r = sum(b for b, x in zip(bits, p[3:7]) if x.lower().startswith("active"))
                    self.rows.append((time.monotonic(), float(p[0]), float(p[1]), float(p[2] or 0), r))
        finally:
            proc.terminate()

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self._thr = threading.Thread(target=self._loop_nvml, args=(nv, h), daemon=True)
        except Exception:
            self._thr = threading.Thread(target=self._loop_smi, daemon=True)
        self._thr.start()
        t_end = time.monotonic() + 10.0
        while not self.rows and self._thr.is_alive() and time.monotonic() < t_end:
            time.sleep(0.005)
        return self

    def start(self):
        self.t0 = time.monotonic()

    def stop(self):
        self.t1 = time.monotonic()

    def __exit__(self, *a):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=3)

    def summary(self):
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        t0 = self.t0 if self.t0 is not None else rows[0][0]
        t1 = self.t1 if self.t1 is not None else rows[-1][0]
        inside = [r for r in rows if t0 <= r[0] <= t1]
        if len(inside) < 2:  # a region shorter than the period: the nearest samples on both sides
            inside = sorted(rows, key=lambda r: min(abs(r[0] - t0), abs(r[0] - t1)))[:2]
        reasons = sorted({name for r in inside for name, bit in self.REASONS if r[4] & bit})
        return {"sm_mhz": float(np.median([r[1] for r in inside])), "sm_max_mhz": max(r[2] for r in inside),
                "reasons": reasons, "samples": len(inside), "power_w": float(np.median([r[3] for r in inside])),
                "region_s": round(t1 - t0, 4)}


def bench_config(args, world):
    """The workload description, byte-identical in both arms (the driver compares them)."""
    n = 4 * args.nx * args.ny * args.nz
    return {"workload": (f"topi 4x{args.nx}x{args.ny}x{args.nz * world} (BASELINE configs[1] per GPU), "
                         f"n_b={args.nb}, one fused chebfd_op degree step per panel"),
            "n_per_gpu": n, "n_total": n * world, "n_b": args.nb, "n_p": args.np, "nnz_per_row": NNZ_ROW,
            "parallelism": (f"row-block z-slabs x{world}, halo "
                            + ("fused into the kernels' stores (peer memory)" if args.halo == "peer"
                               else "NCCL send/recv") if world > 1 else "1 GPU"),
            "l2": "inputs larger than L2 (one n x n_b complex128 panel per operand), no flush needed"}


def bench_inputs(nx, ny, nz, np_):
    import paper_1803_02156_b200 as cf
    H = cf.topi_generate(cf.LatticeSpec(nx, ny, nz))
    lo, hi = cf.gershgorin_bounds(H)
    span = hi - lo
    fc = cf.filter_coefficients(lo + 0.45 * span, lo + 0.55 * span, cf.spectral_map(lo, hi, 0.01), np_)
    return H, fc


# ------------------------------------------------------------------ B200 ---
def run_b200(args):
    import torch

    import paper_1803_02156_b200 as cf
    from paper_1803_02156_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nx, ny, nz, nb, np_ = args.nx, args.ny, args.nz, args.nb, args.np
    dist_setup = None
    if world > 1:
        from paper_1803_02156_b200 import dist as cfd
        import torch.distributed as tdist
        # CHEBFD_DIST_BACKEND=gloo: functional runs of the N>1 path with ranks sharing a GPU
        backend = os.environ.get("CHEBFD_DIST_BACKEND", "nccl")
        t0 = time.time()
        tdist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
        probe = torch.ones(1, device=dev if backend == "nccl" else "cpu")
        tdist.all_reduce(probe)  # communicator set up here (NCCL creates it lazily)
        dist_setup = {"backend": backend, "init_s": round(time.time() - t0, 3),
                      "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else None,
                      "world": world}
        t0 = time.time()
        slab = cfd.TopiSlab(cf.LatticeSpec(nx, ny, nz * world), world, rank)
        H = slab.local_matrix()
        gen_s = time.time() - t0
        lo, hi = -7.0, 7.0  # Gershgorin bounds of the periodic m=t=1 lattice (row-local, rank-independent)
        span = hi - lo
        fc = cf.filter_coefficients(lo + 0.45 * span, lo + 0.55 * span, cf.spectral_map(lo, hi, 0.01), np_)
        n_local, n_rows = slab.local_n, slab.local_n + slab.halo_n
    else:
        t0 = time.time()
        H, fc = bench_inputs(nx, ny, nz, np_)
        n_local = n_rows = H.n
        gen_s = time.time() - t0
    t0 = time.time()
    dm = H.device_matrix(local)
    build_s = time.time() - t0
    n = n_local
    # panels: U, W from the recurrence start on X0 = InitSeededRandom{42} (device-resident)
    init = cf.InitSeededRandom(42, 0 if world == 1 else slab.row_begin)
    peers = exch = None
    if world > 1 and args.halo == "peer":
        X, bx = cfd.peer_block_vector(n_rows, nb, nb, dev)
        cf.blockvec.random_fill_device(X, 42, slab.row_begin)  # halo rows: overwritten by the first push
        U, bu = cfd.peer_block_vector(n_rows, nb, nb, dev)
        W, bw = cfd.peer_block_vector(n_rows, nb, nb, dev)
        peers = cfd.RankPeers(cfd.HaloPlan(slab.plan), {"X": bx[0], "U": bu[0], "W": bw[0]})
    else:
        X = cf.BlockVector(n_rows, nb, nb, init, device=dev)
        U = cf.BlockVector(n_rows, nb, nb, device=dev)
        W = cf.BlockVector(n_rows, nb, nb, device=dev)
    s = fc.map
    mom = cf.MomentSeries(np_, nb, device=dev)
    Xv, Uv, Wv = cf.SubblockView(X, 0), cf.SubblockView(U, 0), cf.SubblockView(W, 0)
    g012 = (fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2])
    if world == 1:
        cf.cheb_init(H, s, Xv, Uv, Wv, *g012)
    elif peers is not None:  # halo rows ride on the kernels' stores (cf_mirror over NVLink peer memory)
        peers.push(X.panel(0))
        cf.spmmv_shifted(H, s, Xv, Uv, mirror=peers.mirror(U.panel(0)))
        peers.barrier()
        cf.cheb_init_tail(H, s, Xv, Uv, Wv, *g012, mirror=peers.mirror(W.panel(0)))
        peers.barrier()
    else:
        exch = cfd.SlabExchange(slab, nb, dev)
        exch.exchange(X.panel(0))
        cf.spmmv_shifted(H, s, Xv, Uv)
        exch.exchange(U.panel(0))
        cf.cheb_init_tail(H, s, Xv, Uv, Wv, *g012)
    p_state = [3]

    def step():
        p = p_state[0]
        cf.swap_blocks(Wv, Uv)
        if exch is not None:
            exch.exchange(U.panel(0))
        if peers is not None:  # halo in the kernel's stores; it raises the neighbours' step flags itself
            sig = peers.step_signal()
            cf.kernels.chebfd_step(H, s, Uv, Wv, Xv, (p, 0, 0.0, 0.0, fc.g[p] * fc.c[p]), mom,
                                   mirror=peers.mirror(W.panel(0)), signal=sig)
            if sig is None:
                peers.barrier()
            else:
                peers.wait(sig[1])
        else:
            cf.chebfd_op(H, s, Uv, Wv, Xv, p, fc.g[p] * fc.c[p], mom)
        p_state[0] = 3 + (p - 2) % (np_ - 2)

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # per-step kernel timing (events bracket each fused step on the launching stream)
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e_all0, e_all1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        clk.start()
        e_all0.record(st)
        for k in range(args.steps):
            ev[k][0].record(st)
            step()
            ev[k][1].record(st)
        e_all1.record(st)
        barrier()
        clk.stop()
    total_ms = e_all0.elapsed_time(e_all1)
    launch_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    if world > 1:
        t = torch.tensor([total_ms, launch_ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        total_ms, launch_ms = t.tolist()
    ms_per_step = total_ms / args.steps
    flops = step_flops(n, nb) * world
    value = flops / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = peaks()
    achieved = step_bytes(n, nb) / (launch_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(workload_key(nx, ny, nz * world if world > 1 else nz, nb))
    clocks = clk.summary()

    # ChebFD time: one full apply_filter (n_p degrees) on the device-resident panel
    chebfd_s = None
    e2e = None
    if world > 1 and peers is not None and not args.no_e2e:
        # the distributed filter (filter_rank_peer: Alg. 4 schedule, halo fused into the
        # kernels) over the full degree, max over ranks
        momf = cf.MomentSeries(np_, nb, device=dev)
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        cfd.filter_rank_peer(cfd.FilterOps(H, fc.map), X, U, W, fc, cfd.CommMode.pipelined, peers, momf)
        a1.record(st)
        barrier()
        t = torch.tensor([a0.elapsed_time(a1) / 1e3], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        chebfd_s = t.item()
        # end to end: every rank uploads its slab of X0 from pinned host memory, filters
        # through the public per-rank driver and reads X back; wall clock, max over ranks
        host = torch.empty((n, nb), dtype=torch.complex128, pin_memory=True)
        host.copy_(torch.from_numpy(cf.seeded_random_host(n, nb, nb, 42, slab.row_begin)[0]))
        back = torch.empty_like(host, pin_memory=True)
        times = []
        for _ in range(args.e2e_steps):
            barrier()
            t0 = time.perf_counter()
            X.panel(0)[:n].copy_(host, non_blocking=True)
            momf.eta.zero_()
            momf.mu.zero_()
            cfd.filter_rank_peer(cfd.FilterOps(H, fc.map), X, U, W, fc, cfd.CommMode.pipelined, peers, momf)
            back.copy_(X.panel(0)[:n], non_blocking=True)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        t = torch.tensor([float(np.median(times))], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        t_e2e = t.item()
        e2e = {"value": step_flops(n, nb) * world * (np_ - 2) / t_e2e / 1e9, "unit": "GFlop/s",
               "h2d_bytes_per_step": int(n * nb * 16) * world, "d2h_bytes_per_step": int(n * nb * 16) * world,
               "what": f"per rank: H2D X slab, filter_rank_peer ({np_ - 2} degree steps), D2H X; max over ranks",
               "seconds_per_call": t_e2e, "calls": args.e2e_steps}
    if world == 1 and not args.no_e2e:
        Xf = cf.BlockVector(n, nb, nb, cf.InitSeededRandom(42), device=dev)
        # untimed warm-up at low degree: the filter's U/W workspace is allocated once per
        # matrix (at configs[0] size the cudaMalloc alone was a quarter of the call)
        cf.apply_filter(H, Xf, cf.filter_coefficients(fc.window_lo, fc.window_hi, fc.map, 4))
        Xf = cf.BlockVector(n, nb, nb, cf.InitSeededRandom(42), device=dev)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        cf.apply_filter(H, Xf, fc)
        a1.record(st)
        torch.cuda.synchronize()
        chebfd_s = a0.elapsed_time(a1) / 1e3
        del Xf
        # end to end through the C ABI with HOST buffers (pinned), H2D + filter + D2H inside the call
        host = torch.empty((1, n, nb), dtype=torch.complex128, pin_memory=True)
        host.copy_(torch.from_numpy(cf.seeded_random_host(n, nb, nb, 42)))
        hx = host.numpy()
        host0 = hx.copy()  # every timed call filters the same X0
        eta = np.zeros((np_ - 2) * nb, np.complex128)
        mu = np.zeros_like(eta)
        times = []
        # the first call (workspace allocation) is an untimed warm-up; then at least
        # --e2e-steps calls, and at small sizes more (until 0.5 s of timed calls, at
        # most 40): single host calls of ~15 ms showed sporadic 80-ms stalls
        it = 0
        while True:
            t0 = time.perf_counter()
            _lib.check(_lib.lib.cf_apply_filter_host(dm.handle, hx.ctypes.data, nb, nb, np_, fc.c.ctypes.data,
                                                     fc.g.ctypes.data, s.alpha, s.beta, eta.ctypes.data,
                                                     mu.ctypes.data))
            if it > 0:
                times.append(time.perf_counter() - t0)
            hx[...] = host0
            it += 1
            if len(times) >= args.e2e_steps and (sum(times) >= 0.5 or len(times) >= 40):
                break
        t_e2e = float(np.median(times))
        e2e = {"value": step_flops(n, nb) * (np_ - 2) / t_e2e / 1e9, "unit": "GFlop/s",
               "h2d_bytes_per_step": int(n * nb * 16), "d2h_bytes_per_step": int(n * nb * 16 + 2 * eta.nbytes),
               "what": f"cf_apply_filter_host: H2D X, cheb_init + {np_ - 2} fused steps, D2H X + moments",
               "seconds_per_call": t_e2e, "calls": len(times)}

    # fused-halo probe (one GPU): the same steps with the two boundary z-planes mirrored
    # into a scratch buffer, i.e. the extra stores a rank of the z-slab partition issues
    # to its neighbours over NVLink (cf_mirror), measured on the device
    mirror_probe = None
    if world == 1 and not args.no_e2e:
        plane = 4 * nx * ny
        scratch = torch.empty((2 * plane, nb), dtype=torch.complex128, device=dev)
        runs = [(0, plane, scratch.data_ptr()), (n - plane, n, scratch[plane:].data_ptr())]
        k = min(args.steps, 30)

        def timed(mirror):
            barrier()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(st)
            for _ in range(k):
                cf.swap_blocks(Wv, Uv)
                cf.chebfd_op(H, s, Uv, Wv, Xv, 3, fc.g[3] * fc.c[3], mom, mirror=mirror)
            b1.record(st)
            barrier()
            return b0.elapsed_time(b1) / k

        pairs = [(timed(None), timed(runs)) for _ in range(3)]  # alternated: clocks drift under the power cap
        plain, mirrored = float(np.median([a for a, _ in pairs])), float(np.median([b for _, b in pairs]))
        mirror_probe = {"what": f"{k} fused steps with the 2 boundary planes ({2 * plane} rows) also stored to a "
                                "second buffer (the N>1 halo stores), vs without",
                        "ms_per_step_plain": round(plain, 4), "ms_per_step_mirrored": round(mirrored, 4),
                        "overhead": round(mirrored / plain - 1.0, 4)}

    # host-staged panels (X larger than one panel lives on the host): the
    # same lattice with n_s = 4 n_b, X in pinned host memory, through cf_apply_filter_host
    # (two device panel slots; panel b+1 copied in and b-1 out while b filters) against
    # cf_apply_filter on a device-resident X: the ratio is how much of the copying hides
    panels_leg = None
    if world == 1 and not args.no_e2e and not args.no_panels:
        npan, npp = 4, 100
        fcp = cf.filter_coefficients(-0.35, 0.35, cf.spectral_map(-7.0, 7.0, 0.01), npp)  # periodic m=t=1 bounds
        Xd = cf.BlockVector(n, npan * nb, nb, device=dev)
        cf.blockvec.random_fill_device(Xd, 42)
        hostp = torch.empty((npan, n, nb), dtype=torch.complex128, pin_memory=True)
        for b in range(npan):
            hostp[b].copy_(Xd.panel(b)[:n])
        torch.cuda.synchronize()
        # untimed first call (workspace, streams, first DMA from the pinned buffer), then restore X0
        cf.apply_filter_host(H, hostp, fcp, device=local)
        for b in range(npan):
            hostp[b].copy_(Xd.panel(b)[:n])
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        cf.apply_filter(H, Xd, fcp)
        a1.record(st)
        torch.cuda.synchronize()
        dev_s = a0.elapsed_time(a1) / 1e3
        ref0 = Xd.panel(npan - 1)[:n].clone()
        del Xd
        # the copies alone (H2D + D2H of every panel, pinned, one stream), for the hidden fraction
        dpan = torch.empty((n, nb), dtype=torch.complex128, device=dev)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(st)
        for b in range(npan):
            dpan.copy_(hostp[b], non_blocking=True)
            hostp[b].copy_(dpan, non_blocking=True)
        c1.record(st)
        torch.cuda.synchronize()
        copy_s = c0.elapsed_time(c1) / 1e3
        del dpan
        t0 = time.perf_counter()
        cf.apply_filter_host(H, hostp, fcp, device=local)
        host_s = time.perf_counter() - t0
        same = bool(torch.equal(hostp[npan - 1].to(dev), ref0))
        del ref0
        panels_leg = {"what": f"cf_apply_filter_host, n_s={npan * nb} ({npan} panels of n_b={nb}), n_p={npp}, "
                              "pinned host X, two device panel slots",
                      "host_panel_bytes": int(npan * n * nb * 16), "seconds": round(host_s, 4),
                      "device_resident_seconds": round(dev_s, 4), "copy_alone_seconds": round(copy_s, 4),
                      "copy_hidden_fraction": round(1.0 - (host_s - dev_s) / copy_s, 3),
                      "gflops": round(step_flops(n, nb) * npan * (npp - 2) / host_s / 1e9, 1),
                      "bit_identical_to_device_path": same}
        del hostp

    # full ChebFD: chebfd_solve (filter -> SVQB -> Rayleigh-Ritz restarts) on the BASELINE
    # configs[0] lattice 4x64x64x40; |E| < 0.05 holds exactly the 12-fold eigenvalue 0
    solve = None
    if world == 1 and not args.no_e2e and not args.no_solve:
        Hs = cf.topi_generate(cf.LatticeSpec(64, 64, 40))
        opt = cf.SolveOptions(n_s=12, n_b=12, n_p=1500, max_restarts=12, spectral_bounds=(-4.0, 4.0))
        Hs.device_matrix(local)
        # untimed warm-up (one short restart: workspaces, first kernel loads)
        cf.chebfd_solve(Hs, -0.05, 0.05, cf.SolveOptions(n_s=12, n_b=12, n_p=20, max_restarts=1,
                                                         spectral_bounds=(-4.0, 4.0)))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = cf.chebfd_solve(Hs, -0.05, 0.05, opt)
        torch.cuda.synchronize()
        t_solve = time.perf_counter() - t0
        solve = {"what": "chebfd_solve topi 4x64x64x40 (n=655360), window (-0.05, 0.05), n_s=12, n_b=12, n_p=1500, "
                         "bounds [-4, 4]",
                 "seconds": round(t_solve, 3), "restarts": res.iterations, "converged": res.converged,
                 "eigenvalues_found": int(len(res.eigenvalues)), "expected": 12,
                 "max_abs_error_vs_analytic": float(np.abs(res.eigenvalues).max()) if len(res.eigenvalues) else None,
                 "max_residual": float(np.max(res.residuals)) if len(res.residuals) else None}
        del Hs

    # device STREAM (perf_model.hpp stream_bench on HBM), same run, for context
    stream = None
    if world == 1 and not args.no_e2e:
        from paper_1803_02156_b200.perf_model import StreamKind, stream_bench
        stream = {k.name: round(stream_bench(1 << 28, k, 5, local) / 1e9, 1) for k in StreamKind}
        stream["unit"] = "GB/s (STREAM accounting, 2^28 doubles per array, best of 5)"

    leg = None
    if not args.no_leg and (world == 1 or args.halo == "peer"):
        torch.cuda.empty_cache()
        leg = leg_large(args, world, rank, local, peaks()[0])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(H, nb, s, args.cpu_steps)

    if rank == 0:
        info = dm.info()
        staged = info.get("staged") and nb == 32
        kernel_name = ("sell_b4_staged_kernel<M_CHEB> + reduce_moments (one fused step)" if staged
                       else f"sell_b4_kernel<M_CHEB,{min(nb, 32)}> + reduce_moments (one fused step)")
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFlop/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
            "config": bench_config(args, world),
            "matrix": {"format": "SELL-C-sigma over 4x4 blocks, C=8 block-rows, chunk-staged U (TMA runs)"
                                 if staged else "SELL-C-sigma over 4x4 blocks, C=8 block-rows",
                       "device_bytes": info["device_bytes"], "work_units": info["units"]},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": kernel_name,
                         "algorithmic_bytes_per_launch": step_bytes(n, nb), "avg_launch_ms": round(launch_ms, 5),
                         "peak_source": peak_src, "traffic_source": traffic_src,
                         "frac_of_8TBs_nominal": round(achieved / 8000.0, 4)},
            "hbm_gbs_algorithmic": round(step_bytes(n, nb) * world / (ms_per_step * 1e-3) / 1e9, 1),
            "chebfd_time_s": chebfd_s,
            "apply_filter": None if chebfd_s is None else {
                "what": (f"cf_apply_filter: cheb_init + {np_ - 2} degree steps on the device-resident panel "
                         "(X updated once per three degrees)" if world == 1 else
                         f"filter_rank_peer on {world} ranks: init + {np_ - 2} degree steps, halo fused into the "
                         "kernels, max over ranks"),
                "ms_per_degree_step": round(chebfd_s * 1e3 / (np_ - 2), 4),
                "gflops": round(step_flops(n, nb) * world * (np_ - 2) / chebfd_s / 1e9, 1),
                # the reference's per-step contract (2,820 B/row at n_b = 32) over the
                # filter time: an effective rate, above the roofline when X is grouped
                "effective_gbs_per_step_contract": round(step_bytes(n, nb) * (np_ - 2) / chebfd_s / 1e9, 1),
                "effective_frac_per_step_contract": round(step_bytes(n, nb) * (np_ - 2) / chebfd_s / 1e9 / peak, 4),
                # the bytes the grouped schedule itself must move (init + degree steps)
                "algorithmic_bytes": filter_bytes(n, nb, np_),
                "algorithmic_gbs_per_gpu": round(filter_bytes(n, nb, np_) / chebfd_s / 1e9, 1),
                "frac_of_peak": round(filter_bytes(n, nb, np_) / chebfd_s / 1e9 / peak, 4)},
            "chebfd_solve": solve,
            "host_staged_panels": panels_leg,
            "halo_mirror_probe": mirror_probe,
            "leg_1e8": leg,
            "stream_device": stream,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": 2 * args.steps,
            "clocks": clocks,
            "setup_s": {"generate": round(gen_s, 2), "build_upload": round(build_s, 2)},
            "dist_setup": dist_setup,
        }
        print(json.dumps(out))
    if world > 1:
        tdist.destroy_process_group()


def leg_large(args, world, rank, local, peak):
    """The >= 1e8-row weak-scaling leg (north_star: ChebFD on a >= 10^8-row Topi
    matrix at >= 80 % parallel efficiency on 8 GPUs): every rank owns a
    4 x nxy x nxy x nz slab (default 4x512x512x12, 12.6M rows; 100.7M rows at
    N = 8) of the lattice 4 x nxy x nxy x (nz N).  T_1 = the same slab as a
    periodic lattice of its own on this GPU (no halo); T_N = the distributed
    steps with the halo fused into the kernels' stores and per-neighbour step
    flags.  Both device-timed over the same step count, max over ranks."""
    import torch

    import paper_1803_02156_b200 as cf
    from paper_1803_02156_b200 import dist as cfd
    nxy, nzr, nb = args.leg_nxy, args.leg_nz, 32
    dev = torch.device("cuda", local)
    fc = cf.filter_coefficients(-0.7, 0.7, cf.spectral_map(-7.0, 7.0, 0.01), args.np)
    s = fc.map
    g012 = (fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2])
    k = max(10, min(args.steps, 60))

    def timed(slab, peers_of):
        H = slab.local_matrix()
        rows = slab.local_n + slab.halo_n
        if peers_of:
            X, bx = cfd.peer_block_vector(rows, nb, nb, dev)
            U, bu = cfd.peer_block_vector(rows, nb, nb, dev)
            W, bw = cfd.peer_block_vector(rows, nb, nb, dev)
            peers = cfd.RankPeers(cfd.HaloPlan(slab.plan), {"X": bx[0], "U": bu[0], "W": bw[0]})
        else:
            X, U, W = (cf.BlockVector(rows, nb, nb, device=dev) for _ in range(3))
            peers = None
        cf.blockvec.random_fill_device(X, 42, slab.row_begin)
        H.device_matrix(local)
        Xv, Uv, Wv = cf.SubblockView(X, 0), cf.SubblockView(U, 0), cf.SubblockView(W, 0)
        mom = cf.MomentSeries(args.np, nb, device=dev)
        if peers:
            peers.push(X.panel(0))
            cf.spmmv_shifted(H, s, Xv, Uv, mirror=peers.mirror(U.panel(0)))
            peers.barrier()
            cf.cheb_init_tail(H, s, Xv, Uv, Wv, *g012, mirror=peers.mirror(W.panel(0)))
            peers.barrier()
        else:
            cf.cheb_init(H, s, Xv, Uv, Wv, *g012)

        def step(p):
            cf.swap_blocks(Wv, Uv)
            if peers:
                sig = peers.step_signal()
                cf.kernels.chebfd_step(H, s, Uv, Wv, Xv, (p, 0, 0.0, 0.0, fc.g[p] * fc.c[p]), mom,
                                       mirror=peers.mirror(W.panel(0)), signal=sig)
                if sig is None:
                    peers.barrier()
                else:
                    peers.wait(sig[1])
            else:
                cf.chebfd_op(H, s, Uv, Wv, Xv, p, fc.g[p] * fc.c[p], mom)

        for p in range(3, 6):
            step(p)
        if world > 1:
            import torch.distributed as tdist
            tdist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.current_stream()
        e0.record(st)
        for i in range(k):
            step(6 + i % (args.np - 6))
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        if peers:
            if world > 1:
                import torch.distributed as tdist
                tdist.barrier()
            peers.close()
        return ms, slab.local_n

    t1, n_local = timed(cfd.TopiSlab(cf.LatticeSpec(nxy, nxy, nzr), 1, 0), False)
    tn = t1
    if world > 1:
        tn, n_local = timed(cfd.TopiSlab(cf.LatticeSpec(nxy, nxy, nzr * world), world, rank), True)
        import torch.distributed as tdist
        t = torch.tensor([t1, tn], device=torch.device("cuda", local), dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        t1, tn = t.tolist()
    torch.cuda.empty_cache()
    n_tot = n_local * world
    return {"workload": f"topi 4x{nxy}x{nxy}x{nzr * world} (n={n_tot}): a 4x{nxy}x{nxy}x{nzr} z-slab per GPU, "
                        f"n_b={nb}, one fused chebfd_op degree step per step",
            "n_total": n_tot, "n_per_gpu": n_local, "steps": k,
            "ms_per_step": round(tn, 5), "ms_per_step_1gpu_slab": round(t1, 5),
            "gflops": round(step_flops(n_local, nb) * world / (tn * 1e-3) / 1e9, 1),
            "roofline_frac_per_gpu": round(step_bytes(n_local, nb) / (tn * 1e-3) / 1e9 / peak, 4),
            "parallel_efficiency": round(t1 / tn, 4),
            "halo": ("fused into the kernels' stores (peer memory), per-neighbour step flags" if world > 1
                     else "none (1 GPU: the slab as a periodic lattice)")}


# ------------------------------------------------------------- reference ---
def _ref_lib():
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle as orc
    if orc.REF is None:
        return None, orc
    return orc.REF, orc


def cpu_baseline_sample(H, nb, s, steps):
    """The reference's chebfd_op (oracle/_ref) on this host: a bounded sample of
    `steps` degree steps of the same cfg workload (setup untimed)."""
    REF, orc = _ref_lib()
    threads = min(os.cpu_count() or 1, 64)
    os.environ["CHEBFILTER_THREADS"] = str(threads)
    kind = "reference"
    if REF is None:
        return {"value": None, "unit": "GFlop/s", "cores": threads, "kind": "unavailable",
                "sample": "oracle/_ref not shipped"}
    R = orc.RefMatrix.from_crs(orc.Crs(H.n, H.row_ptr, H.col_idx, H.values))
    stp = REF.ref_step_state(R.h, nb, 42, s.alpha, s.beta)
    REF.ref_step_run(stp, 0.01)  # warm
    t0 = time.perf_counter()
    for _ in range(steps):
        REF.ref_step_run(stp, 0.01)
    dt = (time.perf_counter() - t0) / steps
    REF.ref_step_free(stp)
    return {"value": round(step_flops(H.n, nb) / dt / 1e9, 3), "unit": "GFlop/s", "cores": threads, "kind": kind,
            "sample": f"{steps} chebfd_op degree steps (+1 warm) on the full n={H.n} x n_b={nb} panel, "
                      f"{dt:.2f} s/step, CHEBFILTER_THREADS={threads}",
            "seconds_per_step": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    REF, orc = _ref_lib()
    if REF is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libchebref.so was not built/shipped"}))
        return
    threads = min(os.cpu_count() or 1, 64)
    os.environ["CHEBFILTER_THREADS"] = str(threads)
    import ctypes as C
    t0 = time.time()
    R = orc.RefMatrix.topi(args.nx, args.ny, args.nz)  # the reference's own topi_generate
    gen_s = time.time() - t0
    lo, hi = C.c_double(), C.c_double()
    REF.ref_gershgorin(R.h, C.byref(lo), C.byref(hi))
    a, b = C.c_double(), C.c_double()
    REF.ref_spectral_map(lo.value, hi.value, 0.01, C.byref(a), C.byref(b))
    n = 4 * args.nx * args.ny * args.nz
    nb = args.nb
    stp = REF.ref_step_state(R.h, nb, 42, a.value, b.value)
    budget = args.ref_budget_s
    for _ in range(args.warmup):
        REF.ref_step_run(stp, 0.01)
    times = []
    t_start = time.perf_counter()
    for k in range(args.steps):
        t0 = time.perf_counter()
        REF.ref_step_run(stp, 0.01)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget:
            break
    REF.ref_step_free(stp)
    dt = float(np.mean(times))
    value = step_flops(n, nb) / dt / 1e9
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFlop/s", "n_gpus": 0,
           "steps": len(times), "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
           "config": bench_config(args, world),
           "cpu_baseline": {"value": round(value, 3), "unit": "GFlop/s", "cores": threads, "kind": "reference",
                            "sample": f"{len(times)} of {args.steps} requested chebfd_op steps (budget {budget:.0f} s) on "
                                      f"one GPU's share, topi 4x{args.nx}x{args.ny}x{args.nz} (n={n}), n_b={nb}; "
                                      f"reference topi_generate {gen_s:.1f} s untimed"},
           "e2e": {"value": round(value, 3), "unit": "GFlop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--ny", type=int, default=128)
    ap.add_argument("--nz", type=int, default=128)
    ap.add_argument("--nb", type=int, default=32)
    ap.add_argument("--degree", "--np", dest="np", type=int, default=500)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--ref-budget-s", type=float, default=120.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-panels", action="store_true")
    ap.add_argument("--no-leg", action="store_true", help="skip the >=1e8-row weak-scaling leg")
    ap.add_argument("--leg-nxy", type=int, default=512)
    ap.add_argument("--leg-nz", type=int, default=12)
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"],
                    help="N>1 halo exchange: fused into the kernels (peer) or NCCL send/recv")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
