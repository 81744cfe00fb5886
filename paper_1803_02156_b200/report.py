"""The bench-kernel report row (proj/tools/chebfilter.cpp:31-67, 275-325).

`ReportRow` carries the fixed columns `run_id,n,n_s,n_b,n_p,workers,mode,
wall_seconds,flops,flop_rate,model_p_star` (:31-43); `rows_to_csv` writes them
with the shortest round-trip decimal of every double (`fmt_double`, :25-29:
std::to_chars without a format), `rows_to_json` the way the CLI's JSON
library dumps them (`json::dump(2)`, :45-57, 87-89), `emit_report` to stdout
or a file (:69-91).  `bench_kernel` is the CLI's bench-kernel command
(:275-325) on the device: topi lattice, Gershgorin map with margin 0.01,
window [lo + 0.45 span, lo + 0.55 span], InitSeededRandom X, then
`apply_filter` (one GPU) or `filter_distributed` (workers > 1) timed, with
flops = flop_count(geometry, n_p - 2) * n_s / n_b and the model's P*.

The JSON library of the CLI (nlohmann::json, vendored by the reference under
the git-ignored proj/vendor/, absent here) serialises objects with sorted keys,
2-space indentation, integers as integers and doubles through its Grisu2
`to_chars` + `format_buffer` (fixed notation for decimal point positions
-4 < n <= 15, a trailing ".0" on integral values, exponent with >= 2 digits);
`_json_double` restates that.
"""
from __future__ import annotations

import json
import math
import sys
import time
from dataclasses import dataclass

REPORT_COLUMNS = "run_id,n,n_s,n_b,n_p,workers,mode,wall_seconds,flops,flop_rate,model_p_star"


def _shortest(v: float) -> tuple[str, int]:
    """Shortest round-trip decimal digits d and exponent e with |v| = d * 10**e."""
    r = repr(abs(v))
    mant, _, exp = r.partition("e")
    e = int(exp) if exp else 0
    ip, _, fp = mant.partition(".")
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0") or "0"
    e -= len(fp)
    stripped = digits.rstrip("0")
    e += len(digits) - len(stripped)
    return stripped or "0", e


def fmt_double(v: float) -> str:
    """std::to_chars(first, last, v) (chebfilter.cpp:25-29): the shortest round-trip
    representation, fixed or scientific whichever has fewer characters (fixed on ties)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0:
        return sign + "0"
    d, e = _shortest(v)
    k = len(d)
    # fixed (an integral value prints its exact integer, as printf("%.0f") does)
    if e >= 0:
        fixed = str(int(abs(v)))
    elif -e < k:
        fixed = d[:k + e] + "." + d[k + e:]
    else:
        fixed = "0." + "0" * (-e - k) + d
    # scientific, printf %e style exponent (sign, at least two digits)
    x = e + k - 1
    sci = d[0] + ("." + d[1:] if k > 1 else "") + "e" + ("-" if x < 0 else "+") + f"{abs(x):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def _json_double(v: float) -> str:
    """nlohmann::json's double serialisation (Grisu2 digits + format_buffer with
    min_exp = -4, max_exp = 15); non-finite values are written as null."""
    if not math.isfinite(v):
        return "null"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0:
        return sign + "0.0"
    d, e = _shortest(v)
    k = len(d)
    n = k + e
    if k <= n <= 15:
        s = d + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = d[:n] + "." + d[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + d
    else:
        x = n - 1
        s = d[0] + ("." + d[1:] if k > 1 else "") + "e" + ("-" if x < 0 else "+") + f"{abs(x):02d}"
    return sign + s


@dataclass
class ReportRow:
    """chebfilter.cpp:31-39."""
    run_id: str = ""
    n: int = 0
    n_s: int = 0
    n_b: int = 0
    n_p: int = 0
    workers: int = 1
    mode: str = "serial"
    wall_seconds: float = 0.0
    flops: float = 0.0
    flop_rate: float = 0.0
    model_p_star: float = 0.0


_INT_FIELDS = ("n", "n_s", "n_b", "n_p", "workers")
_DBL_FIELDS = ("wall_seconds", "flops", "flop_rate", "model_p_star")


def rows_to_csv(rows) -> str:
    """chebfilter.cpp:59-67."""
    out = [REPORT_COLUMNS + "\n"]
    for r in rows:
        out.append(",".join([r.run_id] + [str(int(getattr(r, f))) for f in _INT_FIELDS] + [r.mode]
                            + [fmt_double(float(getattr(r, f))) for f in _DBL_FIELDS]) + "\n")
    return "".join(out)


def _json_value(v, indent: int, level: int) -> str:
    pad, inner = " " * (indent * level), " " * (indent * (level + 1))
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f"{inner}{json.dumps(k)}: {_json_value(v[k], indent, level + 1)}" for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, list):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(inner + _json_value(x, indent, level + 1) for x in v) + "\n" + pad + "]"
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        return _json_double(v)
    return json.dumps(v, ensure_ascii=False)


def row_to_dict(r: ReportRow) -> dict:
    """chebfilter.cpp:45-57 (integers stay integers, doubles stay doubles)."""
    d = {"run_id": r.run_id, "mode": r.mode}
    d.update({f: int(getattr(r, f)) for f in _INT_FIELDS})
    d.update({f: float(getattr(r, f)) for f in _DBL_FIELDS})
    return d


def rows_to_json(rows) -> str:
    """`arr.dump(2) + "\\n"` of the rows (chebfilter.cpp:86-89)."""
    return _json_value([row_to_dict(r) for r in rows], 2, 0) + "\n"


def emit_text(text: str, out_path: str = "") -> None:
    """chebfilter.cpp:69-78: stdout for "" or "-", else the file (RuntimeError when it cannot be written)."""
    if not out_path or out_path == "-":
        sys.stdout.write(text)
        sys.stdout.flush()
        return
    try:
        with open(out_path, "w") as f:
            f.write(text)
    except OSError:
        raise RuntimeError("cannot open output path " + out_path) from None


def emit_report(rows, fmt: str = "json", out_path: str = "") -> None:
    """chebfilter.cpp:80-91: "csv" writes the CSV, anything else the JSON array."""
    emit_text(rows_to_csv(rows) if fmt == "csv" else rows_to_json(rows), out_path)


def bench_kernel(nx: int, ny: int, nz: int, ns: int = 32, nb: int = 32, np_: int = 500, workers: int = 1,
                 mode: str = "vector", seed: int = 42, mass: float = 1.0, hop: float = 1.0,
                 boundary: str = "periodic", bandwidth: float = 540e9, pmax: float = 1e12,
                 device: int = 0, devices=None) -> ReportRow:
    """The bench-kernel command (chebfilter.cpp:275-325) on the device.  The timed
    region is the filter only (apply_filter, or filter_distributed over `workers`
    shards placed on `devices`, default all on `device`), as in the CLI."""
    import torch

    from .dist import CommMode, filter_distributed_native, partition_rows, shard_and_distribute
    from .blockvec import BlockVector, InitSeededRandom
    from .filter import apply_filter, filter_coefficients, spectral_map
    from .perf_model import KernelGeometry, arithmetic_intensity, flop_count, roofline_limit
    from .sparse import Boundary, LatticeSpec, gershgorin_bounds, topi_generate

    if ns == 0 or nb == 0 or ns % nb != 0:
        raise ValueError("n_b must divide n_s")
    if nx < 1 or ny < 1 or nz < 1:
        raise ValueError("lattice extents must be positive")
    if boundary not in ("periodic", "open"):
        raise ValueError("boundary must be periodic or open")
    spec = LatticeSpec(nx, ny, nz, mass, hop, Boundary.periodic if boundary == "periodic" else Boundary.open)
    H = topi_generate(spec)
    if workers > spec.sites():
        raise ValueError("more workers than lattice sites")
    lo, hi = gershgorin_bounds(H)
    fmap = spectral_map(lo, hi, 0.01)
    span = hi - lo
    fc = filter_coefficients(lo + 0.45 * span, lo + 0.55 * span, fmap, np_)
    dev = torch.device("cuda", device)
    X = BlockVector(H.n, ns, nb, InitSeededRandom(seed), device=dev)
    if workers <= 1:
        H.device_matrix(device)  # upload outside the timed region, as the CLI builds H before its clock
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        apply_filter(H, X, fc)
        torch.cuda.synchronize(dev)
        secs = time.perf_counter() - t0
    else:
        plan = partition_rows(H, workers)
        shards = shard_and_distribute(H, X, plan, devices=devices)
        for sh in shards:
            sh.local.device_matrix(sh.X.device.index)
        for d in {sh.X.device for sh in shards}:
            torch.cuda.synchronize(d)
        t0 = time.perf_counter()
        filter_distributed_native(shards, fc, CommMode.pipelined if mode == "pipelined" else CommMode.vector)
        for d in {sh.X.device for sh in shards}:
            torch.cuda.synchronize(d)
        secs = time.perf_counter() - t0
    g = KernelGeometry(n=H.n, n_nzr=H.avg_nnz_per_row(), n_b=nb)
    total = flop_count(g, np_ - 2) * (ns // nb)
    return ReportRow(run_id="bench-kernel", n=H.n, n_s=ns, n_b=nb, n_p=np_, workers=workers,
                     mode="serial" if workers <= 1 else mode, wall_seconds=secs, flops=total,
                     flop_rate=total / secs if secs > 0 else 0.0,
                     model_p_star=roofline_limit(pmax, bandwidth, arithmetic_intensity(g)).p_star)


def main(argv=None) -> int:
    """`python -m paper_1803_02156_b200.report bench-kernel ...` (chebfilter.cpp:122-186, 275-325)."""
    import argparse
    ap = argparse.ArgumentParser(prog="paper_1803_02156_b200.report")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench-kernel")
    for k, v in (("nx", 4), ("ny", 4), ("nz", 4), ("ns", 16), ("nb", 4), ("np", 200), ("workers", 1),
                 ("seed", 42)):  # chebfilter.cpp:128-134
        b.add_argument("--" + k, type=int, default=v)
    b.add_argument("--mass", type=float, default=1.0)
    b.add_argument("--hop", type=float, default=1.0)
    b.add_argument("--boundary", default="periodic")
    b.add_argument("--mode", default="vector", choices=["vector", "pipelined"])
    b.add_argument("--bandwidth", type=float, default=540e9)
    b.add_argument("--pmax", type=float, default=1e12)
    b.add_argument("--emit", default="json", choices=["json", "csv"])
    b.add_argument("--out", default="")
    a = ap.parse_args(argv)
    try:
        row = bench_kernel(a.nx, a.ny, a.nz, a.ns, a.nb, a.np, a.workers, a.mode, a.seed, a.mass, a.hop,
                           a.boundary, a.bandwidth, a.pmax)
        emit_report([row], a.emit, a.out)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except Exception as e:  # noqa: BLE001  (the CLI's internal-error exit)
        print(f"internal error: {e}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
