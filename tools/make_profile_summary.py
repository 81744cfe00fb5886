"""Write profiles/ncu_summary_r<NN>.json (+ .md) from an ncu full capture of the
dominant kernel and the launch list of the same bench command."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
from ncu_summary import raw, source  # noqa: E402


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            hdr, start = r, i + 1
            break
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[start:]:
        if len(r) > vi:
            d[r[ki]].append(float(r[vi].replace(",", "")))
    return {k: {"launches": len(v), "mean_ns": sum(v) / len(v)} for k, v in d.items()}


def main(rnd, rep, launch_csv):
    R = raw(rep)[0]
    S = source(rep)
    val = lambda k: float(R[k].split()[0])
    unit = lambda k: R[k].split()[1]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd = val("dram__bytes_read.sum") * scale[unit("dram__bytes_read.sum")]
    wr = val("dram__bytes_write.sum") * scale[unit("dram__bytes_write.sum")]
    n, nb = 8388608, 32
    alg = n * (13 * 20 + 5 * 16 * nb)
    L = launches(launch_csv)
    step_kernels = {k: v for k, v in L.items()
                    if "sell_b4_kernel<3" in k or "sell_b4_staged_kernel<3" in k or "reduce_moments" in k}
    out = {
        "round": rnd,
        "command": "ncu --set full --clock-control none --import-source on -k regex:sell_b4_ -s 5 -c 1 "
                   "python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline",
        "kernel": R["kernel"],
        "workload": "cfg2 topi 4x128^3, n_b=32, one fused chebfd_op step (M_CHEB)",
        "duration_ms_ncu": val("gpu__time_duration.sum"),
        "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": (rd + wr) / alg,
        "metrics": R, "source_opcodes_pct_inst_pct_stall": S["opcodes"], "top_stall_lines": S["top_stall_lines"],
        "launch_list": L,
        "step_share": {k: v["mean_ns"] / sum(x["mean_ns"] for x in step_kernels.values())
                       for k, v in step_kernels.items()},
    }
    (ROOT / "profiles" / f"ncu_summary_r{rnd:02d}.json").write_text(json.dumps(out, indent=1))
    md = [f"# ncu summary, round {rnd}", "", f"Command: `{out['command']}`", "",
          f"Kernel: `{out['kernel']}` ({out['workload']})", "",
          "| metric | value |", "|---|---|"]
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
              "sm__cycles_elapsed.avg.per_second"]:
        if k in R:
            md.append(f"| `{k}` | {R[k]} |")
    md += ["", f"DRAM traffic per launch: {(rd + wr) / 1e9:.2f} GB vs algorithmic {alg / 1e9:.2f} GB "
               f"(x{(rd + wr) / alg:.3f}).", "", "Launch list (cold-cache, serialised; compare shares):", "",
           "| kernel | launches | mean µs |", "|---|---|---|"]
    for k, v in L.items():
        md.append(f"| `{k[:70]}` | {v['launches']} | {v['mean_ns'] / 1e3:.1f} |")
    md += ["", "Share of the fused step: " + ", ".join(f"`{k[:40]}` {s * 100:.2f}%" for k, s in
                                                      out["step_share"].items()), "",
           "Opcode mix (% instructions, % stall samples): " + json.dumps(S["opcodes"])]
    (ROOT / "profiles" / f"ncu_summary_r{rnd:02d}.md").write_text("\n".join(md) + "\n")
    print(json.dumps({k: out[k] for k in ["duration_ms_ncu", "dram_bytes_per_launch", "traffic_over_algorithmic",
                                          "step_share"]}, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2], sys.argv[3])
