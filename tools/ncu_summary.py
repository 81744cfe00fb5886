"""Summarise an ncu report (raw page + source-page opcode/stall histogram)."""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__grid_size',
        'launch__block_size', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'sm__cycles_elapsed.avg.per_second',
        'launch__shared_mem_per_block_dynamic', 'sm__throughput.avg.pct_of_peak_sustained_elapsed']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {'kernel': vals[hdr.index('Kernel Name')]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


def source(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # one section per profiled kernel ("Kernel Name" line, header, rows): the first one
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    hdr = rows[starts[0] + 1]
    data = [r for r in rows[starts[0] + 2:starts[1]] if len(r) == len(hdr)]
    ia, ss, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    tot = sum(int(r[ia] or 0) for r in data)
    tots = sum(int(r[ss] or 0) for r in data) or 1
    c, s = Counter(), Counter()
    for r in data:
        toks = r[src].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
        op = op.split('.')[0]
        c[op] += int(r[ia] or 0)
        s[op] += int(r[ss] or 0)
    top = sorted(data, key=lambda r: -int(r[ss] or 0))[:12]
    return {'total_inst': tot, 'opcodes': {op: [round(v / tot * 100, 2), round(s[op] / tots * 100, 2)]
                                          for op, v in c.most_common(16)},
            'top_stall_lines': [[r[ss], r[ia], r[src].strip()[:80]] for r in top]}


if __name__ == '__main__':
    rep = sys.argv[1]
    print(json.dumps({'raw': raw(rep), 'source': source(rep)}, indent=1))
