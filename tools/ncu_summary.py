"""Summarise an ncu report: key metrics per kernel, opcode mix, top stall sites.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--sass] > profiles/x.txt
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

METRICS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__shared_mem_per_block_static", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_global_ld.sum",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        rec = dict(zip(hdr, row))
        print("=" * 100)
        print(rec.get("Kernel Name", "?")[:160])
        for m in METRICS:
            if m in rec:
                print(f"  {m:70s} {rec[m]:>14s} {units[hdr.index(m)]}")
    if "--sass" in sys.argv:
        src = run([rep, "--page", "source", "--csv", "--print-source", "sass"])
        blocks = src.split('"Kernel Name"')
        for blk in blocks[1:]:
            lines = list(csv.reader(io.StringIO('"Kernel Name"' + blk)))
            name = lines[0][1][:100]
            h = lines[1]
            data = lines[2:]
            i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
            ts = sum(float(r[i_s] or 0) for r in data) or 1.0
            te = sum(float(r[i_e] or 0) for r in data) or 1.0
            c, cs = Counter(), Counter()
            for r in data:
                toks = r[i_src].split()
                if not toks:
                    continue
                op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
                op = op.split(".")[0]
                c[op] += float(r[i_e] or 0)
                cs[op] += float(r[i_s] or 0)
            print("-" * 100)
            print(name, f"  instructions {te:.3e}")
            for op, v in c.most_common(12):
                print(f"  {op:10s} inst {v / te * 100:5.1f}%   stall-samples {cs[op] / ts * 100:5.1f}%")
            for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:10]:
                print(f"  {float(r[i_s]) / ts * 100:5.1f}%  {r[i_src][:90]}")


if __name__ == "__main__":
    main()
