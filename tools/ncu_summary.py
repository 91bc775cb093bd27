"""Summarise an ncu report (.ncu-rep) into plain text for profiles/.

Usage: python tools/ncu_summary.py <report.ncu-rep> [--top 25] > profiles/<name>.txt
Prints the kernel, launch/occupancy figures, DRAM traffic, pipe usage and
the source lines with the most warp-stall samples (needs -lineinfo and
--import-source on at capture).
"""

import argparse
import csv
import io
import subprocess
from collections import defaultdict

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
       "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_local_ld.sum",
       "sm__cycles_elapsed.avg.per_second"]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    raw = list(csv.reader(io.StringIO(ncu([a.report, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name}")
        for k in RAW:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {row[i]:>20s} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu([a.report, "--page", "source", "--csv", "--print-source=cuda,sass"]))))
    fp = None
    res = []
    ins = []
    hdr = None
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            fp = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "Function Name":
            continue
        if len(r) > 4 and r[2] == "-" and r[0].isdigit() and r[4].isdigit():
            res.append((int(r[4]), fp, int(r[0]), r[1].strip()[:90]))
            if hdr and "Instructions Executed" in hdr:
                v = r[hdr.index("Instructions Executed")].replace(",", "")
                try:
                    ins.append((float(v), fp, int(r[0]), r[1].strip()[:90]))
                except ValueError:
                    pass
    tot = sum(x[0] for x in res) or 1
    per_file = defaultdict(int)
    for s, f, _, _ in res:
        per_file[f] += s
    print("\nwarp-stall samples by file:", {k: f"{100 * v / tot:.1f}%" for k, v in sorted(per_file.items(), key=lambda x: -x[1])})
    print(f"\ntop {a.top} source lines by warp-stall samples:")
    for s, f, ln, text in sorted(res, reverse=True)[: a.top]:
        print(f"  {100 * s / tot:5.1f}%  {f}:{ln}  {text}")
    if ins:
        itot = sum(x[0] for x in ins) or 1
        print(f"\ntop {a.top} source lines by warp instructions executed (total {itot:.3g}):")
        for s, f, ln, text in sorted(ins, reverse=True)[: a.top]:
            print(f"  {100 * s / itot:5.1f}%  {f}:{ln}  {text}")


if __name__ == "__main__":
    main()
