"""Summarise an .ncu-rep (details page) into the metrics DESIGN.md cites."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Ipc Active", "Grid Size", "Block Size",
        "Branch Efficiency", "Mem Busy", "Max Bandwidth"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    res = {}
    for r in rows[1:]:
        res.setdefault((r[idi], r[ki]), {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for n in names:
            if n in h:
                i = h.index(n)
                d[n] = f"{r[i]} {units[i]}".strip()  # ncu picks the unit per value (byte, Kbyte, Mbyte, Gbyte)
        res.append(d)
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    for (i, k), m in details(rep).items():
        print(f"== [{i}] {k[:100]}")
        for key in KEYS:
            if key in m:
                print(f"   {key:40s} {m[key]}")
    names = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
             "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
             "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
             "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
             "smsp__thread_inst_executed_per_inst_executed.ratio", "gpu__time_duration.sum"]
    for d in raw(rep, names):
        print("   raw:", d)
