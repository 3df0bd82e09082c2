"""Summarise ncu captures into the text files committed under profiles/.

  python profiles/summarize_ncu.py full   <report.ncu-rep> <out.txt>
  python profiles/summarize_ncu.py launch <launches.csv>   <out.txt>
  python profiles/summarize_ncu.py hot    <report.ncu-rep> <out.txt>   (per-SASS hot spots)
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__sass_thread_inst_executed_op_integer_pred_on.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_op_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep, dst):
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units = rows[0], rows[1]
    with open(dst, "w") as f:
        for vals in rows[2:]:
            f.write("kernel: %s\n" % vals[hdr.index("Kernel Name")])
            for m in METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    f.write("  %-80s %s %s\n" % (m, vals[i], units[i]))
            f.write("\n")


def launch(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    with open(dst, "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
        f.write("%-90s %5s %14s %14s %7s\n" % ("kernel", "n", "total_ns", "mean_ns", "share"))
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            f.write("%-90s %5d %14.0f %14.0f %6.1f%%\n" % (k[:90], len(v), sum(v), sum(v) / len(v), 100 * sum(v) / tot))


def hot(rep, dst):
    r = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"])
    hdr, rows = r[1], r[2:]
    ie, src, at = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Avg. Threads Executed")
    tot = sum(int(x[ie]) for x in rows)
    with open(dst, "w") as f:
        f.write("%s\ntotal warp instructions executed: %d\n" % (r[0][1], tot))
        f.write("SASS lines with >= 0.1%% of executed warp instructions (idx, count, share, avg threads)\n")
        for i, x in enumerate(rows):
            c = int(x[ie])
            if c >= tot * 0.001:
                f.write("%5d %14d %5.2f%% thr=%5s  %s\n" % (i, c, 100 * c / tot, x[at], x[src].strip()[:70]))


if __name__ == "__main__":
    {"full": full, "launch": launch, "hot": hot}[sys.argv[1]](sys.argv[2], sys.argv[3])
