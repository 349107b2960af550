"""Summarise an ncu report (details page + selected raw counters) as text.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--raw] [--stalls]
"""
import csv
import io
import subprocess
import sys

KEEP = ("Duration", "Elapsed Cycles", "SM Frequency", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Mem Pipes Busy", "No Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Issued Instructions", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Avg. Active Threads Per Warp", "Branch Efficiency")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "sm__sass_thread_inst_executed_op_ffma_pred_on.sum")


def ncu(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu(rep, "details")
    hdr = rows[0]
    iid, iname, imet, iunit, ival = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    seen = {}
    for r in rows[1:]:
        if r[imet] in KEEP:
            key = (r[iid], r[iname].split("(")[0])
            seen.setdefault(key, []).append(f"{r[imet]}={r[ival]} {r[iunit]}".strip())
    for (i, name), vals in seen.items():
        print(f"[{i}] {name}")
        for v in vals:
            print("    " + v)
    if "--raw" in sys.argv or "--stalls" in sys.argv:
        raw = ncu(rep, "raw")
        hdr = raw[0]
        for r in raw[2:]:
            print(f"[raw {r[hdr.index('ID')]}]")
            for k, v in zip(hdr, r):
                if k in RAW or ("--stalls" in sys.argv and k.startswith("smsp__average_warp_latency_issue_stalled")
                                and k.endswith(".ratio")) or ("--stalls" in sys.argv and "warps_issue_stalled" in k and k.endswith("per_warp_active.pct")):
                    print(f"    {k} = {v}")


if __name__ == "__main__":
    main()
