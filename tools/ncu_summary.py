"""Summarise an ncu report (one launch): headline metrics of the details page,
warp-stall reasons per issued instruction, DRAM bytes and pipe utilisation.

    python tools/ncu_summary.py report.ncu-rep > summary.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "Elapsed Cycles", "SM Active Cycles", "SM Frequency", "Executed Instructions",
        "Issued Ipc Active", "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Grid Size",
        "Block Size", "Achieved Active Warps Per SM", "L2 Hit Rate", "L1/TEX Hit Rate", "DRAM Throughput",
        "Memory Throughput", "Compute (SM) Throughput", "Dynamic Shared Memory Per Block")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "sm__ops_path_tensor_src_fp64.sum", "sm__ops_path_tensor_src_fp64.sum.pct_of_peak_sustained_elapsed",
       "sm__ops_path_tensor_src_fp64.sum.per_second",
       "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    kname = None
    print(f"report: {rep}")
    for r in rows[1:]:
        d = dict(zip(h, r))
        kname = kname or d.get("Kernel Name")
        if d.get("Metric Name") in KEYS:
            print(f"  {d['Metric Name']:<40} {d['Metric Value']} {d['Metric Unit']}")
    print(f"kernel: {kname}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    names, units, vals = raw[0], raw[1], raw[2]
    print("raw:")
    for n, u, v in zip(names, units, vals):
        if n in RAW or any(n.startswith(x) for x in ("dram__bytes",)):
            print(f"  {n:<75} {v} {u}")
    print("warp stalls per issued instruction (cycles):")
    st = []
    for n, v in zip(names, vals):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            if f >= 0.01:
                st.append((f, n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    for f, n in sorted(st, reverse=True):
        print(f"  {n:<30} {f:.3f}")


if __name__ == "__main__":
    main()
