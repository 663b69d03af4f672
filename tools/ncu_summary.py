"""Summarise an ncu --set full report (the metrics the roofline claims rest on)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    vals = dict(zip(h, zip(u, v)))
    stalls = sorted(((float(val.replace(",", "")), k) for k, (unit, val) in vals.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not k.endswith("not_issued")), reverse=True)
    lines = [f"# ncu --set full summary of {rep}", f"kernel: {vals.get('Kernel Name', ('', ''))[1]}"]
    for k in KEYS:
        if k in vals:
            lines.append(f"{k:70s} {vals[k][1]:>20s} {vals[k][0]}")
    tot = sum(s for s, _ in stalls) or 1
    lines.append("# warp stall samples (pc sampling), share of total")
    for s, k in stalls[:10]:
        lines.append(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * s / tot:6.2f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
