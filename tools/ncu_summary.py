"""Summarise an ncu report: time, pipes, DRAM, occupancy, stall mix, executed FP op counts."""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__cycles_elapsed.avg.per_second", "sm clk"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__warps_active.avg.per_cycle_active", "warps/smsp"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible/smsp"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "dadd"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "dmul"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "fadd"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "fmul"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "ffma"),
]


def main(path, n=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, val = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, val))
    u = dict(zip(hdr, units))
    print("==", path)
    for k, name in KEYS:
        if k in d:
            extra = ""
            if n and name in ("dadd", "dmul", "dfma", "fadd", "fmul", "ffma"):
                extra = f"  ({float(d[k].replace(',', '')) / n:.1f} /elem)"
            print(f"  {name:14s} {d[k]:>18s} {u.get(k, '')}{extra}")
    st = [(float(v.replace(',', '')), h) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    tot = sum(v for v, _ in st) or 1
    print("  stalls:", ", ".join(f"{h.split('stalled_')[1]} {v / tot:.0%}" for v, h in sorted(st, reverse=True)[:6]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
