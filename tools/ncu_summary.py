"""Summarise an ncu --set full report: per kernel duration, occupancy, issue, stalls, pipes, DRAM."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
want = {
    "gpu__time_duration.sum": "dur",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu%",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu%",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active": "xu%",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem%",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "launch__registers_per_thread": "regs",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "thr/inst",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum": "ffma",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum": "fadd",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum": "fmul",
    "smsp__inst_executed.sum": "inst",
}
for row in r[2:]:
    name = row[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
    out = [name]
    for k, lab in want.items():
        if k in hdr:
            out.append(f"{lab}={row[hdr.index(k)]}{units[hdr.index(k)] if lab in ('dur','dram_rd','dram_wr') else ''}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(row[i])
            except ValueError:
                continue
            if v > 0.15:
                st.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    st.sort(reverse=True)
    out.append("stalls=" + ",".join(f"{n}:{v:.2f}" for v, n in st[:6]))
    print(" | ".join(out))
