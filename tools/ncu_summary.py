"""Key counters of an ncu report (first kernel): python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = [
    ("Kernel Name", "kernel"),
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_static", "smem static"),
    ("launch__shared_mem_per_block_dynamic", "smem dynamic"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("launch__occupancy_limit_warps", "CTA limit (warps)"),
    ("launch__occupancy_limit_blocks", "CTA limit (blocks)"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__waves_per_multiprocessor", "waves/SM"),
    ("sm__inst_executed.sum.pct_of_peak_sustained_elapsed", "issue % (elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps/cycle"),
]
for k, label in keys:
    if k in d:
        print("%-24s %s %s" % (label, d[k], u.get(k, "")))
fp64 = 0.0
for op in ("dfma", "dmul", "dadd"):
    k = "smsp__sass_thread_inst_executed_op_%s_pred_on.sum" % op
    if k in d:
        fp64 += float(d[k])
if fp64:
    print("%-24s %.4g" % ("FP64 thread-ops", fp64))
print("stalls per issued instruction:")
for k in hdr:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            v = float(d[k])
        except ValueError:
            continue
        if v >= 0.05:
            print("   %-28s %.3f" % (k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], v))
