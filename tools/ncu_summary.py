"""Summarise an ncu --set full report: duration, DRAM traffic, occupancy,
issue activity and the top warp-stall reasons.
    python tools/ncu_summary.py gpurun_out/full_x.ncu-rep [launch_index]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head, units, vals = rows[0], rows[1], rows[2 + idx]
m = dict(zip(head, vals))
u = dict(zip(head, units))
print(m.get("Kernel Name", "?")[:100], "grid", m.get("launch__grid_size"), "block", m.get("launch__block_size"))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
          "lts__t_sectors_srcunit_tex_aperture_sysmem.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
          "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]:
    if k in m:
        print(f"  {k:70s} {m[k]:>14s} {u[k]}")
st = [(k, float(v)) for k, v in m.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
      and v.replace('.', '', 1).isdigit()]
tot = sum(v for _, v in st) or 1
print("  stall samples:")
for k, v in sorted(st, key=lambda x: -x[1])[:8]:
    print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * v / tot:5.1f} %")
