"""One-line-per-metric summary of ncu --set full raw CSV exports (the
profiles/ summaries are made with it).
    python tools/ncu_brief.py gpurun_out/ncu_r2b_sparse_fused_raw.csv [...]"""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "registers"), ("smsp__inst_executed.sum", "warp instructions"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %")]


def brief(path):
    rows = list(csv.reader(open(path)))
    head, units, vals = rows[0], rows[1], rows[2]
    m, u = dict(zip(head, vals)), dict(zip(head, units))
    print(m.get("Kernel Name", "?")[:110])
    for k, name in KEYS:
        if k in m:
            print(f"  {name:18s} {m[k]:>14s} {u.get(k, '')}")
    st = []
    for k, v in m.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st.append((k[len("smsp__pcsamp_warps_issue_stalled_"):], float(v)))
            except ValueError:
                pass
    tot = sum(v for _, v in st) or 1.0
    print("  stall samples: " + ", ".join(f"{k} {v / tot:.2f}" for k, v in sorted(st, key=lambda x: -x[1])[:6]))


for p in sys.argv[1:]:
    brief(p)
