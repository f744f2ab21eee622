"""Per-source-line instruction and stall-sample totals from
`ncu -i REP --page source --csv --print-source cuda,sass --kernel-name K`.
    python tools/ncu_lines.py export.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
inst, samp, src = defaultdict(float), defaultdict(float), {}
f = "?"
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = (f, ln)
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        a, b = float(r[ie] or 0), float(r[ss] or 0)
    except ValueError:
        continue
    inst[key] += a
    samp[key] += b
    src[key] = r[1][:70]
ti, ts = sum(inst.values()), sum(samp.values())
print(f"total warp instructions {ti:.4g}, stall samples {ts:.0f}")
for k in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{k[0]}:{k[1]:<5} inst {100 * inst[k] / ti:5.1f}%  stall {100 * samp[k] / max(ts, 1):5.1f}%  {src[k]}")
