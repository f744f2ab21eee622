"""Per-CUDA-source-line warp-stall samples of an ncu report (needs -lineinfo):
    python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
cur_file = "?"
head = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        head = r
        continue
    if head is None or not r[0].isdigit():
        continue
    try:
        samp = int(r[4])
    except (ValueError, IndexError):
        continue
    key = (cur_file, int(r[0]))
    a = agg.setdefault(key, [0, r[1].strip()[:100]])
    a[0] += samp
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (smp, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * smp / tot:5.1f}%  {f}:{ln:<5} {src}")
