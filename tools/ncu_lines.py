"""Aggregate an ncu source page (cuda,sass) per CUDA source line.

    python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = defaultdict(lambda: [0, 0, 0, ""])
cur_file, hdr = "?", None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].strip():  # a source line row
        cur = (cur_file, int(r[0]))
        agg[cur][3] = r[1].strip()[:70]
    try:
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = int(r[hdr.index("Instructions Executed")] or 0)
        tinst = int(r[hdr.index("Thread Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    if cur:
        a = agg[cur]
        a[0] += samp
        a[1] += inst
        a[2] += tinst
S = sum(v[0] for v in agg.values()) or 1
I = sum(v[1] for v in agg.values()) or 1
print(f"total samples {S}, warp insts {I}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    thr = v[2] / v[1] if v[1] else 0
    print(f"{100 * v[0] / S:5.1f}% smp {100 * v[1] / I:5.1f}% inst thr/inst {thr:4.1f}  {k[0]}:{k[1]:<5} {v[3]}")
