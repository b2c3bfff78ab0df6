"""Symbolize SCUBA_OOB_PROF samples (library-relative PCs) with addr2line and
print the hottest functions / source lines (inline chains resolved)."""
import collections
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
path = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "gpurun_out/host_prof.txt")
lib = sys.argv[2] if len(sys.argv) > 2 else str(ROOT / "paper_2601_21552_b200/libscuba_oob.so")
pcs = [ln.strip() for ln in open(path) if ln.strip() and not ln.startswith("#")]
cnt = collections.Counter(pcs)
uniq = list(cnt)
out = subprocess.run(["addr2line", "-f", "-i", "-C", "-a", "-e", lib] + uniq, capture_output=True, text=True).stdout
# addr2line -a prints the address line, then (function, file:line) pairs (inline chain innermost first)
blocks, cur = {}, None
for ln in out.splitlines():
    if ln.startswith("0x"):
        cur = ln[2:].lstrip("0") or "0"
        blocks[cur] = []
    else:
        blocks[cur].append(ln)
fn_self, line_self, outer = collections.Counter(), collections.Counter(), collections.Counter()
for pc, c in cnt.items():
    b = blocks.get(pc.lstrip("0") or "0", [])
    pairs = [(b[i], b[i + 1]) for i in range(0, len(b) - 1, 2)]
    if not pairs:
        continue
    f0, l0 = pairs[0]
    f0 = f0.replace("(anonymous namespace)::", "")
    fn_self[f0.split("(")[0][:90]] += c
    line_self[l0.split("/")[-1].split(" ")[0]] += c
    outer[pairs[-1][0].replace("(anonymous namespace)::", "").split("(")[0][:90]] += c
n = len(pcs)
print(f"{n} samples in the library")
for title, C in (("innermost function", fn_self), ("outermost (non-inlined) function", outer), ("source line", line_self)):
    print(f"--- {title}")
    for k, v in C.most_common(30):
        print(f"{v:6d} {100 * v / n:5.1f}%  {k}")
