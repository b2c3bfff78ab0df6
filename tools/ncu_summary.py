"""Summarise ncu captures into profiles/ (run in the build container).

    python tools/ncu_summary.py full  <report.ncu-rep> <out.md>
    python tools/ncu_summary.py list  <launches.csv>   <out.md>

`full` reads a `--set full` report (`ncu -i ... --page raw --csv`) and keeps the
metrics that explain this engine (time, DRAM bytes, issue / warp occupancy,
SIMT efficiency, ALU pipe utilisation, stall reasons); `list` turns a
`--metrics gpu__time_duration.sum,...` launch list into a per-kernel table.
"""
import csv
import io
import json
import re
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]
STALL = re.compile(r"smsp__pcsamp_warps_issue_stalled_(\w+)$")


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{rep.split('/')[-1]}`", ""]
    summary = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        lines += [f"## {name}", "", "| metric | value | unit |", "|---|---|---|"]
        rec = {}
        for m in KEEP:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"| {m} | {r[i]} | {units[i]} |")
                rec[m] = r[i]
        stalls = []
        for i, h in enumerate(hdr):
            mm = STALL.search(h)
            if mm and r[i] not in ("", "0"):
                try:
                    stalls.append((float(r[i]), mm.group(1)))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(s for s, _ in stalls) or 1
        lines += ["", "stall samples (share): " + ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in stalls[:6]), ""]
        summary[name] = rec
    open(out, "w").write("\n".join(lines) + "\n")
    print(json.dumps(summary, indent=1)[:2000])


def launch_list(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    table = {}
    for r in rows:
        if "oob_" not in r[4]:
            continue
        k = r[4].split("(")[0]
        table.setdefault(k, {})[r[-3]] = r[-1]
    lines = ["| kernel | " + " | ".join(sorted({m for v in table.values() for m in v})) + " |"]
    metrics = sorted({m for v in table.values() for m in v})
    lines.append("|---" * (len(metrics) + 1) + "|")
    for k, v in table.items():
        lines.append(f"| {k} | " + " | ".join(v.get(m, "") for m in metrics) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    {"full": full, "list": launch_list}[sys.argv[1]](sys.argv[2], sys.argv[3])
