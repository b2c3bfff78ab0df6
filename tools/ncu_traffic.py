"""Per-step DRAM traffic and launch list of one plan run (ncu CSV) ->
profiles/ncu_summary.json (read by bench.py for roofline.traffic).

    python tools/ncu_traffic.py <cfg/mode/n> <launches.csv> [profiles/ncu_summary.json]

The key names the workload exactly (config, mode, queries per step), as
bench.py looks it up; the capture is tools/profile_kernels.py <cfg> <n> <mode>.
"""
import collections
import csv
import json
import sys
from pathlib import Path

cfg, path = sys.argv[1], sys.argv[2]
out = Path(sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_summary.json")
rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("==")) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
launch = collections.defaultdict(dict)
for r in rows:
    launch[(int(r[0]), r[4].split("(")[0])][r[-3]] = float(r[-1].replace(",", ""))
per_kernel = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0, "warp_inst": 0.0})
tot = {"ms": 0.0, "dram_bytes": 0.0, "launches": 0, "warp_inst": 0.0}
for (i, name), m in sorted(launch.items()):
    if "oob" not in name:
        continue
    ms = m.get("gpu__time_duration.sum", 0) / 1e6
    by = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    k = per_kernel[name]
    k["launches"] += 1
    k["ms"] += ms
    k["dram_bytes"] += by
    k["warp_inst"] += m.get("smsp__inst_executed.sum", 0)
    tot["warp_inst"] += m.get("smsp__inst_executed.sum", 0)
    tot["ms"] += ms
    tot["dram_bytes"] += by
    tot["launches"] += 1
dom = max(per_kernel.items(), key=lambda kv: kv[1]["ms"])
summary = json.loads(out.read_text()) if out.exists() else {}
keep = {k: v for k, v in summary.get(cfg, {}).items() if k == "alu_evidence"}
summary[cfg] = {
    "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
              f"smsp__inst_executed.sum "
              f"--clock-control none, one plan run (tools/profile_kernels.py {' '.join(cfg.split('/'))}); "
              "launches serialised and cold-cache",
    "dram_bytes_per_step": tot["dram_bytes"],
    "warp_inst_per_step": tot["warp_inst"],
    "serialised_kernel_ms_per_step": round(tot["ms"], 3),
    "launches_per_step": tot["launches"],
    "dominant_kernel": {"name": dom[0], **{k: round(v, 3) if isinstance(v, float) else v for k, v in dom[1].items()}},
    "per_kernel": {k: {kk: round(vv, 3) if isinstance(vv, float) else vv for kk, vv in v.items()}
                   for k, v in per_kernel.items()},
    **keep,
}
out.write_text(json.dumps(summary, indent=1) + "\n")
print(json.dumps(summary[cfg], indent=1)[:1500])
