"""Benchmark of the OOB-query decision engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c4|c5s] [--queries Q]

One STEP = deciding one batch of Q synthetic analyzer-shaped queries (default
config C3: 100K queries, M = 2^31-1, input caps 2^3..2^7, 30% buggy, seed
2601215521) with verdicts and first models identical to the
reference solver.  Under torchrun each rank decides its own Q-query slice of
the stream on its own GPU (weak scaling, no data-path collective: queries are
independent).

  value   queries/s with the compiled records resident in HBM: K launches of
          the decision kernel(s), timed with CUDA events on the engine stream
          (oob_plan_run), L2 flushed between steps, max over ranks.
  e2e     queries/s through the public C-ABI call oob_solve_batch on host
          buffers: host compile + H2D + kernels + D2H + scatter, every step.
  corpus  the 110 solver queries of the reference's 20-program corpus decided
          in one batch (wall time, verdicts vs the golden capture).
  cpu_baseline / --impl reference
          the C restatement of the reference solver (oracle/, kind "port") on
          the host cores, on a bounded sample of the same stream (N=1 only),
          with verdict / node / pass / model-word parity on that sample.
  witness_replay
          every Sat model of the e2e step checked by the restated reference
          evaluator (check_model over constraints + divisor side constraints).
  roofline / roofline.issue
          HBM (contract form: algorithmic bytes / kernel time vs the measured
          copy bandwidth, ncu DRAM bytes as `traffic`) and the integer-issue
          roofline (ncu warp instructions per step / live step time vs the SM
          issue peak), from the committed profiles/ncu_summary.json.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

# the engine runs several kernels per device concurrently; more hardware work
# queues than the default 8 (must be set before any CUDA context exists)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "oob_queries_decided_per_s"
UNIT = "queries/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
HBM_FALLBACK = 6650.0
WORKLOADS = {
    "c3": "C3: analyzer-shaped synthetic queries, 32-bit offsets (M=2^31-1), input caps "
          "2^3..2^7, 30% buggy, templates T1-T7, seed 2601215521",
    "c4": "C4: mixed 32/64-bit (M in {2^31-1, 2^59}), caps 2^3..2^10, templates T1-T8, "
          "seed 2601215522",
    "c5s": "C5 regenerated at caps 2^6 (bug-free, Unsat by construction), seed 2601215523",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="c3", choices=tuple(WORKLOADS))
    ap.add_argument("--queries", type=int, default=100_000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU time of the bounded cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ----- distributed plumbing ---------------------------------------------------

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Dist:
    def __init__(self, world, local, backend="nccl"):
        self.world = world
        self.pg = None
        if world > 1:
            import torch
            import torch.distributed as td
            if backend == "nccl":
                torch.cuda.set_device(local)
            td.init_process_group(backend=backend)
            self.td = td
            self.torch = torch
            self.dev = f"cuda:{local}" if backend == "nccl" else "cpu"

    def barrier(self):
        if self.world > 1:
            self.td.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.td.destroy_process_group()


# ----- clocks during the timed region ------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[3:7]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(self.samples), "reasons": reasons}


def flush_l2(torch_mod, device):
    buf = flush_l2.buf.get(device)
    if buf is None:
        buf = torch_mod.empty(64 * 1024 * 1024, dtype=torch_mod.float32, device=device)  # 256 MiB > L2
        flush_l2.buf[device] = buf
    buf.fill_(1.0)


flush_l2.buf = {}


# ----- CPU baseline (oracle port; test-infrastructure restatement) ----------------

def cpu_baseline(fb_all, target_s: float, threads: int):
    """Bounded sample of the same stream on the host cores via the C oracle."""
    from oracle import oracle
    from paper_2601_21552_b200.wire import FlatBatch  # noqa: F401
    probe = min(fb_all.n, 2000)
    t0 = time.perf_counter()
    oracle.solve_flat(fb_all.slice(0, probe), 30.0, threads=threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    n = int(min(fb_all.n, max(probe, probe * target_s / dt)))
    sample = fb_all.slice(0, n)
    t0 = time.perf_counter()
    out = oracle.solve_flat(sample, 30.0, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": round(n / dt, 1), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {n} queries of the same stream ({dt:.1f} s on {threads} threads; "
                      "oracle/oob_oracle.c restatement of solver.py)"}, out, n


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def load_peak_hbm():
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def ncu_alu(config: str):
    """Issue / ALU-pipe utilisation of the dominant kernel from the committed
    ncu --set full summary (profiles/ncu_summary.json), or None."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
        return d.get(config, {}).get("alu_evidence")
    except Exception:
        return None


def alu_roofline(config: str, launch_ms: float, sms: int = 148):
    """Integer-pipe roofline of the decision kernels: warp instructions of one
    step (ncu smsp__inst_executed.sum over all launches, committed in
    profiles/ncu_summary.json) / the live device time of a step, against the
    SM issue peak (4 schedulers x 1 warp-instruction/clock x sm_max_mhz x
    SMs), next to the measured LOP3 peak (tools/alu_peak.cu,
    profiles/alu_peak.jsonl)."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text()).get(config, {})
        inst = float(d["warp_inst_per_step"])
    except Exception:
        return None
    try:
        mhz = float(json.loads(PEAKS.read_text())["sm_max_mhz"])
    except Exception:
        mhz = 1965.0
    peak = sms * 4 * mhz * 1e6
    lop3 = None
    try:
        for line in (ROOT / "profiles" / "alu_peak.jsonl").read_text().splitlines():
            r = json.loads(line)
            if r["kind"] == "lop3":
                lop3 = r["warp_inst_per_s"]
    except Exception:
        pass
    achieved = inst / (launch_ms / 1e3)
    return {"bound": "issue (integer ALU / latency)", "unit": "warp-inst/s",
            "warp_inst_per_step": inst, "achieved": round(achieved, 1), "issue_peak": peak,
            "frac": round(achieved / peak, 4), "lop3_peak_measured": lop3}


def ncu_traffic(config: str):
    """DRAM bytes of one step (all launches of one plan run) from the
    committed ncu launch-list summary (profiles/ncu_summary.json), or None."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())
        return d.get(config, {}).get("dram_bytes_per_step")
    except Exception:
        return None


# ----- arms -------------------------------------------------------------------------

def run_reference(args, rank, world):
    """--impl reference: the CPU restatement of the reference solver (port) on
    all host threads; rank 0 only."""
    if rank != 0:
        return
    from paper_2601_21552_b200 import synth
    threads = host_threads()
    fb = synth.generate(args.config, args.queries, first=0, names=False)
    per_step = []
    for i in range(args.warmup + args.steps):
        target = args.cpu_seconds / max(args.steps, 1)
        res, _, n = cpu_baseline(fb, max(target, 2.0), threads)
        if i >= args.warmup:
            per_step.append(res["value"])
    value = statistics.median(per_step)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * args.queries / value, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOADS[args.config], "queries_per_gpu": args.queries},
        "cpu_baseline": {**res, "value": value},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch

    from paper_2601_21552_b200 import _lib, synth
    from paper_2601_21552_b200.solver import solve_flat
    from paper_2601_21552_b200.wire import flatten

    ndev = _lib.device_count()
    if ndev < 1:
        raise SystemExit("bench.py needs a CUDA device (the engine has no CPU path)")
    # one rank per GPU over NCCL; with fewer GPUs than ranks (a test of the
    # multi-rank path on a small box) ranks share devices and the barrier /
    # max-over-ranks reductions run over gloo
    dist = Dist(world, local % ndev, backend="nccl" if ndev >= world else "gloo")
    device = local % ndev
    Q = args.queries
    fb = synth.generate(args.config, Q, first=rank * Q, names=False)

    # ---- value: kernels on HBM-resident records --------------------------------
    plan = _lib.Plan(fb, 30.0, n_gpus=1, device=device)
    info = plan.info()
    torch.cuda.set_device(device)
    for _ in range(args.warmup):
        plan.run()
    kernel_ms = []
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(device) as clocks:
        for _ in range(args.steps):
            flush_l2(torch, device)
            torch.cuda.synchronize()
            kernel_ms.append(plan.run())
        torch.cuda.synchronize()
    dist.barrier()
    total_ms = dist.max(sum(kernel_ms))
    res = plan.results()
    if res["status"] != _lib.OOB_OK:
        raise SystemExit(f"engine could not decide the batch: {_lib.last_error()}")
    info = plan.info()  # result bytes of a fetched run (Sat models packed on the device)
    plan.close()  # its device pools are freed before the e2e leg allocates its own
    value = dist.sum(Q) * args.steps / (total_ms / 1e3)

    # ---- e2e: the public C-ABI call on host buffers ------------------------------
    solve_flat(fb, 30.0, n_gpus=1, device=device)  # warm
    e2e_s = []
    dist.barrier()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out = solve_flat(fb, 30.0, n_gpus=1, device=device)
        e2e_s.append(time.perf_counter() - t0)
    dist.barrier()
    e2e_total = dist.max(sum(e2e_s))
    e2e_value = dist.sum(Q) * args.steps / e2e_total
    assert np.array_equal(out["verdict"], res["verdict"]), "plan and solve_batch disagree"
    assert np.array_equal(out["nodes"], res["nodes"])

    # ---- corpus (config C2: the reference's 20 programs, 110 queries) -------------
    corpus = None
    if rank == 0:
        recs = [json.loads(l) for l in open(ROOT / "tests/golden/corpus_m1048576.jsonl")]
        cfb = flatten(recs)
        solve_flat(cfb, 30.0, n_gpus=1, device=device)
        walls = []
        for _ in range(5):
            t0 = time.perf_counter()
            cout = solve_flat(cfb, 30.0, n_gpus=1, device=device)
            walls.append(time.perf_counter() - t0)
        want = np.array([{"unsat": 0, "sat": 1}[r["verdict"]] for r in recs])
        corpus = {"queries": len(recs), "wall_ms_best": round(1e3 * min(walls), 3),
                  "wall_ms_median": round(1e3 * statistics.median(walls), 3),
                  "verdicts_identical": bool(np.array_equal(cout["verdict"], want)),
                  "sat": int((cout["verdict"] == 1).sum()),
                  "reference_python_ms": round(sum(r["ref_ms"] for r in recs), 1)}

    # ---- CPU baseline + parity on its sample ---------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_threads()
        cpu, cres, n = cpu_baseline(fb, args.cpu_seconds, threads)
        mism = int((cres["verdict"][:n] != res["verdict"][:n]).sum())
        mism += int((cres["nodes"][:n] != res["nodes"][:n]).sum())
        mism += int((cres["passes"][:n] != res["passes"][:n]).sum())
        vend = int(fb.var_begin[n])
        model_mism = int((cres["model"][:vend] != out["model"][:vend]).any(axis=1).sum())
        cpu["parity_sample"] = {"queries": n, "verdict_node_or_pass_mismatches": mism,
                                "model_word_mismatches": model_mism}

    # ---- witness replay: every Sat model of the step through the reference's
    # evaluator (check_model over constraints + divisor side constraints,
    # solver.py:319/:345, restated in oracle/) -------------------------------------
    replay = None
    if rank == 0:
        from oracle import oracle
        ok = oracle.check_model_flat(fb, out["model"])
        sat = out["verdict"] == 1
        replay = {"sat_witnesses": int(sat.sum()),
                  "replayed_true": int((ok[sat] == 1).sum()),
                  "evaluator": "check_model(constraints + divisor_side_constraints) restated "
                               "in oracle/oob_oracle.cpp"}

    dist.close()
    if rank != 0:
        return
    peak, peak_kind = load_peak_hbm()
    launch_ms = sum(kernel_ms) / len(kernel_ms)
    alg_bytes = info["record_bytes"] + info["result_bytes"]
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    n_sat = int((res["verdict"] == 1).sum())
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded analyzer-shaped query stream, generated natively)",
        "config": {"workload": WORKLOADS[args.config], "queries_per_gpu": Q,
                   "l2": "flushed (256 MiB write) between timed steps",
                   "classes": info["classes"], "int128_regime_queries": info["wide_queries"],
                   "sat": n_sat, "unsat": int((res["verdict"] == 0).sum()),
                   "parallelism": f"dp{world} (query shards, no collective)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 5),
                     "traffic": ncu_traffic(args.config),
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "note": "interval-propagation DFS is integer-ALU/latency bound; "
                             "bytes = compiled records + results per step, all launches (DESIGN.md)",
                     "alu": ncu_alu(args.config),
                     "issue": alu_roofline(args.config, launch_ms)},
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_value, 1), "unit": UNIT,
                "h2d_bytes_per_step": info["record_bytes"],
                "d2h_bytes_per_step": info["result_bytes"]},
        "clocks": clocks.summary(),
        "gpu_launches": info["launches_per_run"] * args.steps,
        "corpus": corpus,
        "witness_replay": replay,
        "kernel_ms_per_step": [round(x, 3) for x in kernel_ms],
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if world > 1 and "SCUBA_OOB_HOST_THREADS" not in os.environ:
        # one process per GPU on one node: split the host cores between the
        # ranks' host pipelines instead of oversubscribing them
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        os.environ["SCUBA_OOB_HOST_THREADS"] = str(max(1, host_threads() // max(local_world, 1)))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
