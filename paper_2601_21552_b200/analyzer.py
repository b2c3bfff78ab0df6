"""Plugging the B200 engine into the reference analyzer.

The reference analyzer binds `solve` by name (`from .solver import ... solve`,
/root/reference/pkg/src/scuba_mini/analyzer.py:32) and calls it once per
query at analyzer.py:163 (partition-layout checks) and analyzer.py:211 (access
checks).  Two integrations, both leaving the reference front end untouched:

* `install(analyzer_module)` -- replace that binding with the GPU `solve`
  (one device call per query; simplest, launch-latency bound).

* `analyze_batched(analyze, *args)` -- record/replay.  Constraint
  generation never depends on an earlier verdict (analyzer.py:160-243), so
  pass 1 runs the analysis with a recording stub that answers Unsat, ONE GPU
  batch decides every recorded query, and pass 2 re-runs the analysis
  replaying the verdicts in call order.  Diagnostics are identical to the
  reference's because verdicts and models are.  Pass 2 is skipped when every
  recorded query is decided Unsat: the analysis is deterministic, so pass 1
  -- which saw exactly those verdicts -- already is the reference's result
  (most programs: an access is reported only when a query is Sat or times
  out).

Both batched entry points also build the queries natively (`emit.py`,
SURVEY.md 8(f) rank 1): the analyzer's two constraint-set generators are
bound to `csrc/emit_native.cpp`, which creates objects equal to the
reference's `_SetBuilder` output, field for field (`native=False` keeps the
reference's Python generators).
"""
from __future__ import annotations

import contextlib

from .emit import native_emission
from .solver import solve_batch
from .terms import query_to_json


def _types(analyzer_module):
    return (analyzer_module.Sat, analyzer_module.Unsat, analyzer_module.Timeout)


def _gpu_solve(types, mode):
    # one query per call: one device (the in-call multi-device dealing is for
    # batches)
    def gpu_solve(variables, constraints, timeout_s=30.0):
        return solve_batch([(variables, constraints)], timeout_s, n_gpus=1, verdict_types=types, mode=mode)[0]

    return gpu_solve


@contextlib.contextmanager
def installed(analyzer_module, mode="canonical"):
    """Context manager: analyzer_module.solve -> the GPU engine."""
    saved = analyzer_module.solve
    gpu_solve = _gpu_solve(_types(analyzer_module), mode)
    analyzer_module.solve = gpu_solve
    try:
        yield gpu_solve
    finally:
        analyzer_module.solve = saved


def install(analyzer_module, mode="canonical"):
    """Permanently bind the GPU engine into the analyzer module."""
    gpu_solve = _gpu_solve(_types(analyzer_module), mode)
    analyzer_module.solve = gpu_solve
    return gpu_solve


class _Recorder:
    def __init__(self, unsat):
        self.calls = []
        self._unsat = unsat

    def __call__(self, variables, constraints, timeout_s=30.0):
        self.calls.append((variables, constraints, float(timeout_s)))
        return self._unsat()


def decide_calls(calls, types, **engine_kw):
    """One GPU batch per distinct timeout value; verdicts in call order."""
    verdicts = [None] * len(calls)
    by_timeout = {}
    for i, (_, _, t) in enumerate(calls):
        by_timeout.setdefault(t, []).append(i)
    for t, idx in by_timeout.items():
        vs = solve_batch([(calls[i][0], calls[i][1]) for i in idx], t,
                         verdict_types=types, **engine_kw)
        for i, v in zip(idx, vs):
            verdicts[i] = v
    return verdicts


class _Replay:
    """Pass 2: hands back the recorded verdicts in call order and checks that
    the analysis makes exactly the recorded calls."""

    def __init__(self, calls, verdicts):
        self.calls = calls
        self.verdicts = verdicts
        self.i = 0

    def __call__(self, variables, constraints, timeout_s=30.0):
        if self.i >= len(self.calls):
            raise RuntimeError("analysis is not deterministic between passes "
                               f"(pass 2 made more than the {len(self.calls)} recorded solver calls)")
        want = self.calls[self.i]
        if query_to_json(variables, constraints) != query_to_json(want[0], want[1]):
            raise RuntimeError(f"analysis is not deterministic between passes (solver call {self.i} differs)")
        v = self.verdicts[self.i]
        self.i += 1
        return v

    def finish(self):
        if self.i != len(self.calls):
            raise RuntimeError("analysis is not deterministic between passes "
                               f"(pass 2 made {self.i} of the {len(self.calls)} recorded solver calls)")


def _parse_once(analyzer_module, analyze, args, kwargs):
    """analyze_source(text, filename, config) is parse_source + analyze_program
    (analyzer.py:263-267): parse once, so a replayed pass re-runs only the
    analysis (the passes build new objects from the AST and never modify it)."""
    if analyze is not getattr(analyzer_module, "analyze_source", None):
        return analyze, args, kwargs
    import inspect

    bound = inspect.signature(analyze).bind(*args, **kwargs)
    bound.apply_defaults()
    a = bound.arguments
    program = analyzer_module.parse_source(a["text"], a["filename"])
    return analyzer_module.analyze_program, (program, a["config"]), {}


def analyze_batched(analyzer_module, analyze, *args, stats=None, mode="canonical", native=True, **kwargs):
    """Run `analyze(*args, **kwargs)` (e.g. analyzer_module.analyze_source)
    with all of its solver queries decided in one GPU batch."""
    with (native_emission(analyzer_module) if native else contextlib.nullcontext()):
        return _analyze_batched(analyzer_module, analyze, args, kwargs, stats, mode)


def _analyze_batched(analyzer_module, analyze, args, kwargs, stats, mode):
    types = _types(analyzer_module)
    analyze, args, kwargs = _parse_once(analyzer_module, analyze, args, kwargs)
    saved = analyzer_module.solve
    rec = _Recorder(types[1])
    analyzer_module.solve = rec
    try:
        first = analyze(*args, **kwargs)
    finally:
        analyzer_module.solve = saved
    verdicts = decide_calls(rec.calls, types, mode=mode)
    if stats is not None:
        stats["queries"] = len(rec.calls)
        stats["replayed"] = 0
    if all(isinstance(v, types[1]) for v in verdicts):
        return first  # pass 1 saw exactly these verdicts
    replay = _Replay(rec.calls, verdicts)
    analyzer_module.solve = replay
    try:
        result = analyze(*args, **kwargs)
    finally:
        analyzer_module.solve = saved
    replay.finish()
    if stats is not None:
        stats["replayed"] = 1
    return result


def analyze_many(analyzer_module, analyze, jobs, stats=None, mode="canonical", native=True):
    """a whole set of analyses (e.g. the 20-program
    corpus) with ALL their solver queries decided in ONE device batch.

    `jobs` is a list of (args, kwargs) for `analyze`.  Pass 1 runs every
    analysis with a recording stub, one batch decides the union of the
    recorded queries, pass 2 re-runs each analysis replaying its own slice of
    verdicts in call order.  Returns the list of results, in job order."""
    with (native_emission(analyzer_module) if native else contextlib.nullcontext()):
        return _analyze_many(analyzer_module, analyze, jobs, stats, mode)


def _analyze_many(analyzer_module, analyze, jobs, stats, mode):
    types = _types(analyzer_module)
    saved = analyzer_module.solve
    prepared = [_parse_once(analyzer_module, analyze, args, kwargs) for args, kwargs in jobs]
    recs, firsts = [], []
    try:
        for analyze, args, kwargs in prepared:
            rec = _Recorder(types[1])
            analyzer_module.solve = rec
            firsts.append(analyze(*args, **kwargs))
            recs.append(rec)
    finally:
        analyzer_module.solve = saved
    calls = [c for rec in recs for c in rec.calls]
    verdicts = decide_calls(calls, types, mode=mode)
    results = []
    base = 0
    replayed = 0
    for (analyze, args, kwargs), rec, first in zip(prepared, recs, firsts):
        mine = verdicts[base:base + len(rec.calls)]
        base += len(rec.calls)
        if all(isinstance(v, types[1]) for v in mine):
            results.append(first)  # pass 1 saw exactly these verdicts
            continue
        replay = _Replay(rec.calls, mine)
        analyzer_module.solve = replay
        try:
            results.append(analyze(*args, **kwargs))
        finally:
            analyzer_module.solve = saved
        replay.finish()
        replayed += 1
    if stats is not None:
        stats["queries"] = len(calls)
        stats["batches"] = len({c[2] for c in calls})
        stats["replayed"] = replayed
    return results
