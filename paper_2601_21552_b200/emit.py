"""Native constraint-set construction for the analyzer path (SURVEY.md 8(f)
rank 1).

The reference analyzer builds every solver query with `_SetBuilder`
(/root/reference/pkg/src/scuba_mini/constraint_gen.py:84-217), creating one
frozen-dataclass object per term node in interpreted Python -- about 60 us per
query, 40% of an analysis pass once the solver is on the GPU.  `csrc/
emit_native.cpp` performs the same walk through the CPython API and creates
the SAME objects (the reference's own `SolverVar` / `Constraint` / `Lit` /
`VarRef` / `BinE` / `ConstraintSet` classes, fields set as their frozen
`__init__` sets them), so everything downstream -- the analyzer's
`_check_launch`, its result objects, `render_constraint_set`, the solver shim
-- sees sets equal to the reference's, field for field.

`NativeEmission(analyzer_module)` provides drop-ins for the two generators the
analyzer binds by name (analyzer.py:18-25, called at :160 and :188):

    constraint_sets_for_access(module, kernel, ksum, host_summary, launch,
                               access, max_domain, bound, check_underflow=True)
    layout_check_sets(module, kernel, ksum, host_summary, launch, max_domain)

Extent resolution (`target_size_et`, partition sizes) stays the reference's
own code; unknown-leaf naming calls the reference's `_SetBuilder._unknown_name`.
`native_emission(analyzer_module)` binds them for the duration of a block;
`analyzer.analyze_batched` / `analyze_many` use it by default.
"""
from __future__ import annotations

import contextlib
import importlib
import sys


def _native():
    try:
        from . import _emit_native
    except ImportError as e:  # pragma: no cover - build problem
        raise ImportError("paper_2601_21552_b200/_emit_native is not built; run "
                          "`make -C paper_2601_21552_b200/csrc`") from e
    return _emit_native


class _Namer:
    """The `self` the reference's `_SetBuilder._unknown_name` reads (only
    `self.module`)."""

    __slots__ = ("module",)

    def __init__(self, module):
        self.module = module


class NativeEmission:
    def __init__(self, analyzer_module):
        pkg = analyzer_module.__name__.rsplit(".", 1)[0]
        self.cg = cg = sys.modules.get(pkg + ".constraint_gen") or importlib.import_module(pkg + ".constraint_gen")
        self.native = _native()
        self._static = (cg.Lit, cg.VarRef, cg.BinE, cg.Constraint, cg.SolverVar, cg.ConstraintSet,
                        cg.AnalysisError, cg.Const, cg.Unknown, cg.Builtin, cg.LoopVar, cg.BinOp,
                        tuple(cg.COMPARISON_OPS), tuple(cg.ARITH_OPS), dict(cg._ET_REL_TO_SOLVER),
                        tuple(cg.ALL_AXES), tuple(cg.GRID_AXES))
        self._ctx = {}  # (id(module), max_domain) -> (module, ctx tuple)
        self._refs, self._lits = {}, {}  # shared frozen leaves (VarRef by name, Lit by int value)

    def ctx(self, module, max_domain):
        key = (id(module), max_domain)
        hit = self._ctx.get(key)
        if hit is not None and hit[0] is module:
            return hit[1]
        namer = _Namer(module)
        unknown_name = self.cg._SetBuilder._unknown_name.__get__(namer)
        ctx = self._static + (unknown_name, module.defs, max_domain, {}, self._refs, self._lits)
        if len(self._ctx) > 256:
            self._ctx.clear()
        if len(self._refs) + len(self._lits) > 1 << 16:
            self._refs.clear()
            self._lits.clear()
        self._ctx[key] = (module, ctx)
        return ctx

    def constraint_sets_for_access(self, module, kernel, ksum, host_summary, launch, access, max_domain, bound,
                                   check_underflow=True):
        cg = self.cg
        size_et = cg.target_size_et(access, kernel, ksum, launch, bound)
        if size_et is None:
            return cg.AccessSets(access, launch, size_unknown=True)
        result = cg.AccessSets(access, launch, size_unknown=False)
        ctx = self.ctx(module, max_domain)
        checks = ("upper", "lower") if check_underflow else ("upper",)
        for check in checks:
            result.sets.append(self.native.access_set(
                ctx, kernel, ksum, host_summary, launch, access.offset_et, size_et, access.path_guards, check,
                cg.OFFSET_VAR, cg.SIZE_VAR, -max_domain))
        return result

    def layout_check_sets(self, module, kernel, ksum, host_summary, launch, max_domain):
        cg = self.cg
        ctx = self.ctx(module, max_domain)
        checks = []
        for base, records in ksum.partitions.items():
            for earlier, later in zip(records, records[1:]):
                cset = self.native.layout_set(ctx, kernel, ksum, host_summary, launch, later.offset_et,
                                              earlier.offset_et, "layout", [])
                checks.append(cg.LayoutCheck(base, earlier, later, cset))
        return checks


@contextlib.contextmanager
def native_emission(analyzer_module):
    """Bind the native generators into `analyzer_module` for a block."""
    em = NativeEmission(analyzer_module)
    saved = (analyzer_module.constraint_sets_for_access, analyzer_module.layout_check_sets)
    analyzer_module.constraint_sets_for_access = em.constraint_sets_for_access
    analyzer_module.layout_check_sets = em.layout_check_sets
    try:
        yield em
    finally:
        analyzer_module.constraint_sets_for_access, analyzer_module.layout_check_sets = saved
