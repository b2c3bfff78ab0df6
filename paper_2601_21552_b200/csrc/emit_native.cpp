// emit_native.cpp -- native constraint-set construction for the analyzer path
// (SURVEY.md 8(f) rank 1).  The reference builds every solver query in
// interpreted Python: `_SetBuilder` (constraint_gen.py:84-217) walks the
// access's expression trees and creates one frozen-dataclass object per term
// node (Lit / VarRef / BinE / Constraint / SolverVar, solver.py:32-63), about
// 1 us each through the dataclass __init__.  This module does the same walk
// through the CPython API and creates the SAME objects -- the reference's own
// classes, their fields stored exactly as the frozen __init__ stores them
// (object.__setattr__) -- so the analyzer, its result objects and the solver
// shim see values equal to the reference's, field for field.
//
// Rule for rule (constraint_gen.py):
//  * var(name, lo=0, hi=max_domain): first declaration wins, insertion order
//    is the variable order (:98-103);
//  * declare_geometry: the twelve builtins in ALL_AXES order, the six
//    `0 <= idx < dim` pairs, then one equation per GRID_AXES axis and launch
//    grid expression (:105-124);
//  * translate: Const -> Lit, Builtin -> its variable, Unknown -> its named
//    variable + witness / __input() leaves, LoopVar -> its variable plus, on
//    first sight in the set, `>= lower` and `< upper` appended BEFORE the
//    constraint being built, BinOp -> BinE (comparison or unknown operator:
//    AnalysisError) (:142-173);
//  * add_comparison drops `!=` roots (:175-184); add_context: scalar
//    parameter bindings, host asserts, kernel asserts on a dominating path
//    (path-guard prefix, list equality), then the guards (:186-208);
//  * unknown-leaf names come from the reference's own `_unknown_name`
//    (a Python callable handed in), cached per module.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

namespace {

struct Names {
    PyObject *value, *axis, *tag, *lower, *upper, *op, *left, *right, *name, *id, *kind, *operands;
    PyObject *params, *args, *is_pointer, *vid, *value_et, *asserts, *path_guards, *cond_et, *grid_ets;
    PyObject *rel, *lhs, *rhs, *lo, *hi, *ne, *ge, *lt, *eq, *input_def, *loop, *sol, *zero;
};
Names N;
PyObject* g_empty = nullptr;  // ()

bool init_names() {
#define I(f, s) N.f = PyUnicode_InternFromString(s); if (!N.f) return false;
    I(value, "value") I(axis, "axis") I(tag, "tag") I(lower, "lower") I(upper, "upper") I(op, "op")
    I(left, "left") I(right, "right") I(name, "name") I(id, "id") I(kind, "kind") I(operands, "operands")
    I(params, "params") I(args, "args") I(is_pointer, "is_pointer") I(vid, "vid") I(value_et, "value_et")
    I(asserts, "asserts") I(path_guards, "path_guards") I(cond_et, "cond_et") I(grid_ets, "grid_ets")
    I(rel, "rel") I(lhs, "lhs") I(rhs, "rhs") I(lo, "lo") I(hi, "hi") I(ne, "!=") I(ge, ">=") I(lt, "<")
    I(eq, "=") I(input_def, "InputDef") I(loop, "loop") I(sol, "sol")
#undef I
    N.zero = PyLong_FromLong(0);
    g_empty = PyTuple_New(0);
    return N.zero && g_empty;
}

// the reference's classes and constants, unpacked from the ctx tuple the
// Python side builds per (module, max_domain) (emit.py)
struct Ctx {
    PyObject *Lit, *VarRef, *BinE, *Constraint, *SolverVar, *ConstraintSet, *AnalysisError;
    PyObject *Const, *Unknown, *Builtin, *LoopVar, *BinOp;
    PyObject *comparison_ops, *arith_ops, *rel_map, *all_axes, *grid_axes;
    PyObject *unknown_name;  // tag -> (solver name, display): the reference's _SetBuilder._unknown_name
    PyObject *defs;          // module.defs
    PyObject *max_domain;
    PyObject *cache;         // dict (tag, tag.name) -> (name, display, input site or None)
    PyObject *refs, *lits;   // dicts name -> VarRef, int -> Lit: frozen values, shared (equality is by value)
};
constexpr int CTX_FIELDS = 23;

bool unpack(PyObject* t, Ctx& c) {
    if (!PyTuple_Check(t) || PyTuple_GET_SIZE(t) != CTX_FIELDS) {
        PyErr_SetString(PyExc_TypeError, "emit_native: bad context tuple");
        return false;
    }
    PyObject** f[CTX_FIELDS] = {&c.Lit, &c.VarRef, &c.BinE, &c.Constraint, &c.SolverVar, &c.ConstraintSet,
                                &c.AnalysisError, &c.Const, &c.Unknown, &c.Builtin, &c.LoopVar, &c.BinOp,
                                &c.comparison_ops, &c.arith_ops, &c.rel_map, &c.all_axes, &c.grid_axes,
                                &c.unknown_name, &c.defs, &c.max_domain, &c.cache, &c.refs, &c.lits};
    for (int i = 0; i < CTX_FIELDS; i++) *f[i] = PyTuple_GET_ITEM(t, i);
    return true;
}

// an instance of a frozen dataclass with its fields set the way its __init__
// sets them (object.__setattr__), without running the Python __init__
PyObject* make(PyObject* cls, int n, PyObject* const* keys, PyObject* const* vals) {
    PyTypeObject* tp = (PyTypeObject*)cls;
    PyObject* o = tp->tp_new(tp, g_empty, nullptr);  // object.__new__(cls)
    if (!o) return nullptr;
    for (int i = 0; i < n; i++)
        if (PyObject_GenericSetAttr(o, keys[i], vals[i]) < 0) {
            Py_DECREF(o);
            return nullptr;
        }
    return o;
}
// one instance per value of the frozen leaf classes (per context)
PyObject* cached(PyObject* cache, PyObject* cls, PyObject* field, PyObject* v) {
    PyObject* hit = PyDict_GetItemWithError(cache, v);
    if (hit) {
        Py_INCREF(hit);
        return hit;
    }
    if (PyErr_Occurred()) return nullptr;
    PyObject* k[1] = {field};
    PyObject* x[1] = {v};
    PyObject* o = make(cls, 1, k, x);
    if (o && PyDict_SetItem(cache, v, o) < 0) Py_CLEAR(o);
    return o;
}
PyObject* make_lit(const Ctx& c, PyObject* v) {
    if (PyLong_CheckExact(v)) return cached(c.lits, c.Lit, N.value, v);  // (not bool: True == 1)
    PyObject* k[1] = {N.value};
    PyObject* x[1] = {v};
    return make(c.Lit, 1, k, x);
}
PyObject* make_ref(const Ctx& c, PyObject* name) {
    if (PyUnicode_CheckExact(name)) return cached(c.refs, c.VarRef, N.name, name);
    PyObject* k[1] = {N.name};
    PyObject* x[1] = {name};
    return make(c.VarRef, 1, k, x);
}
// steals l and r (either may be null after a failure)
PyObject* make_bin(const Ctx& c, PyObject* op, PyObject* l, PyObject* r) {
    PyObject* o = nullptr;
    if (l && r) {
        PyObject* k[3] = {N.op, N.left, N.right};
        PyObject* x[3] = {op, l, r};
        o = make(c.BinE, 3, k, x);
    }
    Py_XDECREF(l);
    Py_XDECREF(r);
    return o;
}
// steals l and r
PyObject* make_con(const Ctx& c, PyObject* rel, PyObject* l, PyObject* r) {
    PyObject* o = nullptr;
    if (l && r) {
        PyObject* k[3] = {N.rel, N.lhs, N.rhs};
        PyObject* x[3] = {rel, l, r};
        o = make(c.Constraint, 3, k, x);
    }
    Py_XDECREF(l);
    Py_XDECREF(r);
    return o;
}

bool analysis_error(const Ctx& c, PyObject* msg) {  // raise AnalysisError(msg, None); steals msg
    if (!msg) return false;
    PyObject* e = PyObject_CallFunctionObjArgs(c.AnalysisError, msg, Py_None, nullptr);
    Py_DECREF(msg);
    if (e) {
        PyErr_SetObject((PyObject*)Py_TYPE(e), e);
        Py_DECREF(e);
    }
    return false;
}

struct Builder {
    const Ctx& c;
    PyObject* vars = PyDict_New();       // name -> SolverVar (insertion order = variable order)
    PyObject* cons = PyList_New(0);      // Constraint objects
    PyObject* witness = PyDict_New();    // solver name -> display name
    PyObject* inputs = PyDict_New();     // solver name -> __input() site
    PyObject* loop_seen = PySet_New(nullptr);
    explicit Builder(const Ctx& cc) : c(cc) {}
    ~Builder() {
        Py_XDECREF(vars);
        Py_XDECREF(cons);
        Py_XDECREF(witness);
        Py_XDECREF(inputs);
        Py_XDECREF(loop_seen);
    }
    bool ok() const { return vars && cons && witness && inputs && loop_seen; }

    // var(name, lo, hi): a VarRef (new reference); hi null = max_domain
    PyObject* var(PyObject* name, PyObject* lo, PyObject* hi) {
        int has = PyDict_Contains(vars, name);
        if (has < 0) return nullptr;
        if (!has) {
            PyObject* k[3] = {N.name, N.lo, N.hi};
            PyObject* x[3] = {name, lo, hi ? hi : c.max_domain};
            PyObject* sv = make(c.SolverVar, 3, k, x);
            if (!sv) return nullptr;
            int r = PyDict_SetItem(vars, name, sv);
            Py_DECREF(sv);
            if (r < 0) return nullptr;
        }
        return make_ref(c, name);
    }
    bool append(PyObject* con) {  // steals con
        if (!con) return false;
        int r = PyList_Append(cons, con);
        Py_DECREF(con);
        return r == 0;
    }
    // (name, display, input site or None) of an Unknown leaf's tag, cached per module
    PyObject* unknown(PyObject* tag) {  // borrowed (the cache holds it)
        // keyed by (tag, tag.name): ValueId equality is the numeric id only,
        // the display name also reads the name
        PyObject* tname = PyObject_GetAttr(tag, N.name);
        PyObject* key = tname ? PyTuple_Pack(2, tag, tname) : nullptr;
        Py_XDECREF(tname);
        if (!key) return nullptr;
        PyObject* hit = PyDict_GetItemWithError(c.cache, key);
        if (hit || PyErr_Occurred()) {
            Py_DECREF(key);
            return hit;
        }
        PyObject* nd = PyObject_CallOneArg(c.unknown_name, tag);
        if (!nd || !PyTuple_Check(nd) || PyTuple_GET_SIZE(nd) != 2) {
            if (nd) PyErr_SetString(PyExc_TypeError, "_unknown_name must return (name, display)");
            Py_XDECREF(nd);
            Py_DECREF(key);
            return nullptr;
        }
        PyObject* site = Py_None;
        Py_INCREF(site);
        bool okk = true;
        PyObject* st = PyObject_CallMethod(c.defs, "get", "O", tag);  // module.defs.get(tag)
        if (!st) okk = false;
        else if (st != Py_None) {
            PyObject* kind = PyObject_GetAttr(st, N.kind);
            int is_input = kind ? PyObject_RichCompareBool(kind, N.input_def, Py_EQ) : -1;
            Py_XDECREF(kind);
            okk = is_input >= 0;
            if (is_input > 0) {
                PyObject* ops = PyObject_GetAttr(st, N.operands);
                PyObject* s0 = ops ? PySequence_GetItem(ops, 0) : nullptr;
                Py_XDECREF(ops);
                okk = s0 != nullptr;
                if (okk) {
                    Py_DECREF(site);
                    site = s0;
                }
            }
        }
        Py_XDECREF(st);
        PyObject* entry = okk ? PyTuple_Pack(3, PyTuple_GET_ITEM(nd, 0), PyTuple_GET_ITEM(nd, 1), site) : nullptr;
        Py_DECREF(nd);
        Py_DECREF(site);
        int r = entry ? PyDict_SetItem(c.cache, key, entry) : -1;
        Py_DECREF(key);
        Py_XDECREF(entry);
        return r < 0 ? nullptr : entry;
    }

    PyObject* translate(PyObject* et) {  // new reference
        PyTypeObject* t = Py_TYPE(et);
        int kind = t == (PyTypeObject*)c.Const     ? 0
                   : t == (PyTypeObject*)c.Builtin ? 1
                   : t == (PyTypeObject*)c.Unknown ? 2
                   : t == (PyTypeObject*)c.LoopVar ? 3
                   : t == (PyTypeObject*)c.BinOp   ? 4
                                                   : -1;
        if (kind < 0) {  // isinstance, in the reference's order
            PyObject* order[5] = {c.Const, c.Builtin, c.Unknown, c.LoopVar, c.BinOp};
            for (int i = 0; i < 5 && kind < 0; i++) {
                int r = PyObject_IsInstance(et, order[i]);
                if (r < 0) return nullptr;
                if (r) kind = i;
            }
        }
        switch (kind) {
        case 0: {
            PyObject* v = PyObject_GetAttr(et, N.value);
            if (!v) return nullptr;
            PyObject* l = make_lit(c, v);
            Py_DECREF(v);
            return l;
        }
        case 1: {
            PyObject* axis = PyObject_GetAttr(et, N.axis);
            if (!axis) return nullptr;
            PyObject* name = PyUnicode_Concat(N.sol, axis);
            Py_DECREF(axis);
            if (!name) return nullptr;
            PyObject* ref = var(name, N.zero, nullptr);
            Py_DECREF(name);
            return ref;
        }
        case 2: {
            PyObject* tag = PyObject_GetAttr(et, N.tag);
            if (!tag) return nullptr;
            PyObject* u = unknown(tag);
            Py_DECREF(tag);
            if (!u) return nullptr;
            PyObject *name = PyTuple_GET_ITEM(u, 0), *display = PyTuple_GET_ITEM(u, 1), *site = PyTuple_GET_ITEM(u, 2);
            PyObject* ref = var(name, N.zero, nullptr);
            if (!ref) return nullptr;
            PyObject* d = PyDict_SetDefault(witness, name, display);
            if (d && site != Py_None) d = PyDict_SetDefault(inputs, name, site);
            if (!d) {
                Py_DECREF(ref);
                return nullptr;
            }
            return ref;
        }
        case 3: {
            PyObject* tag = PyObject_GetAttr(et, N.tag);
            if (!tag) return nullptr;
            PyObject* tname = PyObject_GetAttr(tag, N.name);
            PyObject* tid = tname ? PyObject_GetAttr(tag, N.id) : nullptr;
            PyObject* name = nullptr;
            if (tid) {
                int truthy = PyObject_IsTrue(tname);
                if (truthy >= 0) name = PyUnicode_FromFormat("sol_%S_v%S", truthy ? tname : N.loop, tid);
            }
            Py_XDECREF(tname);
            Py_XDECREF(tid);
            PyObject* ref = name ? var(name, N.zero, nullptr) : nullptr;
            Py_XDECREF(name);
            if (!ref) {
                Py_DECREF(tag);
                return nullptr;
            }
            int seen = PySet_Contains(loop_seen, tag);
            bool okk = seen >= 0;
            if (okk && !seen) {
                okk = PySet_Add(loop_seen, tag) == 0;
                PyObject* lo_et = okk ? PyObject_GetAttr(et, N.lower) : nullptr;
                PyObject* hi_et = lo_et ? PyObject_GetAttr(et, N.upper) : nullptr;
                PyObject* lower = hi_et ? translate(lo_et) : nullptr;
                PyObject* upper = lower ? translate(hi_et) : nullptr;
                Py_XDECREF(lo_et);
                Py_XDECREF(hi_et);
                okk = upper != nullptr;
                if (okk) {
                    Py_INCREF(ref);
                    okk = append(make_con(c, N.ge, ref, lower));
                    lower = nullptr;
                    if (okk) {
                        Py_INCREF(ref);
                        okk = append(make_con(c, N.lt, ref, upper));
                        upper = nullptr;
                    }
                }
                Py_XDECREF(lower);
                Py_XDECREF(upper);
            }
            Py_DECREF(tag);
            if (!okk) {
                Py_DECREF(ref);
                return nullptr;
            }
            return ref;
        }
        case 4: {
            PyObject* op = PyObject_GetAttr(et, N.op);
            if (!op) return nullptr;
            int cmp = PySequence_Contains(c.comparison_ops, op);
            int ar = cmp == 0 ? PySequence_Contains(c.arith_ops, op) : 0;
            if (cmp < 0 || ar < 0) {
                Py_DECREF(op);
                return nullptr;
            }
            if (cmp) {
                Py_DECREF(op);
                analysis_error(c, PyUnicode_FromString("comparison in arithmetic position"));
                return nullptr;
            }
            if (!ar) {
                analysis_error(c, PyUnicode_FromFormat("unknown operator %R", op));
                Py_DECREF(op);
                return nullptr;
            }
            PyObject* le = PyObject_GetAttr(et, N.left);
            PyObject* re = le ? PyObject_GetAttr(et, N.right) : nullptr;
            PyObject* l = re ? translate(le) : nullptr;
            PyObject* r = l ? translate(re) : nullptr;
            Py_XDECREF(le);
            Py_XDECREF(re);
            if (!r) {
                Py_XDECREF(l);
                Py_DECREF(op);
                return nullptr;
            }
            PyObject* b = make_bin(c, op, l, r);
            Py_DECREF(op);
            return b;
        }
        default: {
            analysis_error(c, PyUnicode_FromFormat("unhandled ET node %s", t->tp_name));
            return nullptr;
        }
        }
    }

    bool add_comparison(PyObject* et) {
        PyObject* op = PyObject_GetAttr(et, N.op);
        if (!op) return false;
        int ne = PyObject_RichCompareBool(op, N.ne, Py_EQ);
        if (ne != 0) {
            Py_DECREF(op);
            return ne > 0;
        }
        PyObject* rel = PyDict_GetItemWithError(c.rel_map, op);
        if (!rel) {
            if (!PyErr_Occurred()) analysis_error(c, PyUnicode_FromFormat("not a comparison root: %R", op));
            Py_DECREF(op);
            return false;
        }
        Py_DECREF(op);
        PyObject* le = PyObject_GetAttr(et, N.left);
        PyObject* re = le ? PyObject_GetAttr(et, N.right) : nullptr;
        PyObject* l = re ? translate(le) : nullptr;
        PyObject* r = l ? translate(re) : nullptr;
        Py_XDECREF(le);
        Py_XDECREF(re);
        if (!r) {
            Py_XDECREF(l);
            return false;
        }
        return append(make_con(c, rel, l, r));
    }

    bool declare_geometry(PyObject* launch) {
        PyObject* axes = c.all_axes;
        const Py_ssize_t na = PyTuple_GET_SIZE(axes);
        for (Py_ssize_t i = 0; i < na; i++) {
            PyObject* name = PyUnicode_Concat(N.sol, PyTuple_GET_ITEM(axes, i));
            PyObject* ref = name ? var(name, N.zero, nullptr) : nullptr;
            Py_XDECREF(name);
            if (!ref) return false;
            Py_DECREF(ref);
        }
        static const char* pairs[6][2] = {{"TidX", "BDimX"}, {"TidY", "BDimY"}, {"TidZ", "BDimZ"},
                                          {"BidX", "GDimX"}, {"BidY", "GDimY"}, {"BidZ", "GDimZ"}};
        for (auto& p : pairs) {
            PyObject* iname = PyUnicode_FromFormat("sol%s", p[0]);
            PyObject* dname = iname ? PyUnicode_FromFormat("sol%s", p[1]) : nullptr;
            bool okk = dname != nullptr;
            if (okk) okk = append(make_con(c, N.ge, make_ref(c, iname), make_lit(c, N.zero)));
            if (okk) okk = append(make_con(c, N.lt, make_ref(c, iname), make_ref(c, dname)));
            Py_XDECREF(iname);
            Py_XDECREF(dname);
            if (!okk) return false;
        }
        PyObject* grid = PyObject_GetAttr(launch, N.grid_ets);
        if (!grid) return false;
        PyObject* it = PyObject_GetIter(grid);
        Py_DECREF(grid);
        if (!it) return false;
        const Py_ssize_t ng = PyTuple_GET_SIZE(c.grid_axes);
        bool okk = true;
        for (Py_ssize_t i = 0; i < ng && okk; i++) {  // zip(GRID_AXES, launch.grid_ets)
            PyObject* et = PyIter_Next(it);
            if (!et) {
                okk = !PyErr_Occurred();
                break;
            }
            PyObject* name = PyUnicode_Concat(N.sol, PyTuple_GET_ITEM(c.grid_axes, i));
            PyObject* ref = name ? make_ref(c, name) : nullptr;
            Py_XDECREF(name);
            PyObject* rhs = ref ? translate(et) : nullptr;
            Py_DECREF(et);
            okk = ref && rhs ? append(make_con(c, N.eq, ref, rhs)) : false;
            if (!okk) {
                if (!rhs) Py_XDECREF(ref);
            }
        }
        Py_DECREF(it);
        return okk;
    }

    // list prefix: len(prefix) <= len(full) and full[:len(prefix)] == prefix
    static int is_prefix(PyObject* prefix, PyObject* full) {
        Py_ssize_t lp = PyObject_Length(prefix), lf = PyObject_Length(full);
        if (lp < 0 || lf < 0) return -1;
        if (lp > lf) return 0;
        PyObject* head = PySequence_GetSlice(full, 0, lp);
        if (!head) return -1;
        int r = PyObject_RichCompareBool(head, prefix, Py_EQ);
        Py_DECREF(head);
        return r;
    }

    bool add_context(PyObject* kernel, PyObject* launch, PyObject* host_summary, PyObject* ksum, PyObject* guards) {
        PyObject* params = PyObject_GetAttr(kernel, N.params);
        PyObject* args = params ? PyObject_GetAttr(launch, N.args) : nullptr;
        PyObject* pi = args ? PyObject_GetIter(params) : nullptr;
        PyObject* ai = pi ? PyObject_GetIter(args) : nullptr;
        Py_XDECREF(params);
        Py_XDECREF(args);
        bool okk = ai != nullptr;
        while (okk) {  // zip(kernel.params, launch.args)
            PyObject* p = PyIter_Next(pi);
            if (!p) {
                okk = !PyErr_Occurred();
                break;
            }
            PyObject* a = PyIter_Next(ai);
            if (!a) {
                Py_DECREF(p);
                okk = !PyErr_Occurred();
                break;
            }
            PyObject* isp = PyObject_GetAttr(p, N.is_pointer);
            int ptr = isp ? PyObject_IsTrue(isp) : -1;
            Py_XDECREF(isp);
            okk = ptr >= 0;
            if (okk && !ptr) {
                PyObject* vid = PyObject_GetAttr(p, N.vid);
                PyObject* u = vid ? unknown(vid) : nullptr;
                Py_XDECREF(vid);
                PyObject* ref = u ? var(PyTuple_GET_ITEM(u, 0), N.zero, nullptr) : nullptr;
                okk = ref != nullptr;
                if (okk) okk = PyDict_SetDefault(witness, PyTuple_GET_ITEM(u, 0), PyTuple_GET_ITEM(u, 1)) != nullptr;
                PyObject* vet = okk ? PyObject_GetAttr(a, N.value_et) : nullptr;
                PyObject* rhs = vet ? translate(vet) : nullptr;
                Py_XDECREF(vet);
                if (rhs) okk = append(make_con(c, N.eq, ref, rhs));
                else {
                    Py_XDECREF(ref);
                    okk = false;
                }
            }
            Py_DECREF(p);
            Py_DECREF(a);
        }
        Py_XDECREF(pi);
        Py_XDECREF(ai);
        if (!okk) return false;
        // host asserts
        PyObject* ha = PyObject_GetAttr(host_summary, N.asserts);
        PyObject* hi = ha ? PyObject_GetIter(ha) : nullptr;
        Py_XDECREF(ha);
        if (!hi) return false;
        for (PyObject* cond; okk && (cond = PyIter_Next(hi));) {
            okk = add_comparison(cond);
            Py_DECREF(cond);
        }
        Py_DECREF(hi);
        if (!okk || PyErr_Occurred()) return false;
        // kernel asserts on a dominating path
        PyObject* ka = PyObject_GetAttr(ksum, N.asserts);
        PyObject* ki = ka ? PyObject_GetIter(ka) : nullptr;
        Py_XDECREF(ka);
        if (!ki) return false;
        for (PyObject* a; okk && (a = PyIter_Next(ki));) {
            PyObject* pg = PyObject_GetAttr(a, N.path_guards);
            int pre = pg ? is_prefix(pg, guards) : -1;
            Py_XDECREF(pg);
            okk = pre >= 0;
            if (okk && pre) {
                PyObject* ce = PyObject_GetAttr(a, N.cond_et);
                okk = ce && add_comparison(ce);
                Py_XDECREF(ce);
            }
            Py_DECREF(a);
        }
        Py_DECREF(ki);
        if (!okk || PyErr_Occurred()) return false;
        // guards along the access path
        PyObject* gi = PyObject_GetIter(guards);
        if (!gi) return false;
        for (PyObject* g; okk && (g = PyIter_Next(gi));) {
            okk = add_comparison(g);
            Py_DECREF(g);
        }
        Py_DECREF(gi);
        return okk && !PyErr_Occurred();
    }

    PyObject* finish(PyObject* check) {  // ConstraintSet(...)
        PyObject* vlist = PyDict_Values(vars);
        if (!vlist) return nullptr;
        PyObject* kw = Py_BuildValue("{sOsOsOsOsO}", "variables", vlist, "constraints", cons, "check", check,
                                     "witness_leaves", witness, "input_leaves", inputs);
        Py_DECREF(vlist);
        if (!kw) return nullptr;
        PyObject* empty = PyTuple_New(0);
        PyObject* cs = empty ? PyObject_Call(c.ConstraintSet, empty, kw) : nullptr;
        Py_XDECREF(empty);
        Py_DECREF(kw);
        return cs;
    }
};

// access_set(ctx, kernel, ksum, host_summary, launch, offset_et, size_et,
//            guards, check, offset_lo, offset_hi) -- constraint_sets_for_access's
// loop body (constraint_gen.py:295-308) for one check ("upper" / "lower")
PyObject* access_set(PyObject*, PyObject* args) {
    PyObject *ctx, *kernel, *ksum, *host_summary, *launch, *offset_et, *size_et, *guards, *check;
    PyObject *offset_name, *size_name, *neg_max;
    if (!PyArg_ParseTuple(args, "OOOOOOOOOOOO", &ctx, &kernel, &ksum, &host_summary, &launch, &offset_et, &size_et,
                          &guards, &check, &offset_name, &size_name, &neg_max))
        return nullptr;
    Ctx c;
    if (!unpack(ctx, c)) return nullptr;
    Builder b(c);
    if (!b.ok()) return nullptr;
    if (!b.declare_geometry(launch)) return nullptr;
    PyObject* offset = b.var(offset_name, neg_max, c.max_domain);
    PyObject* size = offset ? b.var(size_name, N.zero, c.max_domain) : nullptr;
    if (!size) {
        Py_XDECREF(offset);
        return nullptr;
    }
    const int upper = PyUnicode_CompareWithASCIIString(check, "upper") == 0;
    bool okk;
    Py_INCREF(offset);
    if (upper) {
        Py_INCREF(size);
        okk = b.append(make_con(c, N.ge, offset, size));
    } else {
        okk = b.append(make_con(c, N.lt, offset, make_lit(c, N.zero)));
    }
    if (okk) {
        PyObject* rhs = b.translate(offset_et);
        if (rhs) {
            Py_INCREF(offset);
            okk = b.append(make_con(c, N.eq, offset, rhs));
        } else okk = false;
    }
    if (okk) {
        PyObject* rhs = b.translate(size_et);
        if (rhs) {
            Py_INCREF(size);
            okk = b.append(make_con(c, N.eq, size, rhs));
        } else okk = false;
    }
    Py_DECREF(offset);
    Py_DECREF(size);
    if (!okk || !b.add_context(kernel, launch, host_summary, ksum, guards)) return nullptr;
    return b.finish(check);
}

// layout_set(ctx, kernel, ksum, host_summary, launch, later_offset_et,
//            earlier_offset_et, check) -- layout_check_sets's loop body
// (constraint_gen.py:332-344)
PyObject* layout_set(PyObject*, PyObject* args) {
    PyObject *ctx, *kernel, *ksum, *host_summary, *launch, *later, *earlier, *check, *empty_guards;
    if (!PyArg_ParseTuple(args, "OOOOOOOOO", &ctx, &kernel, &ksum, &host_summary, &launch, &later, &earlier, &check,
                          &empty_guards))
        return nullptr;
    Ctx c;
    if (!unpack(ctx, c)) return nullptr;
    Builder b(c);
    if (!b.ok()) return nullptr;
    if (!b.declare_geometry(launch)) return nullptr;
    PyObject* l = b.translate(later);
    PyObject* r = l ? b.translate(earlier) : nullptr;
    if (!r) {
        Py_XDECREF(l);
        return nullptr;
    }
    if (!b.append(make_con(c, N.lt, l, r))) return nullptr;
    if (!b.add_context(kernel, launch, host_summary, ksum, empty_guards)) return nullptr;
    return b.finish(check);
}

PyMethodDef methods[] = {
    {"access_set", access_set, METH_VARARGS, "one access check's ConstraintSet (constraint_gen.py:295-308)"},
    {"layout_set", layout_set, METH_VARARGS, "one partition-layout ConstraintSet (constraint_gen.py:332-344)"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_emit_native",
                      "native constraint-set construction for the analyzer path", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__emit_native(void) {
    if (!init_names()) return nullptr;
    return PyModule_Create(&moddef);
}
