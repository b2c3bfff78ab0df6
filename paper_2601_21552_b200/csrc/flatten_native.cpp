// flatten_native.cpp -- native query emission for the Python shim (SURVEY.md
// 8(f) rank 1): turns reference-shaped queries -- (variables, constraints)
// pairs of the reference's SolverVar / Constraint / Lit / VarRef / BinE
// objects (solver.py:32-63), or the JSON form of terms.py -- into the flat
// oob_batch arrays of include/scuba_oob.h, walking the Python objects through
// the CPython API instead of interpreted Python (wire.py `_Builder`, ~100 us
// per analyzer-shaped query).
//
// Semantics are those of wire.py `_Builder.add` / `finish`, rule for rule:
//  * variables: dict semantics of solver.py:372-374 -- the last declaration of
//    a name wins, the first position is kept; the first empty declaration
//    (lo > hi) is stored into slot 0 so that the query is Unsat before search;
//  * terms are hash-consed per query in post-order (children first), literals
//    deduplicated by value, so structural equality is node-id equality;
//  * a query with an empty domain whose constraints do not resolve keeps no
//    constraints (Unsat before search; the reference never evaluates them)
//  * errors: KeyError(name) for an undeclared variable, ValueError for an
//    unknown operator / relation or a boolean term, OverflowError (raised after
//    the whole batch, as finish() does) for a value outside int128.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

using i128 = __int128;

constexpr int NODE_LIT = 0, NODE_VAR = 1;

struct Interned {
    PyObject *name, *lo, *hi, *rel, *lhs, *rhs, *op, *left, *right, *value, *vars, *cons;
    PyObject *plus, *minus, *times, *div, *mod;
    PyObject *lt, *le, *eq, *ge, *gt;
    PyObject *i128_min, *i128_max, *shift64, *mask64;
};
Interned S;

bool init_interned() {
#define I(f, s) S.f = PyUnicode_InternFromString(s); if (!S.f) return false;
    I(name, "name") I(lo, "lo") I(hi, "hi") I(rel, "rel") I(lhs, "lhs") I(rhs, "rhs") I(op, "op")
    I(left, "left") I(right, "right") I(value, "value") I(vars, "vars") I(cons, "cons")
    I(plus, "+") I(minus, "-") I(times, "*") I(div, "/") I(mod, "%")
    I(lt, "<") I(le, "<=") I(eq, "=") I(ge, ">=") I(gt, ">")
#undef I
    S.i128_min = PyLong_FromString("-170141183460469231731687303715884105728", nullptr, 10);
    S.i128_max = PyLong_FromString("170141183460469231731687303715884105727", nullptr, 10);
    S.shift64 = PyLong_FromLong(64);
    S.mask64 = PyLong_FromString("18446744073709551615", nullptr, 10);
    return S.i128_min && S.i128_max && S.shift64 && S.mask64;
}

int op_code(PyObject* op) {  // wire.OP_CODE; -1 unknown
    if (!PyUnicode_Check(op)) return -1;
    if (PyUnicode_Compare(op, S.plus) == 0) return 2;
    if (PyUnicode_Compare(op, S.minus) == 0) return 3;
    if (PyUnicode_Compare(op, S.times) == 0) return 4;
    if (PyUnicode_Compare(op, S.div) == 0) return 5;
    if (PyUnicode_Compare(op, S.mod) == 0) return 6;
    return -1;
}

int rel_code(PyObject* r) {  // terms.RELS order: < <= = >= >
    if (!PyUnicode_Check(r)) return -1;
    if (PyUnicode_Compare(r, S.lt) == 0) return 0;
    if (PyUnicode_Compare(r, S.le) == 0) return 1;
    if (PyUnicode_Compare(r, S.eq) == 0) return 2;
    if (PyUnicode_Compare(r, S.ge) == 0) return 3;
    if (PyUnicode_Compare(r, S.gt) == 0) return 4;
    return -1;
}

// Python int -> int128; *out_of_range set (value 0) when outside int128.
// Returns false with a Python error set on a conversion failure.
bool to_i128(PyObject* v, i128* out, bool* out_of_range) {
    *out_of_range = false;
    int overflow = 0;
    long long x = PyLong_AsLongLongAndOverflow(v, &overflow);
    if (x == -1 && PyErr_Occurred()) return false;
    if (!overflow) {
        *out = x;
        return true;
    }
    int lt = PyObject_RichCompareBool(v, S.i128_min, Py_LT);
    int gt = PyObject_RichCompareBool(v, S.i128_max, Py_GT);
    if (lt < 0 || gt < 0) return false;
    if (lt || gt) {
        *out = 0;
        *out_of_range = true;
        return true;
    }
    PyObject* hi = PyNumber_Rshift(v, S.shift64);
    PyObject* lo = hi ? PyNumber_And(v, S.mask64) : nullptr;
    if (!lo) {
        Py_XDECREF(hi);
        return false;
    }
    long long h = PyLong_AsLongLong(hi);
    unsigned long long l = PyLong_AsUnsignedLongLong(lo);
    Py_DECREF(hi);
    Py_DECREF(lo);
    if (PyErr_Occurred()) return false;
    *out = ((i128)h << 64) | (i128)l;
    return true;
}

struct Out {
    std::vector<int64_t> var_begin{0}, con_begin{0}, node_begin{0}, lit_begin{0};
    std::vector<i128> var_lo, var_hi, lits;
    std::vector<uint8_t> con_rel, node_op;
    std::vector<int32_t> con_lhs, con_rhs, node_a, node_b;
    // first out-of-range value per array (finish() checks var_lo, var_hi, lits in turn)
    PyObject* bad[3] = {nullptr, nullptr, nullptr};
};

struct KeyHash {
    size_t operator()(uint64_t k) const { return (size_t)(k * 0x9E3779B97F4A7C15ull >> 7); }
};
struct LitHash {
    size_t operator()(const i128& v) const {
        uint64_t a = (uint64_t)v, b = (uint64_t)(v >> 64);
        return (size_t)((a * 0x9E3779B97F4A7C15ull) ^ (b * 0xC2B2AE3D27D4EB4Full));
    }
};

// kinds of term objects, cached per Python type (the reference's Lit / VarRef
// / BinE are plain dataclasses: one hasattr resolution per type per call)
enum Kind { K_LIT = 1, K_VAR = 2, K_BIN = 3 };

class Query {
  public:
    Query(Out& o, std::unordered_map<PyTypeObject*, int>& kinds) : o_(o), kinds_(kinds) {}
    ~Query() {
        Py_XDECREF(index_);
        Py_XDECREF(names_);
        release_bad();
    }
    void release_bad() {
        for (PyObject* b : bad_lo_) Py_XDECREF(b);
        for (PyObject* b : bad_hi_) Py_XDECREF(b);
        bad_lo_.clear();
        bad_hi_.clear();
        Py_XDECREF(e_blo);
        Py_XDECREF(e_bhi);
        e_blo = e_bhi = nullptr;
    }

    bool add(PyObject* variables, PyObject* constraints) {
        // per-query state (containers keep their capacity across queries)
        Py_XDECREF(index_);
        Py_XDECREF(names_);
        index_ = PyDict_New();
        names_ = PyList_New(0);
        if (!index_ || !names_) return false;
        release_bad();
        lo_.clear();
        hi_.clear();
        nodes_.clear();
        lit_index_.clear();
        n_op_.clear();
        n_a_.clear();
        n_b_.clear();
        q_lits_.clear();
        if (!add_vars(variables)) return false;
        // a query with an empty domain is Unsat before its constraints are
        // ever evaluated (solver.py:374): if they do not resolve (undeclared
        // variable, unknown operator -- the reference raises nothing then),
        // the query keeps no constraints
        {
            const size_t c0 = o_.con_rel.size();
            PyObject* seq = PySequence_Fast(constraints, "constraints must be iterable");
            if (!seq) return false;
            bool ok = true;
            const Py_ssize_t nc = PySequence_Fast_GET_SIZE(seq);
            for (Py_ssize_t k = 0; k < nc && ok; k++) ok = add_con(PySequence_Fast_GET_ITEM(seq, k));
            Py_DECREF(seq);
            if (!ok && q_empty_) {
                PyErr_Clear();
                o_.con_rel.resize(c0);
                o_.con_lhs.resize(c0);
                o_.con_rhs.resize(c0);
                nodes_.clear();
                lit_index_.clear();
                n_op_.clear();
                n_a_.clear();
                n_b_.clear();
                q_lits_.clear();
                ok = true;
            }
            if (!ok) return false;
        }
        // append (finish() range-checks the stored values: var_lo, var_hi, lits)
        for (size_t i = 0; i < lo_.size(); i++) {
            o_.var_lo.push_back(lo_[i]);
            o_.var_hi.push_back(hi_[i]);
            if (bad_lo_[i]) note_bad(0, bad_lo_[i]);
            if (bad_hi_[i]) note_bad(1, bad_hi_[i]);
        }
        o_.var_begin.push_back(o_.var_begin.back() + (int64_t)lo_.size());
        o_.con_begin.push_back((int64_t)o_.con_rel.size());
        for (size_t i = 0; i < n_op_.size(); i++) {
            o_.node_op.push_back(n_op_[i]);
            o_.node_a.push_back(n_a_[i]);
            o_.node_b.push_back(n_b_[i]);
        }
        o_.node_begin.push_back(o_.node_begin.back() + (int64_t)n_op_.size());
        for (size_t i = 0; i < q_lits_.size(); i++) o_.lits.push_back(q_lits_[i]);
        o_.lit_begin.push_back(o_.lit_begin.back() + (int64_t)q_lits_.size());
        return true;
    }
    PyObject* take_names() {
        PyObject* n = names_;
        names_ = nullptr;
        return n;
    }

  private:
    Out& o_;
    std::unordered_map<PyTypeObject*, int>& kinds_;
    PyObject* index_ = nullptr;  // name -> position
    PyObject* names_ = nullptr;
    std::vector<i128> lo_, hi_;
    std::vector<PyObject*> bad_lo_, bad_hi_;  // stored out-of-range values (or null)
    PyObject *e_blo = nullptr, *e_bhi = nullptr;
    bool q_empty_ = false;  // the current query has an empty domain
    static int sign_of(PyObject* big) {  // sign of an int beyond the long long range
        int ovf = 0;
        PyLong_AsLongLongAndOverflow(big, &ovf);
        return ovf;
    }
    std::unordered_map<uint64_t, int32_t, KeyHash> nodes_;
    std::unordered_map<i128, int32_t, LitHash> lit_index_;
    std::vector<uint8_t> n_op_;
    std::vector<int32_t> n_a_, n_b_;
    std::vector<i128> q_lits_;

    void note_bad(int arr, PyObject* v) {
        if (!o_.bad[arr]) {
            Py_INCREF(v);
            o_.bad[arr] = v;
        }
    }

    // int(x); an out-of-range value is kept (*bad, new reference) for the
    // range check of the stored values, which happens after the whole batch
    bool int_field(PyObject* raw, i128* out, PyObject** bad) {
        *bad = nullptr;
        PyObject* v = PyNumber_Long(raw);
        if (!v) return false;
        bool oor;
        bool ok = to_i128(v, out, &oor);
        if (ok && oor) {
            *bad = v;
            return true;
        }
        Py_DECREF(v);
        return ok;
    }
    static void set_ref(PyObject*& slot, PyObject* v) {
        Py_XINCREF(v);
        Py_XDECREF(slot);
        slot = v;
    }

    bool add_vars(PyObject* variables) {
        PyObject* seq = PySequence_Fast(variables, "variables must be iterable");
        if (!seq) return false;
        const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
        bool have_empty = false;
        i128 e_lo = 0, e_hi = 0;
        bool ok = true;
        for (Py_ssize_t i = 0; i < n && ok; i++) {
            PyObject* v = PySequence_Fast_GET_ITEM(seq, i);
            PyObject *rn, *rlo, *rhi;
            if (PyList_Check(v) || PyTuple_Check(v)) {
                if (PySequence_Size(v) != 3) {
                    PyErr_SetString(PyExc_ValueError, "variable must be (name, lo, hi)");
                    ok = false;
                    break;
                }
                rn = PySequence_GetItem(v, 0);
                rlo = PySequence_GetItem(v, 1);
                rhi = PySequence_GetItem(v, 2);
            } else {
                rn = PyObject_GetAttr(v, S.name);
                rlo = rn ? PyObject_GetAttr(v, S.lo) : nullptr;
                rhi = rlo ? PyObject_GetAttr(v, S.hi) : nullptr;
            }
            PyObject* name = (rn && rlo && rhi) ? PyObject_Str(rn) : nullptr;
            i128 lo = 0, hi = 0;
            PyObject *blo = nullptr, *bhi = nullptr;
            ok = name && int_field(rlo, &lo, &blo) && int_field(rhi, &hi, &bhi);
            Py_XDECREF(rn);
            Py_XDECREF(rlo);
            Py_XDECREF(rhi);
            if (ok) {
                // lo > hi with Python ints: a value beyond int128 is past every
                // in-range value on its side
                int empty;
                if (blo && bhi) empty = PyObject_RichCompareBool(blo, bhi, Py_GT);
                else if (blo) empty = sign_of(blo) > 0;
                else if (bhi) empty = sign_of(bhi) < 0;
                else empty = lo > hi;
                if (empty < 0) ok = false;
                if (ok && empty && !have_empty) {
                    have_empty = true;
                    e_lo = lo;
                    e_hi = hi;
                    set_ref(e_blo, blo);
                    set_ref(e_bhi, bhi);
                }
                PyObject* at = ok ? PyDict_GetItemWithError(index_, name) : nullptr;
                if (at) {  // last declaration wins, first position kept
                    const Py_ssize_t k = PyLong_AsSsize_t(at);
                    lo_[k] = lo;
                    hi_[k] = hi;
                    set_ref(bad_lo_[k], blo);
                    set_ref(bad_hi_[k], bhi);
                } else if (!ok || PyErr_Occurred()) {
                    ok = false;
                } else {
                    PyObject* pos = PyLong_FromSsize_t((Py_ssize_t)lo_.size());
                    ok = pos && PyDict_SetItem(index_, name, pos) == 0 && PyList_Append(names_, name) == 0;
                    Py_XDECREF(pos);
                    lo_.push_back(lo);
                    hi_.push_back(hi);
                    bad_lo_.push_back(nullptr);
                    bad_hi_.push_back(nullptr);
                    set_ref(bad_lo_.back(), blo);
                    set_ref(bad_hi_.back(), bhi);
                }
            }
            Py_XDECREF(blo);
            Py_XDECREF(bhi);
            Py_XDECREF(name);
        }
        Py_DECREF(seq);
        q_empty_ = ok && have_empty;
        if (ok && have_empty) {  // Unsat before search (solver.py:374)
            lo_[0] = e_lo;
            hi_[0] = e_hi;
            set_ref(bad_lo_[0], e_blo);
            set_ref(bad_hi_[0], e_bhi);
        }
        return ok;
    }

    int32_t node(int op, int32_t a, int32_t b) {
        const uint64_t key = (uint64_t)op | ((uint64_t)(uint32_t)a << 3) | ((uint64_t)(uint32_t)b << 33);
        auto it = nodes_.find(key);
        if (it != nodes_.end()) return it->second;
        const int32_t i = (int32_t)n_op_.size();
        nodes_.emplace(key, i);
        n_op_.push_back((uint8_t)op);
        n_a_.push_back(a);
        n_b_.push_back(b);
        return i;
    }

    int kind_of(PyObject* e) {
        PyTypeObject* t = Py_TYPE(e);
        auto it = kinds_.find(t);
        if (it != kinds_.end()) return it->second;
        int k = 0;
        if (PyObject_HasAttr(e, S.op)) k = K_BIN;
        else if (PyObject_HasAttr(e, S.value)) k = K_LIT;
        else if (PyObject_HasAttr(e, S.name)) k = K_VAR;
        if (k) kinds_.emplace(t, k);
        return k;
    }

    int32_t lit_node(PyObject* v) {  // v: a Python int
        i128 x;
        bool oor;
        if (!to_i128(v, &x, &oor)) return -1;
        if (oor) note_bad(2, v);
        auto it = lit_index_.find(x);
        int32_t li;
        if (oor) {  // distinct out-of-range values never merge (the call fails anyway)
            li = (int32_t)q_lits_.size();
            q_lits_.push_back(0);
        } else if (it != lit_index_.end()) {
            li = it->second;
        } else {
            li = (int32_t)q_lits_.size();
            lit_index_.emplace(x, li);
            q_lits_.push_back(x);
        }
        return node(NODE_LIT, li, 0);
    }

    int32_t var_node(PyObject* name) {
        PyObject* at = PyDict_GetItemWithError(index_, name);
        if (!at) {
            if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, name);
            return -1;
        }
        const int32_t vi = (int32_t)PyLong_AsSsize_t(at);
        return node(NODE_VAR, vi, 0);
    }

    int32_t bin_node(PyObject* op, PyObject* l, PyObject* r) {
        const int code = op_code(op);
        if (code < 0) {
            PyObject* rep = PyObject_Repr(op);
            if (rep) {
                PyErr_Format(PyExc_ValueError, "unknown operator %U", rep);
                Py_DECREF(rep);
            }
            return -1;
        }
        const int32_t li = walk(l);
        if (li < 0) return -1;
        const int32_t ri = walk(r);
        if (ri < 0) return -1;
        return node(code, li, ri);
    }

    int32_t walk(PyObject* e) {  // wire._term_kind + _Builder.walk
        if (PyBool_Check(e)) {
            PyErr_SetString(PyExc_ValueError, "boolean is not a term");
            return -1;
        }
        if (PyLong_Check(e)) return lit_node(e);
        if (PyUnicode_Check(e)) return var_node(e);
        if (PyList_Check(e) || PyTuple_Check(e)) {
            PyObject *a = PySequence_GetItem(e, 0), *b = a ? PySequence_GetItem(e, 1) : nullptr,
                     *c = b ? PySequence_GetItem(e, 2) : nullptr;
            int32_t r = c ? bin_node(a, b, c) : -1;
            Py_XDECREF(a);
            Py_XDECREF(b);
            Py_XDECREF(c);
            return r;
        }
        const int k = kind_of(e);
        if (k == K_BIN) {
            PyObject* op = PyObject_GetAttr(e, S.op);
            PyObject* l = op ? PyObject_GetAttr(e, S.left) : nullptr;
            PyObject* r = l ? PyObject_GetAttr(e, S.right) : nullptr;
            int32_t res = r ? bin_node(op, l, r) : -1;
            Py_XDECREF(op);
            Py_XDECREF(l);
            Py_XDECREF(r);
            return res;
        }
        if (k == K_LIT) {
            PyObject* raw = PyObject_GetAttr(e, S.value);
            PyObject* v = raw ? PyNumber_Long(raw) : nullptr;
            int32_t res = v ? lit_node(v) : -1;
            Py_XDECREF(raw);
            Py_XDECREF(v);
            return res;
        }
        if (k == K_VAR) {
            PyObject* n = PyObject_GetAttr(e, S.name);
            int32_t res = n ? var_node(n) : -1;
            Py_XDECREF(n);
            return res;
        }
        PyObject* rep = PyObject_Repr(e);
        if (rep) {
            PyErr_Format(PyExc_ValueError, "not a term: %U", rep);
            Py_DECREF(rep);
        }
        return -1;
    }

    bool add_con(PyObject* c) {
        PyObject *rel, *l, *r;
        if (PyList_Check(c) || PyTuple_Check(c)) {
            rel = PySequence_GetItem(c, 0);
            l = rel ? PySequence_GetItem(c, 1) : nullptr;
            r = l ? PySequence_GetItem(c, 2) : nullptr;
        } else {
            rel = PyObject_GetAttr(c, S.rel);
            l = rel ? PyObject_GetAttr(c, S.lhs) : nullptr;
            r = l ? PyObject_GetAttr(c, S.rhs) : nullptr;
        }
        bool ok = r != nullptr;
        if (ok) {
            const int code = rel_code(rel);
            if (code < 0) {
                PyObject* rep = PyObject_Repr(rel);
                if (rep) {
                    PyErr_Format(PyExc_ValueError, "unknown relation %U", rep);
                    Py_DECREF(rep);
                }
                ok = false;
            } else {
                const int32_t li = walk(l);
                const int32_t ri = li >= 0 ? walk(r) : -1;
                ok = ri >= 0;
                if (ok) {
                    o_.con_rel.push_back((uint8_t)code);
                    o_.con_lhs.push_back(li);
                    o_.con_rhs.push_back(ri);
                }
            }
        }
        Py_XDECREF(rel);
        Py_XDECREF(l);
        Py_XDECREF(r);
        return ok;
    }
};

template <typename T>
PyObject* bytes_of(const std::vector<T>& v) {
    return PyByteArray_FromStringAndSize(reinterpret_cast<const char*>(v.data()), (Py_ssize_t)(v.size() * sizeof(T)));
}

PyObject* words_of(const std::vector<i128>& v) {  // [k,2] little-endian int64 words
    std::vector<int64_t> w(v.size() * 2);
    for (size_t i = 0; i < v.size(); i++) {
        w[2 * i] = (int64_t)(uint64_t)v[i];
        w[2 * i + 1] = (int64_t)(v[i] >> 64);
    }
    return bytes_of(w);
}

PyObject* flatten(PyObject*, PyObject* args) {
    PyObject* queries;
    if (!PyArg_ParseTuple(args, "O", &queries)) return nullptr;
    PyObject* seq = PySequence_Fast(queries, "queries must be iterable");
    if (!seq) return nullptr;
    Out o;
    std::unordered_map<PyTypeObject*, int> kinds;
    PyObject* names = PyList_New(0);
    bool ok = names != nullptr;
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
    Query qb(o, kinds);
    for (Py_ssize_t q = 0; q < n && ok; q++) {
        PyObject* item = PySequence_Fast_GET_ITEM(seq, q);
        PyObject *vars, *cons;
        if (PyDict_Check(item)) {
            vars = PyDict_GetItemWithError(item, S.vars);
            cons = vars ? PyDict_GetItemWithError(item, S.cons) : nullptr;
            if (!vars || !cons) {
                if (!PyErr_Occurred()) PyErr_SetString(PyExc_KeyError, vars ? "cons" : "vars");
                ok = false;
                break;
            }
            Py_INCREF(vars);
            Py_INCREF(cons);
        } else {
            vars = PySequence_GetItem(item, 0);
            cons = vars ? PySequence_GetItem(item, 1) : nullptr;
            if (!cons) {
                Py_XDECREF(vars);
                ok = false;
                break;
            }
        }
        ok = qb.add(vars, cons);
        Py_DECREF(vars);
        Py_DECREF(cons);
        if (ok) {
            PyObject* nm = qb.take_names();
            ok = PyList_Append(names, nm) == 0;
            Py_DECREF(nm);
        }
    }
    Py_DECREF(seq);
    if (ok) {
        for (int a = 0; a < 3; a++)
            if (o.bad[a]) {  // finish(): ints_to_words(var_lo), (var_hi), (lits)
                PyErr_Format(PyExc_OverflowError, "integer %S does not fit the engine's 128-bit wire format",
                             o.bad[a]);
                ok = false;
                break;
            }
    }
    for (auto* b : o.bad) Py_XDECREF(b);
    if (!ok) {
        Py_XDECREF(names);
        return nullptr;
    }
    return Py_BuildValue("(NNNNNNNNNNNNNN)", bytes_of(o.var_begin), words_of(o.var_lo), words_of(o.var_hi), names,
                         bytes_of(o.con_begin), bytes_of(o.con_rel), bytes_of(o.con_lhs), bytes_of(o.con_rhs),
                         bytes_of(o.node_begin), bytes_of(o.node_op), bytes_of(o.node_a), bytes_of(o.node_b),
                         bytes_of(o.lit_begin), words_of(o.lits));
}

PyMethodDef methods[] = {
    {"flatten", flatten, METH_VARARGS, "queries -> the 14 fields of wire.FlatBatch (buffers + names)"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_flatten_native", "native query emission (wire.flatten)", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__flatten_native(void) {
    if (!init_interned()) return nullptr;
    return PyModule_Create(&module);
}
