// jit.cpp -- run-time specialisation of structure classes (jit_lane.cuh).
//
// For a structure class (the code words of host.cpp compile_query: ncon
// constraint words, ncode postfix node words, 4 membership words per
// variable) this file emits a C++ struct whose prop_k / pass / check
// functions are the reference algorithm (solver.py:112-328) unrolled over the
// class's terms, compiles it with NVRTC for sm_100a and loads the cubin.
// Compiled kernels are cached per class for the life of the process.
//
// Emission rules (each mirrors engine.cuh Lane<T> exactly):
//   * _eval_iv (solver.py:112-149): postfix straight-line interval code; a
//     node without a non-trapping value returns false (contradiction);
//   * _propagate_constraint (:229-261): top-level eval of both sides, the
//     relation's targets with the +-10**18 clamp, then narrow(lhs), narrow(rhs);
//     constraints whose two sides are leaves use the leaf fast path;
//   * _Narrower.narrow (:159-226): pre-order recursion; both child targets are
//     computed from the children's intervals before either child is narrowed
//     (the reference's stale-sibling order).  The children's intervals come
//     from the top-level eval unless a variable of their subtrees may have
//     been narrowed earlier in this constraint, in which case they are
//     re-evaluated when the constraint is dirty (the interpreter's rule);
//   * check_model / _eval_exact (:286-328): exact postfix values, division or
//     modulo by zero falsifies.
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <cerrno>
#include <ctime>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include "format.h"
#include "jit.h"

namespace oob {

// embedded headers (build/jit_src.inc, made by embed.py from the csrc headers)
#include "build/jit_src.inc"

namespace {

inline uint32_t w_op(uint32_t w) { return w & 7u; }
inline uint32_t w_arg(uint32_t w) { return w >> 3; }

struct Gen {
    const uint32_t* cons;
    const uint32_t* code;
    const uint32_t* member;
    uint32_t nv, ncon, ncode, nlit;
    int bits = 64;
    std::ostringstream o;

    uint32_t size_of(uint32_t i) const { return w_op(code[i]) >= NODE_ADD ? w_arg(code[i]) : 1u; }
    uint32_t right(uint32_t i) const { return i - 1; }
    uint32_t left(uint32_t i) const { return i - 1 - size_of(i - 1); }
    void vars_of(uint32_t root, std::set<uint32_t>& out) const {
        for (uint32_t j = root + 1 - size_of(root); j <= root; j++)
            if (w_op(code[j]) == NODE_VAR) out.insert(w_arg(code[j]));
    }
    static std::string V(uint32_t j, const char* s) { return "v" + std::to_string(j) + "_" + s; }

    // interval evaluation of the subtree rooted at `root` into v<j>_lo/_hi
    void eval(uint32_t root, const std::string& ind) {
        for (uint32_t j = root + 1 - size_of(root); j <= root; j++) {
            uint32_t w = code[j], op = w_op(w), a = w_arg(w);
            std::string lo = V(j, "lo"), hi = V(j, "hi");
            if (op == NODE_LIT) {
                o << ind << lo << " = " << hi << " = s.lit[" << a << "];\n";
            } else if (op == NODE_VAR) {
                o << ind << lo << " = s.lo[" << a << "]; " << hi << " = s.hi[" << a << "]; if (" << lo << " > " << hi
                  << ") return false;\n";
            } else {
                uint32_t R = right(j), L = left(j);
                std::string l0 = V(L, "lo"), l1 = V(L, "hi"), r0 = V(R, "lo"), r1 = V(R, "hi");
                switch (op) {
                case NODE_ADD:
                    o << ind << lo << " = " << l0 << " + " << r0 << "; " << hi << " = " << l1 << " + " << r1 << ";\n";
                    break;
                case NODE_SUB:
                    o << ind << lo << " = " << l0 << " - " << r1 << "; " << hi << " = " << l1 << " - " << r0 << ";\n";
                    break;
                case NODE_MUL:
                    o << ind << "{ T k0 = " << l0 << " * " << r0 << ", k1 = " << l0 << " * " << r1 << ", k2 = " << l1
                      << " * " << r0 << ", k3 = " << l1 << " * " << r1 << "; " << lo
                      << " = A::mn(A::mn(k0, k1), A::mn(k2, k3)); " << hi
                      << " = A::mx(A::mx(k0, k1), A::mx(k2, k3)); }\n";
                    break;
                case NODE_DIV:
                    o << ind << "{ T d0 = A::mx(" << r0 << ", T(1)), d1 = " << r1
                      << "; if (d0 > d1) return false; T k0 = cdiv(" << l0 << ", d0), k1 = cdiv(" << l0
                      << ", d1), k2 = cdiv(" << l1 << ", d0), k3 = cdiv(" << l1 << ", d1); " << lo
                      << " = A::mn(A::mn(k0, k1), A::mn(k2, k3)); " << hi
                      << " = A::mx(A::mx(k0, k1), A::mx(k2, k3)); }\n";
                    break;
                default:  // NODE_MOD
                    o << ind << "{ T d0 = A::mx(" << r0 << ", T(1)), d1 = " << r1
                      << "; if (d0 > d1) return false; T m = d1 - T(1); if (" << l0 << " >= T(0)) { " << lo
                      << " = T(0); " << hi << " = A::mn(" << l1 << ", m); } else if (" << l1 << " <= T(0)) { "
                      << lo << " = A::mx(" << l0 << ", -m); " << hi << " = T(0); } else { " << lo << " = A::mx("
                      << l0 << ", -m); " << hi << " = A::mn(" << l1 << ", m); } }\n";
                    break;
                }
            }
        }
    }

    // _Narrower.narrow(node i, [ta, tb]) in pre-order; `seen` collects the
    // variables narrowed so far in this constraint
    void narrow(uint32_t i, const std::string& ta, const std::string& tb, std::set<uint32_t>& seen,
                const std::string& ind) {
        uint32_t w = code[i], op = w_op(w), a = w_arg(w);
        o << ind << "if (" << ta << " > " << tb << ") return false;\n";
        if (op == NODE_LIT) {
            o << ind << "if (!(" << ta << " <= s.lit[" << a << "] && s.lit[" << a << "] <= " << tb
              << ")) return false;\n";
            return;
        }
        if (op == NODE_VAR) {
            o << ind << "if (!s.narrow_var(" << a << ", " << ta << ", " << tb << ")) return false;\n";
            seen.insert(a);
            return;
        }
        uint32_t R = right(i), L = left(i);
        std::set<uint32_t> sub;
        vars_of(L, sub);
        vars_of(R, sub);
        bool stale = false;
        for (uint32_t v : sub)
            if (seen.count(v)) stale = true;
        if (stale) {
            o << ind << "if (s.dirty) {\n";
            eval(L, ind + "    ");
            eval(R, ind + "    ");
            o << ind << "}\n";
        }
        std::string p = "n" + std::to_string(i) + "_";
        std::string l0 = V(L, "lo"), l1 = V(L, "hi"), r0 = V(R, "lo"), r1 = V(R, "hi");
        switch (op) {
        case NODE_ADD:
            o << ind << "{ const T " << p << "la = X::sat(" << ta << " - " << r1 << "), " << p << "lb = X::sat(" << tb
              << " - " << r0 << "), " << p << "ra = X::sat(" << ta << " - " << l1 << "), " << p << "rb = X::sat(" << tb
              << " - " << l0 << ");\n";
            narrow(L, p + "la", p + "lb", seen, ind + "  ");
            narrow(R, p + "ra", p + "rb", seen, ind + "  ");
            o << ind << "}\n";
            break;
        case NODE_SUB:
            o << ind << "{ const T " << p << "la = X::sat(" << ta << " + " << r0 << "), " << p << "lb = X::sat(" << tb
              << " + " << r1 << "), " << p << "ra = X::sat(" << l0 << " - " << tb << "), " << p << "rb = X::sat(" << l1
              << " - " << ta << ");\n";
            narrow(L, p + "la", p + "lb", seen, ind + "  ");
            narrow(R, p + "ra", p + "rb", seen, ind + "  ");
            o << ind << "}\n";
            break;
        case NODE_MUL:
            o << ind << "if (!(" << l0 << " < T(0) || " << r0 << " < T(0))) {\n";
            o << ind << "  if (" << tb << " < T(0)) return false;\n";
            o << ind << "  const T " << p << "t0 = A::mx(" << ta << ", T(0));\n";
            o << ind << "  T " << p << "la = -A::inf(), " << p << "lb = A::inf(), " << p << "ra = -A::inf(), " << p
              << "rb = A::inf();\n";
            o << ind << "  if (" << p << "t0 > T(0)) { if (" << r1 << " == T(0) || " << l1
              << " == T(0)) return false; " << p << "la = A::ceil_div(" << p << "t0, " << r1 << "); " << p
              << "ra = A::ceil_div(" << p << "t0, " << l1 << "); }\n";
            o << ind << "  if (" << r0 << " > T(0)) " << p << "lb = X::big_hi(" << tb << ") ? A::inf() : A::fdiv(" << tb
              << ", " << r0 << ");\n";
            o << ind << "  if (" << l0 << " > T(0)) " << p << "rb = X::big_hi(" << tb << ") ? A::inf() : A::fdiv(" << tb
              << ", " << l0 << ");\n";
            narrow(L, p + "la", p + "lb", seen, ind + "  ");
            narrow(R, p + "ra", p + "rb", seen, ind + "  ");
            o << ind << "}\n";
            break;
        case NODE_DIV:
            if (w_op(code[R]) == NODE_LIT) {
                std::string c = "s.lit[" + std::to_string(w_arg(code[R])) + "]";
                o << ind << "if (" << c << " >= T(1)) {\n";
                o << ind << "  const T " << p << "c = " << c << ";\n";
                o << ind << "  const T " << p << "la = X::big_lo(" << ta << ") ? -A::inf() : (" << ta << " > T(0) ? " << ta
                  << " * " << p << "c : " << ta << " * " << p << "c - (" << p << "c - T(1)));\n";
                o << ind << "  const T " << p << "lb = X::big_hi(" << tb << ") ? A::inf() : (" << tb << " >= T(0) ? " << tb
                  << " * " << p << "c + (" << p << "c - T(1)) : " << tb << " * " << p << "c);\n";
                narrow(L, p + "la", p + "lb", seen, ind + "  ");
                o << ind << "}\n";
            }
            break;
        default:  // NODE_MOD: forward-only
            break;
        }
    }

    void rel_targets(uint32_t rel, const std::string& l0, const std::string& l1, const std::string& r0,
                     const std::string& r1, const std::string& ind) {
        switch (rel) {
        case REL_LT:
            o << ind << "const T a0 = -A::inf(), a1 = " << r1 << " - T(1), b0 = " << l0 << " + T(1), b1 = A::inf();\n";
            break;
        case REL_LE:
            o << ind << "const T a0 = -A::inf(), a1 = " << r1 << ", b0 = " << l0 << ", b1 = A::inf();\n";
            break;
        case REL_EQ:
            o << ind << "const T a0 = A::mx(" << l0 << ", " << r0 << "), a1 = A::mn(" << l1 << ", " << r1
              << "), b0 = a0, b1 = a1;\n";
            break;
        case REL_GE:
            o << ind << "const T a0 = " << r0 << ", a1 = A::inf(), b0 = -A::inf(), b1 = " << l1 << ";\n";
            break;
        default:
            o << ind << "const T a0 = " << r0 << " + T(1), a1 = A::inf(), b0 = -A::inf(), b1 = " << l1
              << " - T(1);\n";
            break;
        }
    }

    void leaf_side(uint32_t w, const char* p0, const char* p1, const std::string& ind) {
        if (w_op(w) == NODE_LIT) {
            o << ind << "const T " << p0 << " = s.lit[" << w_arg(w) << "], " << p1 << " = " << p0 << ";\n";
        } else {
            o << ind << "const T " << p0 << " = s.lo[" << w_arg(w) << "], " << p1 << " = s.hi[" << w_arg(w)
              << "]; if (" << p0 << " > " << p1 << ") return false;\n";
        }
    }
    void leaf_narrow(uint32_t w, const char* ta, const char* tb, const std::string& ind) {
        if (w_op(w) == NODE_LIT) {
            o << ind << "if (" << ta << " > " << tb << ") return false; if (!(" << ta << " <= s.lit[" << w_arg(w)
              << "] && s.lit[" << w_arg(w) << "] <= " << tb << ")) return false;\n";
        } else {
            o << ind << "if (!s.narrow_leaf_var(" << w_arg(w) << ", " << ta << ", " << tb << ")) return false;\n";
        }
    }

    void prop(uint32_t k) {
        uint32_t cw = cons[k], rel = cw & 7u, lr = (cw >> 3) & 0x3FFFu, rr = cw >> 17;
        o << "  template <class L> static __device__ __forceinline__ bool prop" << k << "(L& s) {\n";
        const std::string ind = "    ";
        if (w_op(code[lr]) < NODE_ADD && w_op(code[rr]) < NODE_ADD) {  // leaf fast path
            leaf_side(code[lr], "l0", "l1", ind);
            leaf_side(code[rr], "r0", "r1", ind);
            rel_targets(rel, "l0", "l1", "r0", "r1", ind);
            leaf_narrow(code[lr], "a0", "a1", ind);
            leaf_narrow(code[rr], "b0", "b1", ind);
            o << ind << "return true;\n  }\n";
            return;
        }
        uint32_t start = lr + 1 - size_of(lr);
        o << ind << "T";
        for (uint32_t j = start; j <= rr; j++) o << (j == start ? " " : ", ") << V(j, "lo") << ", " << V(j, "hi");
        o << ";\n";
        o << ind << "s.dirty = false;\n";
        eval(lr, ind);
        eval(rr, ind);
        rel_targets(rel, V(lr, "lo"), V(lr, "hi"), V(rr, "lo"), V(rr, "hi"), ind);
        std::set<uint32_t> seen;
        narrow(lr, "a0", "a1", seen, ind);
        narrow(rr, "b0", "b1", seen, ind);
        o << ind << "return true;\n  }\n";
    }

    void check() {
        o << "  template <class L> static __device__ __forceinline__ bool check(L& s) {\n";
        for (uint32_t k = 0; k < ncon; k++) {
            uint32_t cw = cons[k], rel = cw & 7u, lr = (cw >> 3) & 0x3FFFu, rr = cw >> 17;
            uint32_t start = lr + 1 - size_of(lr);
            o << "    {\n";
            for (uint32_t j = start; j <= rr; j++) {
                uint32_t w = code[j], op = w_op(w), a = w_arg(w);
                std::string x = "x" + std::to_string(j);
                if (op == NODE_LIT) o << "      const T " << x << " = s.lit[" << a << "];\n";
                else if (op == NODE_VAR) o << "      const T " << x << " = s.lo[" << a << "];\n";
                else {
                    std::string l = "x" + std::to_string(left(j)), r = "x" + std::to_string(right(j));
                    if (op == NODE_ADD) o << "      const T " << x << " = " << l << " + " << r << ";\n";
                    else if (op == NODE_SUB) o << "      const T " << x << " = " << l << " - " << r << ";\n";
                    else if (op == NODE_MUL) o << "      const T " << x << " = " << l << " * " << r << ";\n";
                    else
                        o << "      if (" << r << " == T(0)) return false; const T " << x << " = "
                          << (op == NODE_DIV ? "cdiv(" : "cmod(") << l << ", " << r << ");\n";
                }
            }
            static const char* ops[] = {"<", "<=", "==", ">=", ">"};
            o << "      if (!(x" << lr << " " << ops[rel] << " x" << rr << ")) return false;\n    }\n";
        }
        o << "    return true;\n  }\n";
    }

    std::string source(const std::string& kname) {
        o << "#include \"jit_lane.cuh\"\nnamespace oob {\nstruct Cls {\n";
        o << "  typedef " << (bits == 32 ? "int" : (bits == 128 ? "__int128" : "long long"))
          << " T;\n  typedef Arith<T> A;\n  typedef Ext<T> X;\n";
        o << "  static constexpr uint32_t NV = " << nv << ", NCON = " << ncon << ", NCODE = " << ncode
          << ", NLIT = " << nlit << ";\n";
        for (int half = 0; half < 2; half++) {
            o << "  static __device__ __forceinline__ uint64_t M" << half << "(uint32_t v) {\n    switch (v) {\n";
            for (uint32_t v = 0; v < nv; v++) {
                uint64_t m = ((uint64_t)member[4 * v + 2 * half + 1] << 32) | member[4 * v + 2 * half];
                o << "    case " << v << ": return " << m << "ull;\n";
            }
            o << "    default: return 0ull;\n    }\n  }\n";
        }
        for (uint32_t k = 0; k < ncon; k++) prop(k);
        o << "  template <class L> static __device__ __forceinline__ void pass(L& s, bool& dead) {\n";
        for (uint32_t k = 0; k < ncon; k++)
            o << "    if (!s.is_clean(" << k << ") && !s.pass_constraint(" << k << ", [&]() { return prop" << k
              << "(s); })) { dead = true; return; }\n";
        o << "  }\n";
        check();
        o << "};\n}  // namespace oob\n";
        o << "extern \"C\" __global__ void __launch_bounds__(256) " << kname
          << "(oob::LaunchArgs a) { oob::jit_solve<oob::Cls>(a); }\n";
        return o.str();
    }
};

struct Entry {
    std::string key;
    std::string cubin;
    std::string log;
    bool done = false, ok = false;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    int regs = 0;
    double compile_ms = 0;
    bool from_disk = false;
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<Entry>> g_cache;

// every device header the generated source reaches (same order in both lists)
const char* kHeaderNames[] = {"types.h",      "format.h",   "wide.cuh",    "engine.cuh",
                              "frontier.cuh", "symbolic.cuh", "phases.cuh", "jit_lane.cuh"};
const char* kHeaderSrc[] = {kSrc_types_h,      kSrc_format_h,     kSrc_wide_cuh,   kSrc_engine_cuh,
                            kSrc_frontier_cuh, kSrc_symbolic_cuh, kSrc_phases_cuh, kSrc_jit_lane_cuh};
constexpr int kNumHeaders = sizeof(kHeaderNames) / sizeof(kHeaderNames[0]);
static_assert(sizeof(kHeaderSrc) == sizeof(kHeaderNames), "one source per header name");

// On-disk cubin cache shared by the processes of a box (one per GPU under
// torchrun compile the same classes): $SCUBA_OOB_JIT_CACHE, else
// $HOME/.cache/scuba_oob_jit; "0" disables it.  The file name is a hash of the
// complete NVRTC input (generated source, every embedded header, options), so
// a stale entry can never be picked up; files are written to a temporary name
// and renamed (atomic on one file system).
std::string cache_dir() {
    static const std::string d = [] {
        const char* e = std::getenv("SCUBA_OOB_JIT_CACHE");
        if (e && std::string(e) == "0") return std::string();
        if (e && *e) return std::string(e);
        const char* h = std::getenv("HOME");
        return h && *h ? std::string(h) + "/.cache/scuba_oob_jit" : std::string();
    }();
    return d;
}
uint64_t fnv(const std::string& x, uint64_t h = 1469598103934665603ull) {
    for (unsigned char ch : x) {
        h ^= ch;
        h *= 1099511628211ull;
    }
    return h;
}
std::string cache_path(const std::string& src, const std::string& opts) {
    const std::string d = cache_dir();
    if (d.empty()) return "";
    uint64_t h = fnv(src);
    for (const char* hs : kHeaderSrc) h = fnv(hs, h);
    h = fnv(opts, h);
    int maj = 0, min = 0;
    nvrtcVersion(&maj, &min);
    h = fnv(std::to_string(maj) + "." + std::to_string(min), h);
    char name[64];
    std::snprintf(name, sizeof name, "/%016llx.cubin", (unsigned long long)h);
    return d + name;
}
bool read_file(const std::string& path, std::string& out) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    std::fseek(f, 0, SEEK_END);
    long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    out.resize(n > 0 ? (size_t)n : 0);
    bool ok = n > 0 && std::fread(&out[0], 1, (size_t)n, f) == (size_t)n;
    std::fclose(f);
    return ok;
}
void write_file(const std::string& path, const std::string& data) {
    const std::string dir = path.substr(0, path.rfind('/'));
    std::string cmd_dir = dir;
    for (size_t i = 1; i <= cmd_dir.size(); i++)  // mkdir -p
        if (i == cmd_dir.size() || cmd_dir[i] == '/') ::mkdir(cmd_dir.substr(0, i).c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string((unsigned long long)::getpid());
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;
    bool ok = std::fwrite(data.data(), 1, data.size(), f) == data.size();
    ok = (std::fclose(f) == 0) && ok;
    if (ok) std::rename(tmp.c_str(), path.c_str());
    else std::remove(tmp.c_str());
}

std::string compile_entry(Entry& e, const JitClass& c) {
    Gen g;
    g.cons = c.words;
    g.code = c.words + c.ncon;
    g.member = c.words + c.ncon + c.ncode;
    g.nv = c.nv;
    g.ncon = c.ncon;
    g.ncode = c.ncode;
    g.nlit = c.nlit;
    g.bits = c.bits;
    std::string src = g.source("oob_jit_solve");
    auto t0 = std::chrono::steady_clock::now();
    static const char* maxreg_env = std::getenv("SCUBA_OOB_JIT_MAXREG");
    const std::string cpath = cache_path(src, maxreg_env ? maxreg_env : "");
    if (!cpath.empty() && read_file(cpath, e.cubin)) {
        e.from_disk = true;
        e.compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return "";
    }
    // one compiler per class per box: the ranks of a torchrun job compile the
    // same classes at the same moment; the first takes `<cubin>.lock`, the
    // others wait for its cubin (a lock older than 120 s is presumed dead)
    int lock_fd = -1;
    if (!cpath.empty()) {
        const std::string dir = cpath.substr(0, cpath.rfind('/'));
        for (size_t i = 1; i <= dir.size(); i++)  // mkdir -p
            if (i == dir.size() || dir[i] == '/') ::mkdir(dir.substr(0, i).c_str(), 0755);
        const std::string lpath = cpath + ".lock";
        for (int waited = 0;; waited += 50) {
            lock_fd = ::open(lpath.c_str(), O_CREAT | O_EXCL | O_WRONLY, 0644);
            if (lock_fd >= 0) break;
            if (read_file(cpath, e.cubin)) {
                e.from_disk = true;
                e.compile_ms =
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                return "";
            }
            struct stat st;
            if (waited > 120000 || (::stat(lpath.c_str(), &st) == 0 && ::time(nullptr) - st.st_mtime > 120)) {
                std::remove(lpath.c_str());  // stale
                waited = 0;
                continue;
            }
            if (errno != EEXIST) break;  // no lock possible here: just compile
            ::usleep(50000);
        }
    }
    struct LockRelease {
        int fd;
        std::string path;
        ~LockRelease() {
            if (fd >= 0) {
                ::close(fd);
                std::remove(path.c_str());
            }
        }
    } lock_release{lock_fd, cpath + ".lock"};
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "oob_jit_class.cu", kNumHeaders, kHeaderSrc, kHeaderNames) !=
        NVRTC_SUCCESS)
        return "nvrtcCreateProgram failed";
    std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-DOOB_JIT=1",
                                     "--device-int128"};
    static const std::string maxreg = [] {  // SCUBA_OOB_JIT_MAXREG: register cap (occupancy experiments)
        const char* e = std::getenv("SCUBA_OOB_JIT_MAXREG");
        return (e && *e) ? std::string("--maxrregcount=") + e : std::string();
    }();
    if (!maxreg.empty()) opts.push_back(maxreg.c_str());
    nvrtcResult r = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
    size_t logn = 0;
    nvrtcGetProgramLogSize(prog, &logn);
    e.log.resize(logn);
    if (logn) nvrtcGetProgramLog(prog, &e.log[0]);
    if (r != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        return "NVRTC: " + e.log.substr(0, 2000);
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    e.cubin.resize(n);
    nvrtcGetCUBIN(prog, &e.cubin[0]);
    nvrtcDestroyProgram(&prog);
    if (!cpath.empty()) write_file(cpath, e.cubin);
    e.compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return "";
}

}  // namespace

std::string jit_key(const JitClass& c) {
    std::string k((const char*)c.words, (size_t)(c.ncon + c.ncode + 4 * c.nv) * 4);
    uint32_t dims[5] = {c.nv, c.ncon, c.ncode, c.nlit, (uint32_t)c.bits};
    k.append((const char*)dims, sizeof dims);
    return k;
}

std::string jit_prepare(const std::vector<JitClass>& classes, std::vector<const void*>& kernels,
                        std::vector<int>& regs, double* compile_ms, bool load) {
    kernels.assign(classes.size(), nullptr);
    regs.assign(classes.size(), 0);
    std::vector<std::shared_ptr<Entry>> ents(classes.size());
    std::vector<size_t> todo;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (size_t i = 0; i < classes.size(); i++) {
            std::string k = jit_key(classes[i]);
            auto it = g_cache.find(k);
            if (it == g_cache.end()) {
                auto e = std::make_shared<Entry>();
                e->key = k;
                it = g_cache.emplace(k, e).first;
                todo.push_back(i);
            }
            ents[i] = it->second;
        }
    }
    // compile the new classes in parallel (NVRTC is thread-safe)
    std::vector<std::string> errs(classes.size());
    {
        std::atomic<size_t> next{0};
        unsigned nt = std::max(1u, std::min<unsigned>(16u, std::thread::hardware_concurrency()));
        nt = std::min<unsigned>(nt, (unsigned)std::max<size_t>(1, todo.size()));
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; t++)
            th.emplace_back([&]() {
                for (;;) {
                    size_t x = next.fetch_add(1);
                    if (x >= todo.size()) break;
                    size_t i = todo[x];
                    Entry& e = *ents[i];
                    errs[i] = compile_entry(e, classes[i]);
                    e.ok = errs[i].empty();
                    e.done = true;
                }
            });
        for (auto& t : th) t.join();
    }
    double total = 0;
    for (size_t i = 0; i < classes.size(); i++) {
        Entry& e = *ents[i];
        std::lock_guard<std::mutex> lk(g_mu);
        if (!e.done) return "JIT entry not compiled (concurrent compile in progress)";
        if (!e.ok) {
            g_cache.erase(e.key);
            return errs[i].empty() ? "JIT compile failed earlier: " + e.log.substr(0, 500) : errs[i];
        }
        total += e.compile_ms;
        if (!load) continue;
        if (!e.kernel) {
            cudaError_t ce = cudaLibraryLoadData(&e.lib, e.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
            if (ce != cudaSuccess) return std::string("cudaLibraryLoadData: ") + cudaGetErrorString(ce);
            ce = cudaLibraryGetKernel(&e.kernel, e.lib, "oob_jit_solve");
            if (ce != cudaSuccess) return std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(ce);
            cudaFuncAttributes fa{};
            if (cudaFuncGetAttributes(&fa, (const void*)e.kernel) == cudaSuccess) e.regs = fa.numRegs;
            else cudaGetLastError();
        }
        kernels[i] = (const void*)e.kernel;
        regs[i] = e.regs;
    }
    if (compile_ms) *compile_ms = total;
    return "";
}

std::string jit_source(const JitClass& c) {
    Gen g;
    g.cons = c.words;
    g.code = c.words + c.ncon;
    g.member = c.words + c.ncon + c.ncode;
    g.nv = c.nv;
    g.ncon = c.ncon;
    g.ncode = c.ncode;
    g.nlit = c.nlit;
    g.bits = c.bits;
    return g.source("oob_jit_solve");
}

}  // namespace oob
