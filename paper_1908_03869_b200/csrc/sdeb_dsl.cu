// Expression templates -> CUDA -> NVRTC (see sdeb_dsl.h).
#include "sdeb_dsl.h"

#include <nvrtc.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <vector>

namespace {

// ---- tokens -----------------------------------------------------------------

struct Tok {
    enum Kind { NUM, NAME, OP, END } kind;
    std::string text;
    int line, col;
};

struct SyntaxError {
    std::string msg;
    int line, col;
};

std::vector<Tok> lex(const std::string& s) {
    std::vector<Tok> out;
    int line = 1, col = 1;
    size_t k = 0;
    auto adv = [&](size_t n) {
        for (size_t q = 0; q < n; ++q) {
            if (s[k + q] == '\n') {
                ++line;
                col = 1;
            } else {
                ++col;
            }
        }
        k += n;
    };
    while (k < s.size()) {
        const char c = s[k];
        if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
            adv(1);
            continue;
        }
        if (std::isdigit((unsigned char)c) || (c == '.' && k + 1 < s.size() && std::isdigit((unsigned char)s[k + 1]))) {
            size_t e = k;
            while (e < s.size() && std::isdigit((unsigned char)s[e])) ++e;
            if (e < s.size() && s[e] == '.') {
                ++e;
                while (e < s.size() && std::isdigit((unsigned char)s[e])) ++e;
            }
            if (e < s.size() && (s[e] == 'e' || s[e] == 'E')) {
                size_t x = e + 1;
                if (x < s.size() && (s[x] == '+' || s[x] == '-')) ++x;
                if (x < s.size() && std::isdigit((unsigned char)s[x])) {
                    while (x < s.size() && std::isdigit((unsigned char)s[x])) ++x;
                    e = x;
                }
            }
            out.push_back({Tok::NUM, s.substr(k, e - k), line, col});
            adv(e - k);
            continue;
        }
        if (std::isalpha((unsigned char)c) || c == '_') {
            size_t e = k;
            while (e < s.size() && (std::isalnum((unsigned char)s[e]) || s[e] == '_')) ++e;
            out.push_back({Tok::NAME, s.substr(k, e - k), line, col});
            adv(e - k);
            continue;
        }
        if (std::strchr("-+*/^()[],", c)) {
            out.push_back({Tok::OP, std::string(1, c), line, col});
            adv(1);
            continue;
        }
        throw SyntaxError{std::string("unexpected character '") + c + "'", line, col};
    }
    out.push_back({Tok::END, "", line, col});
    return out;
}

// ---- AST ----------------------------------------------------------------------

struct Node {
    enum Kind { NUM, VAR, INDEX, NEG, BIN, CALL, SUM } kind;
    double num = 0.0;
    std::string name;  // VAR name, INDEX base, CALL function, SUM index
    char op = 0;       // BIN operator
    std::unique_ptr<Node> a, b;
    int line = 0, col = 0;
};
using P = std::unique_ptr<Node>;

P make(Node::Kind k, const Tok& at) {
    P n(new Node);
    n->kind = k;
    n->line = at.line;
    n->col = at.col;
    return n;
}

const std::set<std::string> kFunctions = {"sin", "cos", "tan", "exp", "ln", "sqrt", "abs"};

// Precedence climbing over the grammar of dsl.py:12-19:
//   + -  (left, 1)   * /  (left, 2)   unary -  (prefix, looser than ^)
//   ^    (right, tighter than unary minus: its right operand is a unary)
class Parser {
  public:
    explicit Parser(const std::string& src) : t_(lex(src)) {}

    P parse() {
        P e = binary(1);
        if (t_[k_].kind != Tok::END) fail("unexpected trailing input");
        return e;
    }

  private:
    std::vector<Tok> t_;
    size_t k_ = 0;

    [[noreturn]] void fail(const std::string& msg) {
        throw SyntaxError{msg, t_[k_].line, t_[k_].col};
    }
    bool is_op(const char* s) const { return t_[k_].kind == Tok::OP && t_[k_].text == s; }
    void expect(const char* s) {
        if (!is_op(s)) fail(std::string("expected '") + s + "'");
        ++k_;
    }
    static int prec(const Tok& t) {
        if (t.kind != Tok::OP) return 0;
        if (t.text == "+" || t.text == "-") return 1;
        if (t.text == "*" || t.text == "/") return 2;
        return 0;
    }

    P binary(int min_prec) {
        P lhs = prefix();
        for (;;) {
            const int p = prec(t_[k_]);
            if (p == 0 || p < min_prec) return lhs;
            const Tok op = t_[k_++];
            P rhs = binary(p + 1);
            P n = make(Node::BIN, op);
            n->op = op.text[0];
            n->a = std::move(lhs);
            n->b = std::move(rhs);
            lhs = std::move(n);
        }
    }

    P prefix() {
        if (is_op("-")) {
            const Tok at = t_[k_++];
            P n = make(Node::NEG, at);
            n->a = prefix();
            return n;
        }
        P base = atom();
        if (is_op("^")) {
            const Tok at = t_[k_++];
            P n = make(Node::BIN, at);
            n->op = '^';
            n->a = std::move(base);
            n->b = prefix();
            return n;
        }
        return base;
    }

    P atom() {
        const Tok tok = t_[k_];
        if (tok.kind == Tok::NUM) {
            ++k_;
            P n = make(Node::NUM, tok);
            n->num = std::strtod(tok.text.c_str(), nullptr);
            return n;
        }
        if (is_op("(")) {
            ++k_;
            P e = binary(1);
            expect(")");
            return e;
        }
        if (tok.kind != Tok::NAME) fail("expected a number, name or parenthesised expression");
        ++k_;
        if (is_op("[")) {
            if (tok.text != "y" && tok.text != "p" && tok.text != "n")
                throw SyntaxError{"only y, p and n can be indexed", tok.line, tok.col};
            ++k_;
            P n = make(Node::INDEX, tok);
            n->name = tok.text;
            n->a = binary(1);
            expect("]");
            return n;
        }
        if (is_op("(")) {
            ++k_;
            if (tok.text == "sum") {
                if (t_[k_].kind != Tok::NAME) fail("sum(index, body) expects an index name first");
                P n = make(Node::SUM, tok);
                n->name = t_[k_++].text;
                expect(",");
                n->a = binary(1);
                expect(")");
                return n;
            }
            if (!kFunctions.count(tok.text))
                throw SyntaxError{"unknown function '" + tok.text + "'", tok.line, tok.col};
            P n = make(Node::CALL, tok);
            n->name = tok.text;
            n->a = binary(1);
            expect(")");
            return n;
        }
        P n = make(Node::VAR, tok);
        n->name = tok.text;
        return n;
    }
};

// ---- CUDA code generation ------------------------------------------------------

struct GenError {
    std::string msg;
    int line, col;
};

std::string literal(double v) {
    char buf[64];
    if (!std::isfinite(v)) {
        uint64_t bits;
        std::memcpy(&bits, &v, sizeof(bits));
        std::snprintf(buf, sizeof(buf), "__longlong_as_double(0x%016llxll)", (unsigned long long)bits);
        return buf;
    }
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    std::string s = buf;
    if (s.find_first_of(".eE") == std::string::npos) s += ".0";
    return "(" + s + ")";
}

class Gen {
  public:
    explicit Gen(bool has_noise) : has_noise_(has_noise) {}
    bool used_sum = false;

    // Double-valued expression (dsl.py _Evaluator.eval).
    std::string num(const Node& n) {
        switch (n.kind) {
            case Node::NUM:
                return literal(n.num);
            case Node::VAR:
                if (n.name == "t") return "t";
                if (n.name == "N") return "kDslN";
                if (n.name == "i") return "double(i)";
                if (scope_.count(n.name)) return "double(s_" + n.name + ")";
                throw GenError{"unknown variable '" + n.name + "'", n.line, n.col};
            case Node::INDEX: {
                if (n.name == "n" && !has_noise_)
                    throw GenError{"noise n[...] cannot appear in a drift expression", n.line, n.col};
                const std::string arr = n.name == "y" ? "y" : (n.name == "p" ? "p" : "n");
                return arr + "[" + index(*n.a) + "]";
            }
            case Node::NEG:
                return "(-" + num(*n.a) + ")";
            case Node::BIN: {
                if (n.op == '^') {
                    // np.power; x^2 is the correctly rounded square either way
                    if (n.b->kind == Node::NUM && n.b->num == 2.0) return "dsl_sq(" + num(*n.a) + ")";
                    return "pow(" + num(*n.a) + ", " + num(*n.b) + ")";
                }
                const char* fn = n.op == '+' ? "__dadd_rn" : n.op == '-' ? "__dsub_rn"
                               : n.op == '*' ? "__dmul_rn" : "__ddiv_rn";
                return std::string(fn) + "(" + num(*n.a) + ", " + num(*n.b) + ")";
            }
            case Node::CALL: {
                const std::string x = num(*n.a);
                if (n.name == "sin") return "dsl_sin<EXACT>(" + x + ", big)";
                if (n.name == "cos") return "dsl_cos<EXACT>(" + x + ", big)";
                if (n.name == "tan") return "tan(" + x + ")";
                if (n.name == "exp") return "exp(" + x + ")";
                if (n.name == "ln") return "log(" + x + ")";
                if (n.name == "sqrt") return "__dsqrt_rn(" + x + ")";
                return "fabs(" + x + ")";
            }
            case Node::SUM: {
                if (scope_.count(n.name) || n.name == "t" || n.name == "N" || n.name == "i")
                    throw GenError{"sum index '" + n.name + "' shadows a name in scope", n.line, n.col};
                scope_.insert(n.name);
                used_sum = true;
                const std::string body = num(*n.a);
                scope_.erase(n.name);
                return "dsl_sum([&](int s_" + n.name + ") -> double { return " + body + "; })";
            }
        }
        throw GenError{"bad node", n.line, n.col};
    }

    // Integer index sub-expression (dsl.py _index_value): literals, i, N, sum
    // indices and + - * only.
    std::string index(const Node& n) {
        switch (n.kind) {
            case Node::NUM: {
                if (n.num != std::floor(n.num) || std::fabs(n.num) > 1e15)
                    throw GenError{"non-integer constant in index expression", n.line, n.col};
                char buf[32];
                std::snprintf(buf, sizeof(buf), "%lld", (long long)n.num);
                return buf;
            }
            case Node::VAR:
                if (n.name == "i") return "i";
                if (n.name == "N") return "SDB_N";
                if (scope_.count(n.name)) return "s_" + n.name;
                throw GenError{"unknown variable '" + n.name + "' in index expression", n.line, n.col};
            case Node::NEG:
                return "(-" + index(*n.a) + ")";
            case Node::BIN:
                if (n.op == '+' || n.op == '-' || n.op == '*')
                    return "(" + index(*n.a) + " " + n.op + " " + index(*n.b) + ")";
                throw GenError{std::string("operator '") + n.op + "' not allowed in index expressions",
                               n.line, n.col};
            default:
                throw GenError{"index expressions must be integer arithmetic", n.line, n.col};
        }
    }

  private:
    bool has_noise_;
    std::set<std::string> scope_;
};

bool gen_function(const std::string& text, bool diffusion, std::string* out, std::string* err,
                  bool* used_sum) {
    try {
        Parser ps(text);
        P root = ps.parse();
        Gen g(diffusion);
        const std::string body = g.num(*root);
        *used_sum = *used_sum || g.used_sum;
        if (diffusion) {
            *out = "template <bool EXACT>\n"
                   "__device__ __forceinline__ double sdeb::sdb_diffusion(int i, double t, "
                   "const DVec& y, const double* __restrict__ p, const DVec& n, bool& big) {\n"
                   "    (void)i; (void)t; (void)y; (void)p; (void)n; (void)big;\n"
                   "    return " + body + ";\n}\n";
        } else {
            *out = "template <bool EXACT>\n"
                   "__device__ __forceinline__ double sdeb::sdb_drift(int i, double t, "
                   "const DVec& y, const double* __restrict__ p, bool& big) {\n"
                   "    (void)i; (void)t; (void)y; (void)p; (void)big;\n    return " + body + ";\n}\n";
        }
        return true;
    } catch (const SyntaxError& e) {
        char buf[64];
        std::snprintf(buf, sizeof(buf), "line %d, column %d: ", e.line, e.col);
        *err = std::string(diffusion ? "diffusion: " : "drift: ") + buf + e.msg;
    } catch (const GenError& e) {
        char buf[64];
        std::snprintf(buf, sizeof(buf), "line %d, column %d: ", e.line, e.col);
        *err = std::string(diffusion ? "diffusion: " : "drift: ") + buf + e.msg;
    }
    return false;
}

// Headers the generated programs include, embedded at build time
// (_build.py writes sdeb_rtc_headers.inc from csrc/).
struct RtcHeader {
    const char* name;
    const char* text;
};
#include "sdeb_rtc_headers.inc"

}  // namespace

sdb_model::~sdb_model() {
    for (auto& kv : programs)
        if (kv.second.lib) cudaLibraryUnload(kv.second.lib);
}

namespace sdeb_dsl {

int state_words(const sdb_model* m) {
    const int nb = (m->nnoise + 3) / 4;
    return m->nequat + (m->nnoise > 0 ? 4 * nb : 0);
}

// Stage the sincos / log tables in shared memory unless the templates carry
// sums: there the O(N^2) table reads per step compete with the state-column
// reads for the shared-memory pipe (measured: Kuramoto templates 2.44e9 ->
// 1.53e9 orbit-steps/s staged; the OU template 1.94e10 -> 2.26e10).
bool stage_tables(const sdb_model* m) { return !m->uses_sum; }

int lanes_for(const sdb_model* m) {
    if (const char* e = std::getenv("SDEB200_DSL_LANES")) {
        const int v = std::atoi(e);
        if (v >= 1 && v <= 32 && (v & (v - 1)) == 0) return v;
    }
    const int per_lane = m->uses_sum ? 4 : 16;
    const int want = (m->nequat + per_lane - 1) / per_lane;
    int l = 1;
    while (l < want && l < 32) l <<= 1;
    return l;
}

// the columns of a CTA's 128 / lanes orbits must fit the 96 KB opt-in
bool global_state(const sdb_model* m, int lanes) {
    return size_t(state_words(m)) * 8 * size_t(kBlock / lanes) > size_t(kSmemMax);
}

size_t scratch_doubles(const sdb_model* m, int lanes, int64_t rows) {
    if (!global_state(m, lanes)) return 0;
    const int64_t slots = kBlock / lanes;
    return size_t(state_words(m)) * size_t((rows + slots - 1) / slots * slots);
}

bool generate(sdb_model* m, std::string* err) {
    m->uses_sum = false;
    return gen_function(m->drift_text, false, &m->drift_cu, err, &m->uses_sum) &&
           gen_function(m->diffusion_text, true, &m->diffusion_cu, err, &m->uses_sum);
}

std::string program_source(const sdb_model* m, int kind, int lanes) {
    // unrolled equation loops keep f / g / RK4 stages in registers; the
    // unrolled model code grows as (N / lanes) x (drift evaluations per
    // step), and ptxas time with it, so larger systems run the loops rolled
    // (stack arrays)
    const int epl = (m->nequat + lanes - 1) / lanes;
    const int evals = (kind == sdeb::DK_RUN_RK4 || kind == sdeb::DK_STEP_RK4) ? 4
                      : (kind <= sdeb::DK_RUN_XOSHIRO || kind == sdeb::DK_STEP_EM) ? 2 : 1;
    const int unroll = epl * evals <= kUnrollWork ? epl : 1;
    char head[360];
    std::snprintf(head, sizeof(head),
                  "#define SDB_N %d\n#define SDB_NP %d\n#define SDB_NN %d\n#define SDB_KIND %d\n"
                  "#define SDB_LANES %d\n#define SDB_UNROLL %d\n#define SDB_GLOBAL_STATE %d\n%s",
                  m->nequat, m->nparams, m->nnoise, kind, lanes, unroll,
                  global_state(m, lanes) ? 1 : 0,
                  stage_tables(m) ? "#define SDEB_SMEM_TABLES 1\n" : "");
    return std::string("// generated by sdeb200 from expression templates\n") + head +
           "#include \"sdeb_dsl_kernel.cuh\"\n\n// drift: " + m->drift_text + "\n" + m->drift_cu +
           "\n// diffusion: " + m->diffusion_text + "\n" + m->diffusion_cu;
}

namespace {

// NVRTC: generated source -> sm_100a cubin.
cudaError_t nvrtc_cubin(const sdb_model* m, int kind, int lanes, std::vector<char>* cubin,
                        std::string* log, std::string* err) {
    const std::string src = program_source(m, kind, lanes);
    nvrtcProgram prog;
    std::vector<const char*> names, texts;
    for (const RtcHeader& h : kRtcHeaders) {
        names.push_back(h.name);
        texts.push_back(h.text);
    }
    nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), "sdb_model.cu", int(names.size()),
                                       texts.data(), names.data());
    if (r != NVRTC_SUCCESS) {
        *err = std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r);
        return cudaErrorInvalidSource;
    }
    const char* opts[] = {"-arch=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo"};
    r = nvrtcCompileProgram(prog, int(sizeof(opts) / sizeof(opts[0])), opts);
    size_t log_size = 0;
    nvrtcGetProgramLogSize(prog, &log_size);
    std::string text(log_size, '\0');
    if (log_size) nvrtcGetProgramLog(prog, &text[0]);
    *log = text;
    if (r != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        *err = std::string("NVRTC compile failed: ") + nvrtcGetErrorString(r) + "\n" + text;
        return cudaErrorInvalidSource;
    }
    size_t cubin_size = 0;
    nvrtcGetCUBINSize(prog, &cubin_size);
    cubin->resize(cubin_size);
    nvrtcGetCUBIN(prog, cubin->data());
    nvrtcDestroyProgram(&prog);
    return cudaSuccess;
}

cudaError_t compile(sdb_model* m, int kind, int lanes, sdb_model::Program* out, std::string* err) {
    std::vector<char> cubin;
    cudaError_t e = nvrtc_cubin(m, kind, lanes, &cubin, &out->log, err);
    if (e != cudaSuccess) return e;
    e = cudaLibraryLoadData(&out->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&out->kernel, out->lib, "sdb_dsl_main");
    if (e != cudaSuccess) *err = std::string("loading the compiled program: ") + cudaGetErrorString(e);
    return e;
}

}  // namespace

cudaError_t compile_only(sdb_model* m, int kind, int lanes, std::string* err) {
    std::vector<char> cubin;
    std::string log;
    cudaError_t e = nvrtc_cubin(m, kind, lanes, &cubin, &log, err);
    std::lock_guard<std::mutex> lock(m->mu);
    m->error = e == cudaSuccess ? log : *err;
    return e;
}

cudaError_t kernel_for(sdb_model* m, int kind, int lanes, cudaKernel_t* out, std::string* err) {
    std::lock_guard<std::mutex> lock(m->mu);
    const int key = kind + 64 * lanes;
    auto it = m->programs.find(key);
    if (it == m->programs.end()) {
        sdb_model::Program prog;
        cudaError_t e = compile(m, kind, lanes, &prog, err);
        if (e != cudaSuccess) return e;
        it = m->programs.emplace(key, prog).first;
    }
    *out = it->second.kernel;
    return cudaSuccess;
}

cudaError_t launch(sdb_model* m, int kind, const sdeb::DslArgs& a, cudaStream_t st,
                   std::string* err) {
    const int lanes = lanes_for(m);
    cudaKernel_t k = nullptr;
    cudaError_t e = kernel_for(m, kind, lanes, &k, err);
    if (e != cudaSuccess) return e;
    if (a.rows <= 0) return cudaSuccess;
    const int64_t slots = kBlock / lanes;
    size_t smem = 0;
    if (global_state(m, lanes)) {
        if (!a.scratch) {
            *err = "expression-template program needs a global scratch buffer";
            return cudaErrorInvalidValue;
        }
    } else {
        smem = size_t(slots) * state_words(m) * sizeof(double);
    }
    // the staged math tables are static shared memory on top of the columns
    if (smem + (stage_tables(m) ? kTableSmem : 0) > 48 * 1024) {
        e = cudaFuncSetAttribute(reinterpret_cast<const void*>(k),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) {
            *err = std::string("shared-memory opt-in: ") + cudaGetErrorString(e);
            return e;
        }
    }
    const dim3 grid(unsigned((a.rows + slots - 1) / slots)), block(kBlock);
    sdeb::DslArgs copy = a;
    void* args[] = {&copy};
    e = cudaLaunchKernel(reinterpret_cast<const void*>(k), grid, block, args, smem, st);
    if (e != cudaSuccess) *err = std::string("expression-template kernel launch: ") + cudaGetErrorString(e);
    return e;
}

}  // namespace sdeb_dsl
