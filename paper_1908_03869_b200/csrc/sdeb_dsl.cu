// Expression templates -> CUDA -> NVRTC (see sdeb_dsl.h).
#include "sdeb_dsl.h"
#include "sdeb_log_table.cuh"
#include "sdeb_sincos_table.cuh"

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

// Does `n` read variable `v` (sum indices shadow)?
bool uses(const Node& n, const std::string& v) {
    switch (n.kind) {
        case Node::NUM: return false;
        case Node::VAR: return n.name == v;
        case Node::SUM: return n.name != v && uses(*n.a, v);
        case Node::BIN: return uses(*n.a, v) || uses(*n.b, v);
        default: return uses(*n.a, v);  // INDEX, NEG, CALL
    }
}

P clone(const Node& n) {
    P c(new Node);
    c->kind = n.kind;
    c->num = n.num;
    c->name = n.name;
    c->op = n.op;
    c->line = n.line;
    c->col = n.col;
    if (n.a) c->a = clone(*n.a);
    if (n.b) c->b = clone(*n.b);
    return c;
}

// `other` is `jside` with sum index j replaced by the equation index i
// (e.g. y[i] against y[j]): the equation's angle is one of the j-terms.
bool same_at_i(const Node& other, const Node& jside, const std::string& j) {
    if (jside.kind == Node::VAR && jside.name == j) return other.kind == Node::VAR && other.name == "i";
    if (other.kind != jside.kind || other.name != jside.name || other.op != jside.op) return false;
    if (jside.kind == Node::NUM) return other.num == jside.num;
    if (jside.kind == Node::SUM && jside.name == j) return false;  // shadowed: keep it simple
    if (bool(other.a) != bool(jside.a) || bool(other.b) != bool(jside.b)) return false;
    if (jside.a && !same_at_i(*other.a, *jside.a, j)) return false;
    if (jside.b && !same_at_i(*other.b, *jside.b, j)) return false;
    return true;
}

class Gen {
  public:
    // factor: rewrite sum(j, sin|cos(A_j - B)) with the addition formulas so
    // the j-sums no longer depend on the equation (meanfield form, changes
    // rounding by a few ulp); hoisting of equation-independent sums is always
    // on (bit-identical: the same value for every equation).
    Gen(bool has_noise, bool factor, int n) : has_noise_(has_noise), factor_(factor), n_(n) {}
    bool used_sum = false;
    bool eq_sum = false;               // a sum is still evaluated per equation
    std::vector<std::string> hoisted;  // prologue statements H[k] = ...

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
                used_sum = true;
                if (factor_) {
                    std::string f;
                    if (factored(n, &f)) return f;
                }
                const bool hoist = hoistable(n);
                std::set<std::string> saved;
                if (hoist) saved.swap(scope_);  // the prologue sees no enclosing sums
                scope_.insert(n.name);
                const std::string body = num(*n.a);
                scope_.erase(n.name);
                const std::string code =
                    "dsl_sum([&](int s_" + n.name + ") -> double { return " + body + "; })";
                if (!hoist) {
                    eq_sum = true;
                    return code;
                }
                scope_.swap(saved);
                return hoist_value(code);
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
    bool has_noise_, factor_;
    int n_;  // equation count (kept-term slots)
    std::set<std::string> scope_;

    // Same value for every equation: reads neither i nor an enclosing sum index.
    bool hoistable(const Node& sum) const {
        if (uses(sum, "i")) return false;
        for (const std::string& v : scope_)
            if (uses(sum, v)) return false;
        return true;
    }

    std::string hoist_value(const std::string& code) {
        const std::string ref = "H[" + std::to_string(hoisted.size()) + "]";
        hoisted.push_back(ref + " = " + code + ";");
        return ref;
    }

    // sum(j, sin(A - B)) / sum(j, cos(A - B)) with exactly one side reading j
    // (and that side free of i and enclosing sums): the addition formulas turn
    // it into two equation-independent sums of sin / cos of the j-side, done
    // in one pass (one sincos per term) and hoisted.
    bool factored(const Node& sum, std::string* out) {
        const Node& body = *sum.a;
        if (body.kind != Node::CALL || (body.name != "sin" && body.name != "cos")) return false;
        const Node& arg = *body.a;
        if (arg.kind != Node::BIN || arg.op != '-') return false;
        const std::string& j = sum.name;
        const bool ja = uses(*arg.a, j), jb = uses(*arg.b, j);
        if (ja == jb) return false;
        const Node& jside = ja ? *arg.a : *arg.b;
        const Node& other = ja ? *arg.b : *arg.a;
        if (uses(jside, "i")) return false;
        for (const std::string& v : scope_)
            if (uses(jside, v)) return false;
        // the j-side's sums of sin and cos, one pass
        std::set<std::string> saved;
        saved.swap(scope_);
        scope_.insert(j);
        const std::string term = num(jside);
        scope_.erase(j);
        scope_.swap(saved);
        const size_t k = hoisted.size();
        const std::string hs = "H[" + std::to_string(k) + "]", hc = "H[" + std::to_string(k + 1) + "]";
        std::string so, co;
        if (same_at_i(other, jside, j)) {
            // the equation's angle is the j-term at j = i: keep every term's
            // (sin, cos) from the pass (H[k+2 ..], H[k+2+N ..]) instead of a
            // second sincos per equation
            const std::string ks = std::to_string(k + 2), kc = std::to_string(k + 2) + " + SDB_N";
            hoisted.push_back("dsl_sum_sincos_keep<EXACT>([&](int s_" + j + ") -> double { return " +
                              term + "; }, big, " + hs + ", " + hc + ", &H[" + ks + "], &H[" + kc +
                              "]);");
            for (int q = 0; q < 1 + 2 * n_; ++q) hoisted.push_back("");  // H[k+1], kept terms
            so = "H[" + ks + " + i]";
            co = "H[" + kc + " + i]";
        } else {
            hoisted.push_back("dsl_sum_sincos<EXACT>([&](int s_" + j + ") -> double { return " +
                              term + "; }, big, " + hs + ", " + hc + ");");
            hoisted.push_back("");  // the slot H[k+1] is written by the same statement
            const std::string o = num(other);  // the equation-side angle
            so = "dsl_sin<EXACT>(" + o + ", big)";
            co = "dsl_cos<EXACT>(" + o + ", big)";
        }
        // A = j-side, B = other.  sin(A-B) = sinA cosB - cosA sinB; sin(B-A) = -(...)
        // cos(A-B) = cos(B-A) = cosA cosB + sinA sinB
        if (body.name == "cos") {
            *out = "__dadd_rn(__dmul_rn(" + hc + ", " + co + "), __dmul_rn(" + hs + ", " + so + "))";
        } else if (ja) {
            *out = "__dsub_rn(__dmul_rn(" + hs + ", " + co + "), __dmul_rn(" + hc + ", " + so + "))";
        } else {
            *out = "__dsub_rn(__dmul_rn(" + so + ", " + hc + "), __dmul_rn(" + co + ", " + hs + "))";
        }
        return true;
    }
};

// Device functions of one template: a prologue computing the equation-
// independent (hoisted) values H[] once per evaluation, and the per-equation
// function reading them.
bool gen_function(const std::string& text, bool diffusion, bool factor, int n, std::string* out,
                  int* nhoist, std::string* err, bool* eq_sum) {
    try {
        Parser ps(text);
        P root = ps.parse();
        Gen g(diffusion, factor, n);
        const std::string body = g.num(*root);
        *eq_sum = *eq_sum || g.eq_sum;
        const std::string name = diffusion ? "diffusion" : "drift";
        const std::string hn = diffusion ? "SDB_DIFF_H" : "SDB_DRIFT_H";
        const std::string params = diffusion
            ? "const DVec& y, const double* __restrict__ p, const DVec& n, bool& big"
            : "const DVec& y, const double* __restrict__ p, bool& big";
        const std::string unused = diffusion ? "(void)t; (void)y; (void)p; (void)n; (void)big;"
                                             : "(void)t; (void)y; (void)p; (void)big;";
        std::string pro;
        for (const std::string& st : g.hoisted)
            if (!st.empty()) pro += "    " + st + "\n";
        *nhoist = int(std::max<size_t>(1, g.hoisted.size()));
        *out = "template <bool EXACT>\n"
               "__device__ __forceinline__ void sdeb::sdb_" + name + "_pre(double t, " + params +
               ", double (&H)[" + hn + "]) {\n    " + unused + " (void)H;\n" + pro + "}\n"
               "template <bool EXACT>\n"
               "__device__ __forceinline__ double sdeb::sdb_" + name + "(int i, double t, " + params +
               ", const double (&H)[" + hn + "]) {\n    (void)i; " + unused + " (void)H;\n"
               "    return " + body + ";\n}\n";
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

static_assert(kTableSmem == 16 * (sdeb::kSinCosN + (1 << sdeb::kLogTableBits)),
              "kTableSmem must match the staged tables (sdeb_math.cuh)");

int state_words(const sdb_model* m) {
    const int nb = (m->nnoise + 3) / 4;
    return m->nequat + (m->nnoise > 0 ? 4 * nb : 0);
}

// Stage the sincos / log tables in shared memory unless the templates carry
// sums: there the O(N^2) table reads per step compete with the state-column
// reads for the shared-memory pipe (measured: Kuramoto templates 2.44e9 ->
// 1.53e9 orbit-steps/s staged; the OU template 1.94e10 -> 2.26e10).
bool stage_tables(const sdb_model* m, bool factor) {
    // SDEB200_DSL_SMEM_TABLES=0/1 overrides (experiments)
    if (const char* e = std::getenv("SDEB200_DSL_SMEM_TABLES")) return std::atoi(e) != 0;
    return !m->eq_sum[factor ? 1 : 0];
}

int lanes_for(const sdb_model* m, bool factor) {
    if (const char* e = std::getenv("SDEB200_DSL_LANES")) {
        const int v = std::atoi(e);
        if (v >= 1 && v <= 32 && (v & (v - 1)) == 0) return v;
    }
    // O(N) work per equation (sums left in the equation): ~4 equations per lane;
    // O(1) (no sums, or all hoisted into the per-evaluation prologue, which
    // every lane of a group would repeat): ~16
    const int per_lane = m->eq_sum[factor ? 1 : 0] ? 4 : 16;
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
    for (int f = 0; f < 2; ++f) {
        m->eq_sum[f] = false;
        if (!gen_function(m->drift_text, false, f == 1, m->nequat, &m->drift_cu[f], &m->drift_h[f],
                          err, &m->eq_sum[f]) ||
            !gen_function(m->diffusion_text, true, f == 1, m->nequat, &m->diffusion_cu[f],
                          &m->diffusion_h[f], err, &m->eq_sum[f]))
            return false;
    }
    return true;
}

std::string program_source(const sdb_model* m, int kind, int lanes, bool factor) {
    // unrolled equation loops keep f / g / RK4 stages in registers; the
    // unrolled model code grows as (N / lanes) x (drift evaluations per
    // step), and ptxas time with it, so larger systems run the loops rolled
    // (stack arrays)
    const int epl = (m->nequat + lanes - 1) / lanes;
    const int evals = (kind == sdeb::DK_RUN_RK4 || kind == sdeb::DK_STEP_RK4) ? 4
                      : (kind <= sdeb::DK_RUN_XOSHIRO || kind == sdeb::DK_STEP_EM) ? 2 : 1;
    const int unroll = epl * evals <= kUnrollWork ? epl : 1;
    char head[420];
    std::snprintf(head, sizeof(head),
                  "#define SDB_N %d\n#define SDB_NP %d\n#define SDB_NN %d\n#define SDB_KIND %d\n"
                  "#define SDB_LANES %d\n#define SDB_UNROLL %d\n#define SDB_GLOBAL_STATE %d\n"
                  "#define SDB_DRIFT_H %d\n#define SDB_DIFF_H %d\n%s",
                  m->nequat, m->nparams, m->nnoise, kind, lanes, unroll,
                  global_state(m, lanes) ? 1 : 0, m->drift_h[factor ? 1 : 0],
                  m->diffusion_h[factor ? 1 : 0],
                  stage_tables(m, factor) ? "#define SDEB_SMEM_TABLES 1\n" : "");
    // SDEB200_DSL_MINB=b: __launch_bounds__(128, b) for the generated kernel
    // (experiments: caps registers so b CTAs fit per SM)
    std::string minb;
    if (const char* e = std::getenv("SDEB200_DSL_MINB")) minb = std::string("#define SDB_MINB ") + e + "\n";
    return std::string("// generated by sdeb200 from expression templates\n") + head + minb +
           "#include \"sdeb_dsl_kernel.cuh\"\n\n// drift: " + m->drift_text +
           (factor ? "  (sums factored)" : "") + "\n" + m->drift_cu[factor ? 1 : 0] +
           "\n// diffusion: " + m->diffusion_text + "\n" + m->diffusion_cu[factor ? 1 : 0];
}

namespace {

// NVRTC: generated source -> sm_100a cubin.
cudaError_t nvrtc_cubin(const sdb_model* m, int kind, int lanes, bool factor,
                        std::vector<char>* cubin, std::string* log, std::string* err) {
    const std::string src = program_source(m, kind, lanes, factor);
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

cudaError_t compile(sdb_model* m, int kind, int lanes, bool factor, sdb_model::Program* out,
                    std::string* err) {
    std::vector<char> cubin;
    cudaError_t e = nvrtc_cubin(m, kind, lanes, factor, &cubin, &out->log, err);
    if (e != cudaSuccess) return e;
    e = cudaLibraryLoadData(&out->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&out->kernel, out->lib, "sdb_dsl_main");
    if (e != cudaSuccess) *err = std::string("loading the compiled program: ") + cudaGetErrorString(e);
    return e;
}

}  // namespace

cudaError_t compile_only(sdb_model* m, int kind, int lanes, bool factor, std::string* err) {
    std::vector<char> cubin;
    std::string log;
    cudaError_t e = nvrtc_cubin(m, kind, lanes, factor, &cubin, &log, err);
    std::lock_guard<std::mutex> lock(m->mu);
    m->error = e == cudaSuccess ? log : *err;
    return e;
}

cudaError_t kernel_for(sdb_model* m, int kind, int lanes, bool factor, cudaKernel_t* out,
                       std::string* err) {
    std::lock_guard<std::mutex> lock(m->mu);
    const int key = kind + 64 * lanes + (factor ? 4096 : 0);
    auto it = m->programs.find(key);
    if (it == m->programs.end()) {
        sdb_model::Program prog;
        cudaError_t e = compile(m, kind, lanes, factor, &prog, err);
        if (e != cudaSuccess) return e;
        it = m->programs.emplace(key, prog).first;
    }
    *out = it->second.kernel;
    return cudaSuccess;
}

cudaError_t launch(sdb_model* m, int kind, const sdeb::DslArgs& a, cudaStream_t st,
                   std::string* err, bool factor) {
    const int lanes = lanes_for(m, factor);
    cudaKernel_t k = nullptr;
    cudaError_t e = kernel_for(m, kind, lanes, factor, &k, err);
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
    if (smem + (stage_tables(m, factor) ? kTableSmem : 0) > 48 * 1024) {
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
