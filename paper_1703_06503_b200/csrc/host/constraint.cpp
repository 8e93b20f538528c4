// constraint.cpp -- the constraint language (grammar in ktb/constraint.hpp):
// a scanner, a table-driven precedence parser that emits the postfix
// program directly (no parse tree), and the evaluator.
//
// Parity with the reference (constraint.hpp:137-485): the whole text is
// scanned before parsing, so a lexical error anywhere wins over a syntax
// error; diagnostics carry the same messages and byte offsets; nesting is
// refused with the same depth accounting (every precedence level and every
// unary '!' or '(' descends one level; the check runs when an "or" level or
// an operand is entered, against 256); comparisons do not chain.
#include "ktb/constraint.hpp"

#include <cctype>
#include <limits>

namespace ktb {

namespace {

using Op = ConstraintExpr::Op;
using Insn = ConstraintExpr::Insn;

enum class Sym : uint8_t { number, name, open, close, bang, binop, end };

struct Lexeme {
    Sym sym;
    Op op = Op::lit;  // binop: which operator
    uint32_t begin = 0, end = 0;
    Value number = 0;
};

struct Punct {
    const char* text;
    Sym sym;
    Op op;
};

// Longest match first within each leading character.
constexpr Punct kPuncts[] = {
    {"||", Sym::binop, Op::or_jump}, {"&&", Sym::binop, Op::and_jump},
    {"==", Sym::binop, Op::eq},      {"!=", Sym::binop, Op::ne},
    {"<=", Sym::binop, Op::le},      {">=", Sym::binop, Op::ge},
    {"<", Sym::binop, Op::lt},       {">", Sym::binop, Op::gt},
    {"+", Sym::binop, Op::add},      {"-", Sym::binop, Op::sub},
    {"*", Sym::binop, Op::mul},      {"/", Sym::binop, Op::div},
    {"%", Sym::binop, Op::mod},      {"!", Sym::bang, Op::lnot},
    {"(", Sym::open, Op::lit},       {")", Sym::close, Op::lit},
};

[[noreturn]] void syntax(const std::string& text, size_t off, const std::string& what) {
    throw SyntaxError(text, off, what);
}

std::vector<Lexeme> scan(const std::string& s) {
    std::vector<Lexeme> out;
    size_t i = 0;
    while (i < s.size()) {
        const unsigned char c = static_cast<unsigned char>(s[i]);
        const uint32_t b = uint32_t(i);
        if (std::isspace(c)) {
            ++i;
        } else if (std::isdigit(c)) {
            Value v = 0;
            for (; i < s.size() && std::isdigit(static_cast<unsigned char>(s[i])); ++i) {
                const int d = s[i] - '0';
                if (v > (std::numeric_limits<Value>::max() - d) / 10)
                    syntax(s, b, "integer literal too large");
                v = v * 10 + d;
            }
            out.push_back({Sym::number, Op::lit, b, uint32_t(i), v});
        } else if (std::isalpha(c) || c == '_') {
            while (i < s.size() && (std::isalnum(static_cast<unsigned char>(s[i])) || s[i] == '_')) ++i;
            out.push_back({Sym::name, Op::param, b, uint32_t(i), 0});
        } else {
            const Punct* hit = nullptr;
            for (const Punct& p : kPuncts)
                if (s.compare(i, std::char_traits<char>::length(p.text), p.text) == 0) {
                    hit = &p;
                    break;
                }
            if (!hit) {
                // A lone '=', '&' or '|' names the operator it falls short of.
                if (c == '=') syntax(s, b, "single '=' (use '==')");
                if (c == '&') syntax(s, b, "single '&' (use '&&')");
                if (c == '|') syntax(s, b, "single '|' (use '||')");
                syntax(s, b, std::string("unexpected character '") + char(c) + "'");
            }
            i += std::char_traits<char>::length(hit->text);
            out.push_back({hit->sym, hit->op, b, uint32_t(i), 0});
        }
    }
    out.push_back({Sym::end, Op::lit, uint32_t(s.size()), uint32_t(s.size()), 0});
    return out;
}

// Binary precedence levels, loosest first.  `chain`: left-associative
// repetition; otherwise at most one operator at that level.
struct Level {
    Op ops[6];
    int n;
    bool chain;
};
constexpr Level kLevels[] = {
    {{Op::or_jump}, 1, true},
    {{Op::and_jump}, 1, true},
    {{Op::eq, Op::ne, Op::le, Op::ge, Op::lt, Op::gt}, 6, false},
    {{Op::add, Op::sub}, 2, true},
    {{Op::mul, Op::div, Op::mod}, 3, true},
};
constexpr int kLevelCount = 5;
constexpr int kMaxDepth = 256;

bool at_level(int level, Op op) {
    for (int k = 0; k < kLevels[level].n; ++k)
        if (kLevels[level].ops[k] == op) return true;
    return false;
}

struct Span {
    uint32_t begin, end;
};

class Emitter {
  public:
    Emitter(const std::string& text, const Configuration::Names& names, std::vector<Insn>& code,
            std::vector<uint32_t>& params)
        : text_(text), names_(names), code_(code), params_(params), lex_(scan(text)) {}

    void run() {
        level(0, 0);
        if (lex_[at_].sym != Sym::end) syntax(text_, lex_[at_].begin, "unexpected trailing input");
    }

  private:
    void guard(int depth) const {
        if (depth > kMaxDepth) syntax(text_, lex_[at_].begin, "expression nested too deeply");
    }

    void emit(Op op, Span s, uint32_t arg = 0, Value lit = 0) {
        Insn in;
        in.op = op;
        in.arg = arg;
        in.lit = lit;
        in.begin = s.begin;
        in.end = s.end;
        code_.push_back(in);
    }

    // One precedence level at `depth`; its operands are the next level at
    // depth + 1 (operands of the tightest level are primaries).
    Span level(int lv, int depth) {
        if (lv == 0) guard(depth);
        if (lv == kLevelCount) return primary(depth);
        Span lhs = level(lv + 1, depth + 1);
        for (bool once = false; lex_[at_].sym == Sym::binop && at_level(lv, lex_[at_].op);) {
            if (once && !kLevels[lv].chain) break;
            once = true;
            const Op op = lex_[at_++].op;
            if (op == Op::and_jump || op == Op::or_jump) {
                const size_t jump = code_.size();
                emit(op, lhs);
                const Span rhs = level(lv + 1, depth + 1);
                lhs = {lhs.begin, rhs.end};
                emit(Op::to_bool, lhs);
                code_[jump].arg = uint32_t(code_.size());
                code_[jump].end = lhs.end;
            } else {
                const Span rhs = level(lv + 1, depth + 1);
                lhs = {lhs.begin, rhs.end};
                emit(op, lhs);
            }
        }
        return lhs;
    }

    Span primary(int depth) {
        guard(depth);
        const Lexeme t = lex_[at_];
        switch (t.sym) {
            case Sym::bang: {
                ++at_;
                const Span x = primary(depth + 1);
                const Span s{t.begin, x.end};
                emit(Op::lnot, s);
                return s;
            }
            case Sym::open: {
                ++at_;
                level(0, depth + 1);
                if (lex_[at_].sym != Sym::close) syntax(text_, lex_[at_].begin, "expected ')'");
                // Diagnostics quote a parenthesized operand with its
                // parentheses: widen the span of its root (the last insn).
                const Span s{t.begin, lex_[at_++].end};
                code_.back().begin = s.begin;
                code_.back().end = s.end;
                return s;
            }
            case Sym::number:
                ++at_;
                emit(Op::lit, {t.begin, t.end}, 0, t.number);
                return {t.begin, t.end};
            case Sym::name: {
                ++at_;
                const std::string name = text_.substr(t.begin, t.end - t.begin);
                uint32_t slot = 0;
                while (slot < names_.size() && names_[slot] != name) ++slot;
                if (slot == names_.size()) throw UnknownParameter(name);
                bool seen = false;
                for (uint32_t q : params_) seen = seen || q == slot;
                if (!seen) params_.push_back(slot);
                emit(Op::param, {t.begin, t.end}, slot);
                return {t.begin, t.end};
            }
            case Sym::end: syntax(text_, t.begin, "unexpected end of input");
            default: syntax(text_, t.begin, "expected a value, identifier, '!' or '('");
        }
    }

    const std::string& text_;
    const Configuration::Names& names_;
    std::vector<Insn>& code_;
    std::vector<uint32_t>& params_;
    std::vector<Lexeme> lex_;
    size_t at_ = 0;
};

}  // namespace

ConstraintExpr ConstraintExpr::parse(std::string text,
                                     std::shared_ptr<const Configuration::Names> names) {
    if (!names) names = std::make_shared<const Configuration::Names>();
    ConstraintExpr e;
    e.text_ = std::move(text);
    e.names_ = std::move(names);
    Emitter(e.text_, *e.names_, e.code_, e.param_order_).run();
    // Stack depth of the postfix program.
    int depth = 0, peak = 0;
    for (const Insn& in : e.code_) {
        if (in.op == Op::lit || in.op == Op::param) ++depth;
        else if (in.op != Op::lnot && in.op != Op::to_bool) --depth;
        peak = std::max(peak, depth + 1);
    }
    e.max_stack_ = uint32_t(peak + 1);
    return e;
}

ConstraintExpr ConstraintExpr::parse(std::string text, Configuration::Names names) {
    return parse(std::move(text), std::make_shared<const Configuration::Names>(std::move(names)));
}

template <typename Fetch>
Value ConstraintExpr::run(Fetch&& fetch) const {
    if (code_.empty()) throw Error("evaluating a default-constructed constraint");
    Value small[64];
    std::vector<Value> big;
    Value* st = small;
    if (max_stack_ > 64) {
        big.resize(max_stack_);
        st = big.data();
    }
    int sp = -1;
    const size_t n = code_.size();
    for (size_t pc = 0; pc < n;) {
        const Insn& in = code_[pc];
        switch (in.op) {
            case Op::lit: st[++sp] = in.lit; break;
            case Op::param: st[++sp] = fetch(in.arg); break;
            case Op::lnot: st[sp] = st[sp] == 0 ? 1 : 0; break;
            case Op::to_bool: st[sp] = st[sp] != 0 ? 1 : 0; break;
            case Op::and_jump:
                if (st[sp] == 0) {
                    pc = in.arg;
                    continue;
                }
                --sp;
                break;
            case Op::or_jump:
                if (st[sp] != 0) {
                    st[sp] = 1;
                    pc = in.arg;
                    continue;
                }
                --sp;
                break;
            default: {
                const Value r = st[sp--];
                Value& l = st[sp];
                switch (in.op) {
                    case Op::mul: l = l * r; break;
                    case Op::div:
                        if (r == 0) throw DivisionByZero(text_.substr(in.begin, in.end - in.begin));
                        l = l / r;
                        break;
                    case Op::mod:
                        if (r == 0) throw DivisionByZero(text_.substr(in.begin, in.end - in.begin));
                        l = l % r;
                        break;
                    case Op::add: l = l + r; break;
                    case Op::sub: l = l - r; break;
                    case Op::lt: l = l < r; break;
                    case Op::le: l = l <= r; break;
                    case Op::gt: l = l > r; break;
                    case Op::ge: l = l >= r; break;
                    case Op::eq: l = l == r; break;
                    case Op::ne: l = l != r; break;
                    default: throw Error("corrupt constraint program");
                }
            }
        }
        ++pc;
    }
    return st[0];
}

Value ConstraintExpr::evaluate_values(const Value* values) const {
    return run([values](uint32_t i) { return values[i]; });
}

Value ConstraintExpr::evaluate_value(const Configuration& config) const {
    if (config.names_ptr() == names_) {
        const Value* v = config.values().data();
        return run([v](uint32_t i) { return v[i]; });
    }
    return run([&](uint32_t i) { return config.at((*names_)[i]); });
}

std::vector<std::string> ConstraintExpr::referenced() const {
    std::vector<std::string> out;
    for (uint32_t i : param_order_) out.push_back((*names_)[i]);
    return out;
}

}  // namespace ktb
