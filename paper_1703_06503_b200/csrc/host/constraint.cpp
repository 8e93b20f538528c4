// constraint.cpp -- parser and postfix evaluator of ktb::ConstraintExpr.
#include "ktb/constraint.hpp"

#include <cctype>
#include <limits>

namespace ktb {

namespace {

enum class Tok : uint8_t {
    integer, identifier, lparen, rparen, bang, star, slash, percent, plus, minus,
    lt, le, gt, ge, eq, ne, land, lor, end
};

struct Token {
    Tok kind;
    uint32_t begin, end;
    Value number = 0;
};

using Op = ConstraintExpr::Op;

struct Node {
    Op op;
    Value lit = 0;
    uint32_t param = 0;
    int lhs = -1, rhs = -1;
    uint32_t begin = 0, end = 0;
};

constexpr int kMaxDepth = 256;

}  // namespace

// Recursive descent with the reference's depth accounting (each grammar
// level adds one), so pathological nesting is refused at the same point.
class ConstraintParser {
  public:
    ConstraintParser(const std::string& text, const Configuration::Names& names)
        : text_(text), names_(names) {
        tokenize();
    }

    int run() {
        int root = parse_or(0);
        if (peek().kind != Tok::end) fail(peek().begin, "unexpected trailing input");
        return root;
    }

    std::vector<Node> nodes;

  private:
    [[noreturn]] void fail(size_t off, const std::string& what) const {
        throw SyntaxError(text_, off, what);
    }

    void push(Tok k, size_t b, size_t e, Value v = 0) {
        toks_.push_back(Token{k, uint32_t(b), uint32_t(e), v});
    }

    void tokenize() {
        const std::string& s = text_;
        size_t i = 0;
        auto two = [&](char next) { return i + 1 < s.size() && s[i + 1] == next; };
        while (i < s.size()) {
            const unsigned char c = static_cast<unsigned char>(s[i]);
            const size_t b = i;
            if (std::isspace(c)) {
                ++i;
                continue;
            }
            if (std::isdigit(c)) {
                Value v = 0;
                while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) {
                    const int dgt = s[i] - '0';
                    if (v > (std::numeric_limits<Value>::max() - dgt) / 10)
                        fail(b, "integer literal too large");
                    v = v * 10 + dgt;
                    ++i;
                }
                push(Tok::integer, b, i, v);
                continue;
            }
            if (std::isalpha(c) || c == '_') {
                while (i < s.size() &&
                       (std::isalnum(static_cast<unsigned char>(s[i])) || s[i] == '_'))
                    ++i;
                push(Tok::identifier, b, i);
                continue;
            }
            Tok k;
            size_t len = 1;
            switch (c) {
                case '(': k = Tok::lparen; break;
                case ')': k = Tok::rparen; break;
                case '*': k = Tok::star; break;
                case '/': k = Tok::slash; break;
                case '%': k = Tok::percent; break;
                case '+': k = Tok::plus; break;
                case '-': k = Tok::minus; break;
                case '!':
                    if (two('=')) k = Tok::ne, len = 2;
                    else k = Tok::bang;
                    break;
                case '<':
                    if (two('=')) k = Tok::le, len = 2;
                    else k = Tok::lt;
                    break;
                case '>':
                    if (two('=')) k = Tok::ge, len = 2;
                    else k = Tok::gt;
                    break;
                case '=':
                    if (!two('=')) fail(b, "single '=' (use '==')");
                    k = Tok::eq, len = 2;
                    break;
                case '&':
                    if (!two('&')) fail(b, "single '&' (use '&&')");
                    k = Tok::land, len = 2;
                    break;
                case '|':
                    if (!two('|')) fail(b, "single '|' (use '||')");
                    k = Tok::lor, len = 2;
                    break;
                default:
                    fail(b, std::string("unexpected character '") + char(c) + "'");
            }
            i += len;
            push(k, b, i);
        }
        push(Tok::end, s.size(), s.size());
    }

    const Token& peek() const { return toks_[pos_]; }
    Token take() { return toks_[pos_++]; }
    bool accept(Tok k) {
        if (toks_[pos_].kind != k) return false;
        ++pos_;
        return true;
    }
    void depth_check(int d) const {
        if (d > kMaxDepth) fail(peek().begin, "expression nested too deeply");
    }

    int add(Node n) {
        nodes.push_back(n);
        return int(nodes.size()) - 1;
    }
    int binary(Op op, int l, int r) {
        Node n;
        n.op = op;
        n.lhs = l;
        n.rhs = r;
        n.begin = nodes[size_t(l)].begin;
        n.end = nodes[size_t(r)].end;
        return add(n);
    }

    int parse_or(int d) {
        depth_check(d);
        int l = parse_and(d + 1);
        while (accept(Tok::lor)) l = binary(Op::or_jump, l, parse_and(d + 1));
        return l;
    }
    int parse_and(int d) {
        int l = parse_cmp(d + 1);
        while (accept(Tok::land)) l = binary(Op::and_jump, l, parse_cmp(d + 1));
        return l;
    }
    int parse_cmp(int d) {
        int l = parse_sum(d + 1);
        Op op;
        switch (peek().kind) {
            case Tok::eq: op = Op::eq; break;
            case Tok::ne: op = Op::ne; break;
            case Tok::le: op = Op::le; break;
            case Tok::ge: op = Op::ge; break;
            case Tok::lt: op = Op::lt; break;
            case Tok::gt: op = Op::gt; break;
            default: return l;
        }
        take();
        return binary(op, l, parse_sum(d + 1));
    }
    int parse_sum(int d) {
        int l = parse_term(d + 1);
        for (;;) {
            if (accept(Tok::plus)) l = binary(Op::add, l, parse_term(d + 1));
            else if (accept(Tok::minus)) l = binary(Op::sub, l, parse_term(d + 1));
            else return l;
        }
    }
    int parse_term(int d) {
        int l = parse_factor(d + 1);
        for (;;) {
            if (accept(Tok::star)) l = binary(Op::mul, l, parse_factor(d + 1));
            else if (accept(Tok::slash)) l = binary(Op::div, l, parse_factor(d + 1));
            else if (accept(Tok::percent)) l = binary(Op::mod, l, parse_factor(d + 1));
            else return l;
        }
    }
    int parse_factor(int d) {
        depth_check(d);
        const Token& t = peek();
        switch (t.kind) {
            case Tok::bang: {
                Token bang = take();
                int x = parse_factor(d + 1);
                Node n;
                n.op = Op::lnot;
                n.lhs = x;
                n.begin = bang.begin;
                n.end = nodes[size_t(x)].end;
                return add(n);
            }
            case Tok::lparen: {
                Token open = take();
                int inner = parse_or(d + 1);
                if (!accept(Tok::rparen)) fail(peek().begin, "expected ')'");
                nodes[size_t(inner)].begin = open.begin;  // diagnostics quote the parentheses
                nodes[size_t(inner)].end = toks_[pos_ - 1].end;
                return inner;
            }
            case Tok::integer: {
                Token lit = take();
                Node n;
                n.op = Op::lit;
                n.lit = lit.number;
                n.begin = lit.begin;
                n.end = lit.end;
                return add(n);
            }
            case Tok::identifier: {
                Token id = take();
                const std::string name = text_.substr(id.begin, id.end - id.begin);
                size_t idx = names_.size();
                for (size_t i = 0; i < names_.size(); ++i)
                    if (names_[i] == name) {
                        idx = i;
                        break;
                    }
                if (idx == names_.size()) throw UnknownParameter(name);
                Node n;
                n.op = Op::param;
                n.param = uint32_t(idx);
                n.begin = id.begin;
                n.end = id.end;
                return add(n);
            }
            case Tok::end: fail(t.begin, "unexpected end of input");
            default: fail(t.begin, "expected a value, identifier, '!' or '('");
        }
    }

    const std::string& text_;
    const Configuration::Names& names_;
    std::vector<Token> toks_;
    size_t pos_ = 0;
};

namespace {

void emit(const std::vector<Node>& nodes, int at, std::vector<ConstraintExpr::Insn>& code) {
    const Node& n = nodes[size_t(at)];
    ConstraintExpr::Insn in;
    in.op = n.op;
    in.begin = n.begin;
    in.end = n.end;
    switch (n.op) {
        case Op::lit:
            in.lit = n.lit;
            code.push_back(in);
            return;
        case Op::param:
            in.arg = n.param;
            code.push_back(in);
            return;
        case Op::lnot:
            emit(nodes, n.lhs, code);
            code.push_back(in);
            return;
        case Op::and_jump:
        case Op::or_jump: {
            emit(nodes, n.lhs, code);
            const size_t jump = code.size();
            code.push_back(in);
            emit(nodes, n.rhs, code);
            ConstraintExpr::Insn b;
            b.op = Op::to_bool;
            code.push_back(b);
            code[jump].arg = uint32_t(code.size());
            return;
        }
        default:
            emit(nodes, n.lhs, code);
            emit(nodes, n.rhs, code);
            code.push_back(in);
    }
}

}  // namespace

ConstraintExpr ConstraintExpr::parse(std::string text,
                                     std::shared_ptr<const Configuration::Names> names) {
    if (!names) names = std::make_shared<const Configuration::Names>();
    ConstraintExpr e;
    e.text_ = std::move(text);
    e.names_ = std::move(names);
    ConstraintParser p(e.text_, *e.names_);
    const int root = p.run();
    emit(p.nodes, root, e.code_);
    for (const Node& n : p.nodes) {
        if (n.op != Op::param) continue;
        bool seen = false;
        for (uint32_t q : e.param_order_) seen = seen || q == n.param;
        if (!seen) e.param_order_.push_back(n.param);
    }
    // Stack depth of the postfix program.
    int depth = 0, peak = 0;
    for (const Insn& in : e.code_) {
        switch (in.op) {
            case Op::lit:
            case Op::param: ++depth; break;
            case Op::lnot:
            case Op::to_bool: break;
            case Op::and_jump:
            case Op::or_jump: --depth; break;  // the fall-through path pops
            default: --depth; break;
        }
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
