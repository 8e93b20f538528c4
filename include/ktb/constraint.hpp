// ktb/constraint.hpp -- constraint expressions over a space's parameters
// (reference constraint.hpp).  Same grammar, precedence, integer semantics,
// short-circuit && / ||, error types and error offsets:
//
//   expr   := or
//   or     := and ( "||" and )*
//   and    := cmp ( "&&" cmp )*
//   cmp    := sum ( ("==" | "!=" | "<=" | ">=" | "<" | ">") sum )?
//   sum    := term ( ("+" | "-") term )*
//   term   := factor ( ("*" | "/" | "%") factor )*
//   factor := "!" factor | "(" expr ")" | integer | identifier
//
// The parse tree is flattened into a postfix program with short-circuit
// jumps, so the enumeration hot loop (2.65M GEMM configurations x 9
// constraints) evaluates without recursion or allocation.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "ktb/config.hpp"

namespace ktb {

class ConstraintExpr {
  public:
    ConstraintExpr() = default;

    static ConstraintExpr parse(std::string text,
                                std::shared_ptr<const Configuration::Names> names);
    static ConstraintExpr parse(std::string text, Configuration::Names names);

    Value evaluate_value(const Configuration& config) const;
    bool evaluate(const Configuration& config) const { return evaluate_value(config) != 0; }
    // Fast path: `values` laid out in this expression's name order.
    Value evaluate_values(const Value* values) const;

    const std::string& text() const { return text_; }
    std::vector<std::string> referenced() const;
    const std::shared_ptr<const Configuration::Names>& names() const { return names_; }

    enum class Op : uint8_t {
        lit, param, lnot, mul, div, mod, add, sub, lt, le, gt, ge, eq, ne,
        and_jump,  // top == 0 ? (top = 0, jump) : pop
        or_jump,   // top != 0 ? (top = 1, jump) : pop
        to_bool    // top = top != 0
    };
    struct Insn {
        Op op;
        uint32_t arg = 0;  // param index / jump target
        Value lit = 0;
        uint32_t begin = 0, end = 0;  // source span (division diagnostics)
    };

  private:
    template <typename Fetch>
    Value run(Fetch&& fetch) const;

    std::string text_;
    std::shared_ptr<const Configuration::Names> names_;
    std::vector<Insn> code_;
    std::vector<uint32_t> param_order_;  // params in order of first appearance
    uint32_t max_stack_ = 0;
};

}  // namespace ktb
