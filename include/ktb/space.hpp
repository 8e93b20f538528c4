// ktb/space.hpp -- parameter spaces (reference space.hpp): parameters,
// constraint expressions and native predicates; odometer enumeration (first
// parameter slowest) cached and shared between copies; streaming counts;
// the sorted raw ranks of the valid points that the strategies' Lattice
// samples and walks on.
//
// B200-side differences (same results): enumeration runs on all host cores
// (the raw space is split on its leading parameters and the per-thread
// results are concatenated in order) and is stored as one flat value table;
// Configuration objects are materialized from it on demand.
#pragma once

#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "ktb/config.hpp"
#include "ktb/constraint.hpp"
#include "ktb/rng.hpp"

namespace ktb {

struct Parameter {
    std::string name;
    std::vector<Value> values;
    std::vector<std::string> labels;
    const std::string* label_of(Value v) const;
};

struct Predicate {
    std::string label;
    std::function<bool(const Configuration&)> fn;
};

class SearchSpace {
  public:
    static constexpr unsigned long long kEnumerationLimit = 10'000'000ull;

    SearchSpace() = default;
    SearchSpace(const SearchSpace& other);
    SearchSpace& operator=(const SearchSpace& other);

    SearchSpace& add_parameter(std::string name, std::vector<Value> values,
                               std::vector<std::string> labels = {});
    SearchSpace& add_constraint(std::string text);
    SearchSpace& add_predicate(std::string label, std::function<bool(const Configuration&)> fn);
    SearchSpace& add_predicate(Predicate p);

    const std::vector<Parameter>& parameters() const { return params_; }
    const std::vector<ConstraintExpr>& constraints() const { return constraints_; }
    const std::vector<Predicate>& predicates() const { return predicates_; }
    size_t parameter_index(std::string_view name) const;
    const Parameter& parameter(std::string_view name) const;
    bool has_parameter(std::string_view name) const;
    const std::shared_ptr<const Configuration::Names>& names() const { return names_; }
    unsigned long long raw_size() const;

    bool satisfies(const Configuration& c) const;
    bool is_valid(const Configuration& c) const;
    Configuration make_configuration(std::vector<Value> values) const;

    // All valid configurations, enumeration order (cached).
    const std::vector<Configuration>& enumerate_valid() const;
    // The same as a flat table: row i = values of configuration i (cached).
    const std::vector<Value>& valid_table() const;
    Configuration config_at(size_t index) const;
    unsigned long long valid_count() const;
    unsigned long long constraint_only_count() const;

    // Odometer ranks (mixed-radix index in the raw space, first parameter
    // most significant) of the valid configurations, ascending: row i of
    // valid_table() is rank valid_ranks()[i].  Sampling and neighbourhoods
    // live in ktb/lattice.hpp on top of this.
    const std::vector<uint64_t>& valid_ranks() const;

  private:
    struct Cache {
        std::shared_ptr<const std::vector<Value>> table;
        std::shared_ptr<const std::vector<uint64_t>> ranks;
        std::shared_ptr<const std::vector<Configuration>> configs;
        std::optional<unsigned long long> count;
    };
    void rebuild_names();
    void invalidate();
    void require_parameters() const;
    bool satisfies_values(const Value* v, Configuration& scratch) const;
    // Enumerates valid rows (values, and their raw ranks) of the raw space;
    // parallel over threads.
    std::vector<Value> enumerate_table(std::vector<uint64_t>* ranks) const;
    unsigned long long count_valid(bool predicates) const;

    std::vector<Parameter> params_;
    std::shared_ptr<const Configuration::Names> names_;
    std::vector<ConstraintExpr> constraints_;
    std::vector<Predicate> predicates_;
    mutable std::mutex mu_;
    mutable Cache cache_;
};

}  // namespace ktb
