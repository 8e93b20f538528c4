// ktb/search.hpp -- search strategies (reference search.hpp): the strategy
// description, the search outcome record (best, trace, counters), and the
// entry points.  The strategies themselves walk a Lattice (ktb/lattice.hpp)
// and reproduce the reference's visits for the same seed.
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "ktb/space.hpp"

namespace ktb {

using Evaluator = std::function<std::optional<double>(const Configuration&)>;
// Optional hint: `config` is likely to be evaluated soon (compile it ahead).
// Never changes what a strategy does -- only how early a backend starts work.
using Prefetcher = std::function<void(const Configuration&)>;

enum class StrategyKind { full, random, annealing, pso };
const char* to_string(StrategyKind k);
StrategyKind strategy_kind_from(const std::string& name);

struct StrategySpec {
    StrategyKind kind = StrategyKind::full;
    double fraction = 1.0;
    double temperature = 4.0;
    double alpha = 0.4;
    double beta = 0.0;
    double gamma = 0.4;
    size_t swarm = 3;
};

struct TraceEntry {
    size_t step = 0;
    Configuration config;
    std::optional<double> time_ms;
    std::optional<double> best_so_far;
};

struct SearchOutcome {
    std::optional<Configuration> best_config;
    std::optional<double> best_time_ms;
    std::vector<TraceEntry> trace;
    size_t budget = 0;
    size_t unique_evaluations = 0;
    size_t failed_evaluations = 0;
    size_t total_steps = 0;
};

// floor(count * fraction), at least 1 (reference search.hpp:86-102).
size_t budget(unsigned long long valid_count, double fraction);
// Metropolis acceptance probability of moving from time t to t_prime.
double sa_acceptance(double t, double t_prime, double temperature);

// Runs one search (full sweep, random sample, simulated annealing or particle
// swarm) over `space`; implementation: csrc/host/strategies.cpp.
SearchOutcome run_search(const SearchSpace& space, const Evaluator& evaluate,
                         const StrategySpec& strategy, uint64_t seed,
                         const Prefetcher& prefetch = nullptr);

// The unit list a sharded executor distributes: the enumeration indices a
// full search visits (0..N-1) or the random search's sample, in visit order.
// Only defined for the order-independent strategies (full, random).
std::vector<uint64_t> planned_indices(const SearchSpace& space, const StrategySpec& strategy,
                                      uint64_t seed, size_t* budget_out);

}  // namespace ktb
