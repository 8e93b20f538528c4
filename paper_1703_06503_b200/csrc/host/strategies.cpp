// strategies.cpp -- the four search strategies of the ktune API (reference
// search.hpp:47-395) as walks over a Lattice (include/ktb/lattice.hpp).
//
// Every strategy is a small state machine driven by one loop (drive()):
//   begin()   draws the starting point(s)
//   next()    the point to evaluate at this step, or nothing when done
//   observe() the evaluated time; updates the walk
// The Ledger in front of the user's evaluator memoizes by point identity,
// counts distinct evaluations, keeps the best (strictly smaller times
// replace it, so ties keep the earliest) and records the trace.  Budgets,
// step caps, cooling schedule, acceptance rule and swarm moves follow the
// reference definitions cited at each piece, with the same random-number
// draws in the same order, so results are identical to the reference's for
// the same seed (tests/test_search.py: byte-identical results CSVs).
#include "ktb/search.hpp"

#include <cmath>
#include <limits>
#include <unordered_map>

#include "ktb/lattice.hpp"

namespace ktb {

const char* to_string(StrategyKind k) {
    static const char* const names[] = {"full", "random", "annealing", "pso"};
    const int i = int(k);
    return i >= 0 && i < 4 ? names[i] : "?";
}

StrategyKind strategy_kind_from(const std::string& n) {
    for (StrategyKind k : {StrategyKind::full, StrategyKind::random, StrategyKind::annealing,
                           StrategyKind::pso})
        if (n == to_string(k)) return k;
    throw Error("unknown strategy \"" + n + "\" (expected full, random, annealing or pso)");
}

// search.hpp:86-102: floor(count * fraction) with a 1e-9 guard, at least 1.
size_t budget(unsigned long long count, double fraction) {
    if (!(fraction > 0.0)) throw Error("fraction must be > 0, got " + std::to_string(fraction));
    const long double scaled = std::floor((long double)count * (long double)fraction + 1e-9L);
    constexpr long double kMax = (long double)std::numeric_limits<size_t>::max();
    return scaled < 1.0L ? size_t(1) : scaled >= kMax ? std::numeric_limits<size_t>::max()
                                                      : size_t(scaled);
}

// search.hpp:112-123: Metropolis acceptance; a failed neighbour (+inf) is
// never accepted, an improvement always.
double sa_acceptance(double t, double tp, double temperature) {
    if (!(temperature > 0.0)) throw NonPositiveTemperature(temperature);
    if (tp < t) return 1.0;
    return std::isinf(tp) ? 0.0 : std::exp((t - tp) / temperature);
}

namespace {

void require_probabilities(double a, double b, double g) {
    for (double p : {a, b, g})
        if (!(p >= 0.0 && p <= 1.0))
            throw InvalidProbabilities("each of alpha, beta, gamma must lie in [0, 1]");
    if (a + b + g > 1.0 + 1e-12) throw InvalidProbabilities("alpha + beta + gamma must not exceed 1");
}

double or_inf(const std::optional<double>& t) {
    return t ? *t : std::numeric_limits<double>::infinity();
}

class Ledger {
  public:
    Ledger(const Lattice& lat, const Evaluator& fn, SearchOutcome& out)
        : lat_(lat), fn_(fn), out_(out) {}

    std::optional<double> visit(const Digits& x) {
        auto [it, fresh] = seen_.try_emplace(lat_.key(x));
        if (!fresh) return it->second;
        Configuration c = lat_.configuration(x);
        const std::optional<double> t = fn_(c);
        it->second = t;
        const size_t step = ++out_.unique_evaluations;
        if (!t) ++out_.failed_evaluations;
        else if (!out_.best_time_ms || *t < *out_.best_time_ms) {
            out_.best_time_ms = t;
            out_.best_config = c;
        }
        out_.trace.push_back(TraceEntry{step, std::move(c), t, out_.best_time_ms});
        return t;
    }
    size_t distinct() const { return out_.unique_evaluations; }

  private:
    const Lattice& lat_;
    const Evaluator& fn_;
    SearchOutcome& out_;
    std::unordered_map<std::string, std::optional<double>> seen_;
};

// ------------------------------------------------------------- strategies
struct Walk {
    virtual ~Walk() = default;
    virtual void begin(Rng& rng) = 0;
    virtual std::optional<Digits> next(Rng& rng) = 0;
    virtual void observe(const Digits& x, const std::optional<double>& t, Rng& rng) = 0;
};

// Full sweep (search.hpp:246-260) and random sample (:263-277): a fixed
// visit list, one evaluation per step.
struct ListWalk final : Walk {
    std::vector<Digits> list;
    size_t at = 0;
    void begin(Rng&) override {}
    std::optional<Digits> next(Rng&) override {
        if (at == list.size()) return std::nullopt;
        return list[at++];
    }
    void observe(const Digits&, const std::optional<double>&, Rng&) override {}
};

// Simulated annealing (search.hpp:282-321): a ±1 move of one parameter per
// step from the current point, accepted with exp(-dt/T_k), where the
// temperature cools linearly with the spent budget to a 5% floor.
struct Annealer final : Walk {
    const Lattice& lat;
    const Ledger& ledger;
    const Prefetcher& prefetch;
    double t0;
    size_t budget;
    Digits cur;
    double cur_t = 0.0;
    bool started = false;
    std::string warmed;  // point whose moves were prefetched
    Annealer(const Lattice& l, const Ledger& led, const Prefetcher& pf, double temp, size_t b)
        : lat(l), ledger(led), prefetch(pf), t0(temp), budget(b) {}

    void begin(Rng& rng) override { cur = lat.draw(rng); }
    std::optional<Digits> next(Rng& rng) override {
        if (!started) return cur;
        if (prefetch) {  // every move of the current point is a possible next step
            std::string k = lat.key(cur);
            if (k != warmed) {
                for (const Digits& m : lat.moves(cur)) prefetch(lat.configuration(m));
                warmed = std::move(k);
            }
        }
        return lat.hop(cur, rng);
    }
    void observe(const Digits& x, const std::optional<double>& time, Rng& rng) override {
        const double t = or_inf(time);  // a failed point is infinitely slow
        if (!started) {
            cur_t = t;
            started = true;
            return;
        }
        const double spent = double(ledger.distinct()) / double(budget);
        const double temp = t0 * std::max(1.0 - spent, 0.05);
        if (uniform01(rng) < sa_acceptance(cur_t, t, temp)) {
            cur = x;
            cur_t = t;
        }
    }
};

// Particle swarm (search.hpp:326-375, pso_move :150-178): particles take
// turns; after each evaluation the particle's next position draws every
// digit from {random, personal best, global best, stay} with probabilities
// alpha, beta, gamma, rest -- redrawn (up to 100 times) until valid.
struct Swarm final : Walk {
    const Lattice& lat;
    const Prefetcher& prefetch;
    size_t size;
    double alpha, beta, gamma;
    std::vector<Digits> pos;
    std::vector<std::optional<std::pair<Digits, double>>> own;
    std::optional<std::pair<Digits, double>> all;
    size_t turn = 0, cur = 0;
    Swarm(const Lattice& l, const Prefetcher& pf, size_t s, double a, double b, double g)
        : lat(l), prefetch(pf), size(s), alpha(a), beta(b), gamma(g), own(s) {}

    void begin(Rng& rng) override {
        for (size_t i = 0; i < size; ++i) pos.push_back(lat.draw(rng));
        if (prefetch)
            for (const Digits& p : pos) prefetch(lat.configuration(p));
    }
    std::optional<Digits> next(Rng&) override {
        cur = turn++ % size;
        return pos[cur];
    }
    Digits move(const Digits& x, const Digits& p, const Digits& g, Rng& rng) const {
        Digits y(x.size());
        for (int attempt = 0; attempt < 100; ++attempt) {
            for (size_t d = 0; d < x.size(); ++d) {
                const double u = uniform01(rng);
                y[d] = u < alpha                  ? uint32_t(uniform_index(rng, lat.radix(d)))
                       : u < alpha + beta         ? p[d]
                       : u < alpha + beta + gamma ? g[d]
                                                  : x[d];
            }
            if (lat.member(y)) return y;
        }
        return x;
    }
    void observe(const Digits& x, const std::optional<double>& t, Rng& rng) override {
        if (t) {
            if (!own[cur] || *t < own[cur]->second) own[cur] = {x, *t};
            if (!all || *t < all->second) all = {x, *t};
        }
        const Digits& p = own[cur] ? own[cur]->first : x;
        const Digits& g = all ? all->first : x;
        pos[cur] = move(x, p, g, rng);
        if (prefetch) prefetch(lat.configuration(pos[cur]));  // this particle's next evaluation
    }
};

// One loop for every strategy: a step is one requested point (cached or
// not); stops at the budget of distinct evaluations or at the step cap.
void drive(Walk& walk, Ledger& ledger, SearchOutcome& out, size_t cap, Rng& rng) {
    walk.begin(rng);
    while (ledger.distinct() < out.budget && out.total_steps < cap) {
        std::optional<Digits> x = walk.next(rng);
        if (!x) break;
        ++out.total_steps;
        walk.observe(*x, ledger.visit(*x), rng);
    }
}

unsigned long long nonempty_count(const Lattice& lat) {
    const unsigned long long n = lat.count();
    if (n == 0) throw EmptySpace();
    return n;
}

size_t affordable(unsigned long long count, double fraction) {
    const size_t b = budget(count, fraction);
    if (b > count) throw BudgetExceedsSpace(b, count);
    return b;
}

}  // namespace

SearchOutcome run_search(const SearchSpace& space, const Evaluator& evaluate,
                         const StrategySpec& s, uint64_t seed, const Prefetcher& prefetch) {
    if (s.kind == StrategyKind::annealing && !(s.temperature > 0.0))
        throw NonPositiveTemperature(s.temperature);
    if (s.kind == StrategyKind::pso) {
        if (s.swarm == 0) throw Error("swarm size must be >= 1");
        require_probabilities(s.alpha, s.beta, s.gamma);
    }
    SearchOutcome out;
    if (s.kind == StrategyKind::full && space.raw_size() > SearchSpace::kEnumerationLimit)
        throw ExplicitEnumerationTooLarge(space.raw_size(), SearchSpace::kEnumerationLimit);
    const Lattice lat(space);
    Ledger ledger(lat, evaluate, out);
    Rng rng(seed);
    switch (s.kind) {
        case StrategyKind::full: {
            ListWalk w;
            const unsigned long long n = nonempty_count(lat);
            w.list.reserve(size_t(n));
            for (uint64_t i = 0; i < n; ++i) w.list.push_back(lat.row(i));
            out.budget = size_t(n);
            drive(w, ledger, out, std::numeric_limits<size_t>::max(), rng);
            break;
        }
        case StrategyKind::random: {
            ListWalk w;
            out.budget = affordable(nonempty_count(lat), s.fraction);
            w.list = lat.sample(out.budget, rng);
            drive(w, ledger, out, std::numeric_limits<size_t>::max(), rng);
            break;
        }
        case StrategyKind::annealing: {
            out.budget = affordable(nonempty_count(lat), s.fraction);
            Annealer w(lat, ledger, prefetch, s.temperature, out.budget);
            drive(w, ledger, out, 50 * out.budget, rng);
            break;
        }
        case StrategyKind::pso: {
            out.budget = affordable(nonempty_count(lat), s.fraction);
            Swarm w(lat, prefetch, s.swarm, s.alpha, s.beta, s.gamma);
            drive(w, ledger, out, 50 * out.budget, rng);
            break;
        }
    }
    return out;
}

std::vector<uint64_t> planned_indices(const SearchSpace& space, const StrategySpec& s,
                                      uint64_t seed, size_t* budget_out) {
    if (s.kind != StrategyKind::full && s.kind != StrategyKind::random)
        throw Error("planned_indices: only full and random searches have a fixed visit order");
    const Lattice lat(space);
    const unsigned long long n = nonempty_count(lat);
    if (s.kind == StrategyKind::full) {
        std::vector<uint64_t> idx(static_cast<size_t>(n));
        for (uint64_t i = 0; i < n; ++i) idx[size_t(i)] = i;
        *budget_out = size_t(n);
        return idx;
    }
    Rng rng(seed);
    *budget_out = affordable(n, s.fraction);
    return lat.sample_indices(*budget_out, rng);
}

}  // namespace ktb
