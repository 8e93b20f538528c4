// lattice.cpp -- digit-vector view of a search space (include/ktb/lattice.hpp).
#include "ktb/lattice.hpp"

#include <algorithm>
#include <cstring>
#include <unordered_map>
#include <unordered_set>

namespace ktb {

namespace {
constexpr size_t kDrawCap = 1'000'000;  // uniform raw draws before giving up
}

Lattice::Lattice(const SearchSpace& space) : space_(space) {
    const std::vector<Parameter>& ps = space.parameters();
    if (ps.empty()) throw Error("the space has no parameters");
    radix_.reserve(ps.size());
    for (const Parameter& p : ps) radix_.push_back(uint32_t(p.values.size()));
    if (space.raw_size() <= SearchSpace::kEnumerationLimit) {
        stride_.assign(ps.size(), 1);
        for (size_t d = ps.size() - 1; d-- > 0;) stride_[d] = stride_[d + 1] * radix_[d + 1];
        enumerable_ = true;
    }
}

const std::vector<uint64_t>& Lattice::ranks() const {
    if (!ranks_) ranks_ = &space_.valid_ranks();
    return *ranks_;
}

uint64_t Lattice::rank(const Digits& x) const {
    uint64_t r = 0;
    for (size_t d = 0; d < x.size(); ++d) r += uint64_t(x[d]) * stride_[d];
    return r;
}

Digits Lattice::unrank(uint64_t r) const {
    Digits x(radix_.size());
    for (size_t d = 0; d < x.size(); ++d) {
        x[d] = uint32_t(r / stride_[d]);
        r %= stride_[d];
    }
    return x;
}

unsigned long long Lattice::count() const {
    if (enumerable_) return ranks().size();
    if (!count_) count_ = space_.valid_count();
    return *count_;
}

bool Lattice::member(const Digits& x) const {
    if (enumerable_) return std::binary_search(ranks().begin(), ranks().end(), rank(x));
    return space_.satisfies(configuration(x));
}

Digits Lattice::row(uint64_t i) const {
    if (i >= ranks().size())
        throw InvalidConfiguration("enumeration index " + std::to_string(i) + " out of range");
    return unrank(ranks()[size_t(i)]);
}

std::optional<uint64_t> Lattice::index(const Digits& x) const {
    const std::vector<uint64_t>& r = ranks();
    auto it = std::lower_bound(r.begin(), r.end(), rank(x));
    if (it == r.end() || *it != rank(x)) return std::nullopt;
    return uint64_t(it - r.begin());
}

Digits Lattice::draw(Rng& rng) const {
    if (enumerable_) {
        const uint64_t n = ranks().size();
        if (n == 0) throw EmptySpace();
        return row(uniform_index(rng, n));
    }
    Digits x(radix_.size());
    for (size_t attempt = 0; attempt < kDrawCap; ++attempt) {
        for (size_t d = 0; d < x.size(); ++d) x[d] = uint32_t(uniform_index(rng, radix_[d]));
        if (member(x)) return x;
    }
    throw EmptySpace("no valid configuration found after " + std::to_string(kDrawCap) +
                     " uniform draws; the space is empty or vanishingly sparse");
}

std::vector<Digits> Lattice::moves(const Digits& x) const {
    std::vector<Digits> out;
    Digits y = x;
    for (size_t d = 0; d < x.size(); ++d) {
        if (x[d] > 0) {
            y[d] = x[d] - 1;
            if (member(y)) out.push_back(y);
        }
        if (x[d] + 1 < radix_[d]) {
            y[d] = x[d] + 1;
            if (member(y)) out.push_back(y);
        }
        y[d] = x[d];
    }
    return out;
}

Digits Lattice::hop(const Digits& x, Rng& rng) const {
    if (!member(x))
        throw InvalidConfiguration("random_neighbor called with a configuration outside the space");
    std::vector<Digits> m = moves(x);
    if (!m.empty()) return m[size_t(uniform_index(rng, m.size()))];
    if (count() <= 1) return x;
    for (;;) {
        Digits y = draw(rng);
        if (y != x) return y;
    }
}

std::vector<uint64_t> Lattice::sample_indices(size_t n, Rng& rng) const {
    if (n == 0) return {};
    const size_t total = ranks().size();
    if (n > total) throw BudgetExceedsSpace(n, total);
    // Partial Fisher-Yates; the permutation is kept sparse (only displaced
    // slots are stored), so a small sample of a large space costs O(n).
    std::unordered_map<uint64_t, uint64_t> moved;
    auto at = [&](uint64_t i) {
        auto it = moved.find(i);
        return it == moved.end() ? i : it->second;
    };
    std::vector<uint64_t> out;
    out.reserve(n);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t j = i + uniform_index(rng, total - i);
        const uint64_t vi = at(i), vj = at(j);
        moved[j] = vi;
        out.push_back(vj);
    }
    return out;
}

std::vector<Digits> Lattice::sample(size_t n, Rng& rng) const {
    if (n == 0) return {};
    std::vector<Digits> out;
    if (enumerable_) {
        for (uint64_t i : sample_indices(n, rng)) out.push_back(row(i));
        return out;
    }
    const unsigned long long avail = count();
    if (n > avail) throw BudgetExceedsSpace(n, avail);
    std::unordered_set<std::string> seen;
    size_t misses = 0;
    while (out.size() < n) {
        Digits x = draw(rng);
        if (seen.insert(key(x)).second) {
            out.push_back(std::move(x));
            misses = 0;
        } else if (++misses > kDrawCap) {
            throw Error("sample_unique stalled: could not find a fresh valid configuration after " +
                        std::to_string(kDrawCap) + " draws");
        }
    }
    return out;
}

Configuration Lattice::configuration(const Digits& x) const {
    const std::vector<Parameter>& ps = space_.parameters();
    std::vector<Value> v(x.size());
    for (size_t d = 0; d < x.size(); ++d) v[d] = ps[d].values[x[d]];
    return Configuration(space_.names(), std::move(v));
}

Digits Lattice::digits_of(const Configuration& c) const {
    const std::vector<Parameter>& ps = space_.parameters();
    Digits x(ps.size());
    for (size_t d = 0; d < ps.size(); ++d) {
        const Value v = c.at(ps[d].name);
        auto it = std::find(ps[d].values.begin(), ps[d].values.end(), v);
        if (it == ps[d].values.end())
            throw InvalidConfiguration("value " + std::to_string(v) +
                                       " is not in the list of parameter \"" + ps[d].name + "\"");
        x[d] = uint32_t(it - ps[d].values.begin());
    }
    return x;
}

std::string Lattice::key(const Digits& x) const {
    std::string k(x.size() * sizeof(uint32_t), '\0');
    std::memcpy(k.data(), x.data(), k.size());
    return k;
}

}  // namespace ktb
