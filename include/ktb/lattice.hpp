// ktb/lattice.hpp -- the search strategies' view of a parameter space.
//
// A position is a digit vector: digit d is the position of parameter d's
// value in its value list (parameters in declaration order).  Enumeration
// order (first parameter slowest) is then the order of the mixed-radix
// number the digits spell -- its *rank* in the raw space -- so an
// enumerable space (raw size within the enumeration limit) is fully
// described by the sorted ranks of its valid points:
//
//   member(x)   binary search of rank(x)           (no constraint evaluation)
//   row(i)      digits of the i-th valid rank        (enumeration index i)
//   index(x)    position of rank(x) among the valid ranks
//
// Above the limit there is no table; membership falls back to evaluating
// the space's constraints and predicates.  Every sampling primitive the
// strategies use lives here, with the reference's random-number consumption
// (rng.hpp uniform_index / uniform01 draws in the same order and with the
// same bounds), so seeded searches visit the same configurations as the
// reference tuner (tests/test_search.py compares results CSVs byte for byte).
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "ktb/rng.hpp"
#include "ktb/space.hpp"

namespace ktb {

using Digits = std::vector<uint32_t>;

class Lattice {
  public:
    explicit Lattice(const SearchSpace& space);

    size_t dims() const { return radix_.size(); }
    uint32_t radix(size_t d) const { return radix_[d]; }
    bool enumerable() const { return enumerable_; }
    const SearchSpace& space() const { return space_; }

    // Valid points (streams the whole raw space once when not enumerable).
    unsigned long long count() const;
    bool member(const Digits& x) const;
    // Enumeration index <-> digits (enumerable spaces only).
    Digits row(uint64_t index) const;
    std::optional<uint64_t> index(const Digits& x) const;

    // A uniformly drawn valid point: one uniform_index over the valid count
    // (enumerable), else rejection over uniform raw points.
    Digits draw(Rng& rng) const;
    // The valid one-digit moves of x, in parameter order, -1 before +1.
    std::vector<Digits> moves(const Digits& x) const;
    // One uniformly chosen move; with none, any other valid point.
    Digits hop(const Digits& x, Rng& rng) const;
    // `n` distinct valid points, uniformly without replacement, as
    // enumeration indices (partial Fisher-Yates) ...
    std::vector<uint64_t> sample_indices(size_t n, Rng& rng) const;
    // ... or as points (any space; rejection with a seen-set above the limit).
    std::vector<Digits> sample(size_t n, Rng& rng) const;

    Configuration configuration(const Digits& x) const;
    Digits digits_of(const Configuration& c) const;  // c must use the space's values
    // Identity of a point for evaluation caches (one byte per digit run).
    std::string key(const Digits& x) const;

  private:
    uint64_t rank(const Digits& x) const;
    Digits unrank(uint64_t r) const;
    const std::vector<uint64_t>& ranks() const;  // enumerates on first use

    const SearchSpace& space_;
    std::vector<uint32_t> radix_;
    std::vector<uint64_t> stride_;                 // rank weights (enumerable)
    bool enumerable_ = false;
    mutable const std::vector<uint64_t>* ranks_ = nullptr;  // sorted valid ranks
    mutable std::optional<unsigned long long> count_;
};

}  // namespace ktb
