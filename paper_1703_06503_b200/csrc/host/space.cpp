// space.cpp -- ktb::SearchSpace.
#include "ktb/space.hpp"

#include <algorithm>
#include <atomic>
#include <cctype>
#include <limits>
#include <thread>
#include <unordered_map>

namespace ktb {

const std::string* Parameter::label_of(Value v) const {
    if (labels.empty()) return nullptr;
    for (size_t i = 0; i < values.size(); ++i)
        if (values[i] == v) return &labels[i];
    return nullptr;
}

SearchSpace::SearchSpace(const SearchSpace& o) {
    std::lock_guard<std::mutex> lk(o.mu_);
    params_ = o.params_;
    names_ = o.names_;
    constraints_ = o.constraints_;
    predicates_ = o.predicates_;
    cache_ = o.cache_;
}

SearchSpace& SearchSpace::operator=(const SearchSpace& o) {
    if (this != &o) {
        SearchSpace copy(o);
        std::lock_guard<std::mutex> lk(mu_);
        params_ = std::move(copy.params_);
        names_ = std::move(copy.names_);
        constraints_ = std::move(copy.constraints_);
        predicates_ = std::move(copy.predicates_);
        cache_ = std::move(copy.cache_);
    }
    return *this;
}

static bool valid_identifier(const std::string& n) {
    if (n.empty() || !(std::isalpha(static_cast<unsigned char>(n[0])) || n[0] == '_')) return false;
    for (char c : n)
        if (!(std::isalnum(static_cast<unsigned char>(c)) || c == '_')) return false;
    return true;
}

namespace {

// Value-list checks of add_parameter: the earliest offending position
// decides which diagnostic is raised (a negative value, or a value listed
// again later); at the same position the negative value is reported.
void check_values(const std::string& name, const std::vector<Value>& values) {
    if (values.empty()) throw EmptyValueList(name);
    constexpr size_t none = static_cast<size_t>(-1);
    size_t negative = none, repeated = none;
    std::unordered_map<Value, size_t> first;  // value -> first position
    for (size_t i = 0; i < values.size(); ++i) {
        if (values[i] < 0 && negative == none) negative = i;
        auto [it, fresh] = first.try_emplace(values[i], i);
        if (!fresh) repeated = std::min(repeated, it->second);
    }
    if (negative != none && negative <= repeated)
        throw Error("parameter \"" + name + "\" has a negative value " +
                    std::to_string(values[negative]));
    if (repeated != none)
        throw Error("parameter \"" + name + "\" lists value " + std::to_string(values[repeated]) +
                    " twice");
}

}  // namespace

SearchSpace& SearchSpace::add_parameter(std::string name, std::vector<Value> values,
                                        std::vector<std::string> labels) {
    if (!valid_identifier(name))
        throw Error("parameter name \"" + name + "\" must match [A-Za-z_][A-Za-z0-9_]*");
    if (has_parameter(name)) throw DuplicateParameter(name);
    check_values(name, values);
    if (!labels.empty() && labels.size() != values.size())
        throw Error("parameter \"" + name + "\" has " + std::to_string(labels.size()) +
                    " labels for " + std::to_string(values.size()) + " values");
    params_.push_back(Parameter{std::move(name), std::move(values), std::move(labels)});
    rebuild_names();
    invalidate();
    return *this;
}

SearchSpace& SearchSpace::add_constraint(std::string text) {
    constraints_.push_back(ConstraintExpr::parse(std::move(text), names_));
    invalidate();
    return *this;
}

SearchSpace& SearchSpace::add_predicate(std::string label,
                                        std::function<bool(const Configuration&)> fn) {
    predicates_.push_back(Predicate{std::move(label), std::move(fn)});
    invalidate();
    return *this;
}

SearchSpace& SearchSpace::add_predicate(Predicate p) {
    predicates_.push_back(std::move(p));
    invalidate();
    return *this;
}

size_t SearchSpace::parameter_index(std::string_view name) const {
    for (size_t i = 0; i < params_.size(); ++i)
        if (params_[i].name == name) return i;
    throw UnknownParameter(std::string(name));
}

const Parameter& SearchSpace::parameter(std::string_view name) const {
    return params_[parameter_index(name)];
}

bool SearchSpace::has_parameter(std::string_view name) const {
    for (const Parameter& p : params_)
        if (p.name == name) return true;
    return false;
}

unsigned long long SearchSpace::raw_size() const {
    if (params_.empty()) return 0;
    unsigned long long prod = 1;
    for (const Parameter& p : params_) {
        const unsigned long long n = p.values.size();
        if (prod > std::numeric_limits<unsigned long long>::max() / n)
            return std::numeric_limits<unsigned long long>::max();
        prod *= n;
    }
    return prod;
}

void SearchSpace::rebuild_names() {
    auto n = std::make_shared<Configuration::Names>();
    for (const Parameter& p : params_) n->push_back(p.name);
    names_ = std::move(n);
}

void SearchSpace::invalidate() {
    std::lock_guard<std::mutex> lk(mu_);
    cache_ = Cache{};
}

void SearchSpace::require_parameters() const {
    if (params_.empty()) throw Error("the space has no parameters");
}

bool SearchSpace::satisfies(const Configuration& c) const {
    for (const ConstraintExpr& e : constraints_)
        if (!e.evaluate(c)) return false;
    for (const Predicate& p : predicates_)
        if (!p.fn(c)) return false;
    return true;
}

// Constraints were parsed against a prefix of the current name list
// (parameters are only ever appended), so their parameter indices address
// the value row directly.
bool SearchSpace::satisfies_values(const Value* v, Configuration& scratch) const {
    for (const ConstraintExpr& e : constraints_)
        if (e.evaluate_values(v) == 0) return false;
    if (!predicates_.empty()) {
        for (size_t i = 0; i < params_.size(); ++i) scratch.set_value_at(i, v[i]);
        for (const Predicate& p : predicates_)
            if (!p.fn(scratch)) return false;
    }
    return true;
}

bool SearchSpace::is_valid(const Configuration& c) const {
    if (c.size() != params_.size()) return false;
    for (const Parameter& p : params_) {
        const size_t at = c.find(p.name);
        if (at == Configuration::npos) return false;
        if (std::find(p.values.begin(), p.values.end(), c.value_at(at)) == p.values.end())
            return false;
    }
    return satisfies(c);
}

Configuration SearchSpace::make_configuration(std::vector<Value> values) const {
    if (values.size() != params_.size())
        throw InvalidConfiguration("expected " + std::to_string(params_.size()) + " values, got " +
                                   std::to_string(values.size()));
    for (size_t i = 0; i < values.size(); ++i) {
        const Parameter& p = params_[i];
        if (std::find(p.values.begin(), p.values.end(), values[i]) == p.values.end())
            throw InvalidConfiguration("value " + std::to_string(values[i]) +
                                       " is not in the list of parameter \"" + p.name + "\"");
    }
    return Configuration(names_, std::move(values));
}

namespace {

// Runs fn(thread, begin, end) over [0, raw) split into contiguous chunks.
template <typename Fn>
void split_raw(unsigned long long raw, Fn&& fn, size_t* used_threads) {
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    size_t threads = raw < 200000 ? 1 : std::min<size_t>(hw, 64);
    *used_threads = threads;
    if (threads == 1) {
        fn(size_t(0), 0ull, raw);
        return;
    }
    std::vector<std::thread> pool;
    const unsigned long long chunk = (raw + threads - 1) / threads;
    for (size_t t = 0; t < threads; ++t) {
        const unsigned long long b = std::min(raw, chunk * t), e = std::min(raw, chunk * (t + 1));
        pool.emplace_back([&fn, t, b, e] { fn(t, b, e); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

std::vector<Value> SearchSpace::enumerate_table(std::vector<uint64_t>* ranks) const {
    const unsigned long long raw = raw_size();
    const size_t np = params_.size();
    std::vector<std::vector<Value>> parts(64);
    std::vector<std::vector<uint64_t>> rank_parts(64);
    std::vector<std::string> errors(64);
    size_t used = 1;
    split_raw(
        raw,
        [&](size_t t, unsigned long long begin, unsigned long long end) {
            try {
                // Decode `begin` into odometer digits (last parameter fastest).
                std::vector<size_t> digit(np);
                unsigned long long rem = begin;
                for (size_t i = np; i-- > 0;) {
                    digit[i] = size_t(rem % params_[i].values.size());
                    rem /= params_[i].values.size();
                }
                std::vector<Value> v(np);
                for (size_t i = 0; i < np; ++i) v[i] = params_[i].values[digit[i]];
                Configuration scratch(names_, v);
                std::vector<Value>& out = parts[t];
                std::vector<uint64_t>& rk = rank_parts[t];
                for (unsigned long long idx = begin; idx < end; ++idx) {
                    if (satisfies_values(v.data(), scratch)) {
                        out.insert(out.end(), v.begin(), v.end());
                        rk.push_back(idx);
                    }
                    for (size_t s = np; s-- > 0;) {
                        if (++digit[s] < params_[s].values.size()) {
                            v[s] = params_[s].values[digit[s]];
                            break;
                        }
                        digit[s] = 0;
                        v[s] = params_[s].values[0];
                    }
                }
            } catch (const std::exception& e) {
                errors[t] = e.what();
            }
        },
        &used);
    for (size_t t = 0; t < used; ++t)
        if (!errors[t].empty()) throw Error(errors[t]);
    std::vector<Value> table;
    size_t total = 0;
    for (size_t t = 0; t < used; ++t) total += parts[t].size();
    table.reserve(total);
    ranks->clear();
    ranks->reserve(total / std::max<size_t>(np, 1));
    for (size_t t = 0; t < used; ++t) {
        table.insert(table.end(), parts[t].begin(), parts[t].end());
        ranks->insert(ranks->end(), rank_parts[t].begin(), rank_parts[t].end());
    }
    return table;
}

const std::vector<Value>& SearchSpace::valid_table() const {
    require_parameters();
    std::lock_guard<std::mutex> lk(mu_);
    if (!cache_.table) {
        const unsigned long long raw = raw_size();
        if (raw > kEnumerationLimit) throw ExplicitEnumerationTooLarge(raw, kEnumerationLimit);
        auto r = std::make_shared<std::vector<uint64_t>>();
        auto t = std::make_shared<std::vector<Value>>(enumerate_table(r.get()));
        cache_.count = t->size() / params_.size();
        cache_.table = std::move(t);
        cache_.ranks = std::move(r);
    }
    return *cache_.table;
}

const std::vector<uint64_t>& SearchSpace::valid_ranks() const {
    valid_table();
    std::lock_guard<std::mutex> lk(mu_);
    return *cache_.ranks;
}

const std::vector<Configuration>& SearchSpace::enumerate_valid() const {
    const std::vector<Value>& table = valid_table();
    std::lock_guard<std::mutex> lk(mu_);
    if (!cache_.configs) {
        const size_t np = params_.size();
        auto cs = std::make_shared<std::vector<Configuration>>();
        cs->reserve(table.size() / np);
        for (size_t i = 0; i < table.size(); i += np)
            cs->emplace_back(names_, std::vector<Value>(table.begin() + long(i),
                                                        table.begin() + long(i + np)));
        cache_.configs = std::move(cs);
    }
    return *cache_.configs;
}

Configuration SearchSpace::config_at(size_t index) const {
    const std::vector<Value>& table = valid_table();
    const size_t np = params_.size();
    if ((index + 1) * np > table.size())
        throw InvalidConfiguration("enumeration index " + std::to_string(index) + " out of range");
    return Configuration(names_, std::vector<Value>(table.begin() + long(index * np),
                                                    table.begin() + long((index + 1) * np)));
}

unsigned long long SearchSpace::count_valid(bool with_predicates) const {
    const unsigned long long raw = raw_size();
    const size_t np = params_.size();
    std::vector<unsigned long long> counts(64, 0);
    std::vector<std::string> errors(64);
    size_t used = 1;
    split_raw(
        raw,
        [&](size_t t, unsigned long long begin, unsigned long long end) {
            try {
                std::vector<size_t> digit(np);
                unsigned long long rem = begin;
                for (size_t i = np; i-- > 0;) {
                    digit[i] = size_t(rem % params_[i].values.size());
                    rem /= params_[i].values.size();
                }
                std::vector<Value> v(np);
                for (size_t i = 0; i < np; ++i) v[i] = params_[i].values[digit[i]];
                Configuration scratch(names_, v);
                unsigned long long c = 0;
                for (unsigned long long idx = begin; idx < end; ++idx) {
                    bool ok;
                    if (with_predicates) {
                        ok = satisfies_values(v.data(), scratch);
                    } else {
                        ok = true;
                        for (const ConstraintExpr& e : constraints_)
                            if (e.evaluate_values(v.data()) == 0) {
                                ok = false;
                                break;
                            }
                    }
                    c += ok;
                    for (size_t s = np; s-- > 0;) {
                        if (++digit[s] < params_[s].values.size()) {
                            v[s] = params_[s].values[digit[s]];
                            break;
                        }
                        digit[s] = 0;
                        v[s] = params_[s].values[0];
                    }
                }
                counts[t] = c;
            } catch (const std::exception& e) {
                errors[t] = e.what();
            }
        },
        &used);
    unsigned long long total = 0;
    for (size_t t = 0; t < used; ++t) {
        if (!errors[t].empty()) throw Error(errors[t]);
        total += counts[t];
    }
    return total;
}

unsigned long long SearchSpace::valid_count() const {
    require_parameters();
    {
        std::lock_guard<std::mutex> lk(mu_);
        if (cache_.count) return *cache_.count;
    }
    const unsigned long long c = count_valid(true);
    std::lock_guard<std::mutex> lk(mu_);
    cache_.count = c;
    return c;
}

unsigned long long SearchSpace::constraint_only_count() const {
    require_parameters();
    return count_valid(false);
}

}  // namespace ktb
