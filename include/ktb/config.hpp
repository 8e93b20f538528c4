// ktb/config.hpp -- one point of a parameter space (reference config.hpp).
// Names are shared by every configuration of a space; a configuration holds
// only its values.  canonical() ("name=value" pairs sorted by name, ';'
// joined) keys caches, replay tables and report rows.
#pragma once

#include <initializer_list>
#include <memory>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "ktb/errors.hpp"

namespace ktb {

using Value = long long;

class Configuration {
  public:
    using Names = std::vector<std::string>;
    static constexpr size_t npos = static_cast<size_t>(-1);

    Configuration() = default;
    Configuration(std::shared_ptr<const Names> names, std::vector<Value> values);
    explicit Configuration(std::initializer_list<std::pair<std::string, Value>> entries);

    size_t size() const { return values_.size(); }
    bool empty() const { return values_.empty(); }
    const Names& names() const;
    const std::shared_ptr<const Names>& names_ptr() const { return names_; }
    const std::vector<Value>& values() const { return values_; }
    const std::string& name_at(size_t i) const { return names().at(i); }
    Value value_at(size_t i) const { return values_.at(i); }
    void set_value_at(size_t i, Value v) { values_.at(i) = v; }
    bool has(std::string_view name) const { return find(name) != npos; }
    size_t find(std::string_view name) const;
    Value at(std::string_view name) const;  // throws UnknownParameter
    std::string canonical() const;

    friend bool operator==(const Configuration& a, const Configuration& b);
    friend bool operator!=(const Configuration& a, const Configuration& b) { return !(a == b); }

  private:
    std::shared_ptr<const Names> names_;
    std::vector<Value> values_;
};

}  // namespace ktb
