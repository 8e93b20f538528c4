// basics.cpp -- argument recipes, digests and configurations of the ktb host
// library (reference arguments.hpp, config.hpp).
#include <algorithm>
#include <bit>
#include <cstring>
#include <cstdlib>
#include <numeric>
#include <thread>

#include "ktb/arguments.hpp"
#include "ktb/config.hpp"
#include "ktb/rng.hpp"

namespace ktb {

const char* to_string(ArgRole role) {
    return role == ArgRole::input ? "input" : role == ArgRole::output ? "output" : "scalar";
}

const char* to_string(ElementType type) { return type == ElementType::f32 ? "f32" : "i32"; }

ArgRole arg_role_from(const std::string& n) {
    if (n == "input") return ArgRole::input;
    if (n == "output") return ArgRole::output;
    if (n == "scalar") return ArgRole::scalar;
    throw Error("unknown argument role \"" + n + "\" (expected input, output or scalar)");
}

ElementType element_type_from(const std::string& n) {
    if (n == "f32") return ElementType::f32;
    if (n == "i32") return ElementType::i32;
    throw Error("unknown element type \"" + n + "\" (expected f32 or i32)");
}

size_t buffer_length(const Buffer& b) {
    return std::visit([](const auto& v) { return v.size(); }, b);
}

ElementType buffer_type(const Buffer& b) {
    return std::holds_alternative<BufferF32>(b) ? ElementType::f32 : ElementType::i32;
}

FillRecipe parse_fill(const std::string& fill) {
    FillRecipe r;
    if (fill.empty() || fill == "none") return r;
    if (fill == "ramp") {
        r.kind = FillRecipe::Kind::ramp;
        return r;
    }
    const size_t colon = fill.find(':');
    const std::string head = fill.substr(0, colon);
    const std::string tail = colon == std::string::npos ? "" : fill.substr(colon + 1);
    try {
        size_t used = 0;
        if (head == "constant") {
            r.kind = FillRecipe::Kind::constant;
            r.constant = std::stod(tail, &used);
            if (used == tail.size()) return r;
        } else if (head == "uniform") {
            r.kind = FillRecipe::Kind::uniform;
            r.seed = std::stoull(tail, &used);
            if (used == tail.size()) return r;
        } else {
            throw Error("unknown fill recipe \"" + fill +
                        "\" (expected none, constant:<v>, ramp or uniform:<seed>)");
        }
    } catch (const Error&) {
        throw;
    } catch (const std::exception&) {
    }
    throw Error("malformed fill recipe \"" + fill + "\"");
}

// Host threads for large uniform recipes (KTC_MATERIALIZE_THREADS; default:
// the hardware threads, at most 32).
int materialize_threads() {
    static const int n = [] {
        if (const char* e = std::getenv("KTC_MATERIALIZE_THREADS")) return std::max(1, std::atoi(e));
        return int(std::min(32u, std::max(1u, std::thread::hardware_concurrency())));
    }();
    return n;
}

void materialize_into(const ArgumentSpec& arg, void* out) {
    if (arg.role == ArgRole::scalar) throw Error("materialize_argument called on a scalar argument");
    const FillRecipe r = parse_fill(arg.fill);
    const size_t n = arg.length;
    if (arg.type == ElementType::f32) {
        float* d = static_cast<float*>(out);
        switch (r.kind) {
            case FillRecipe::Kind::none: std::fill(d, d + n, 0.0f); break;
            case FillRecipe::Kind::constant: std::fill(d, d + n, static_cast<float>(r.constant)); break;
            case FillRecipe::Kind::ramp:
                for (size_t i = 0; i < n; ++i) d[i] = static_cast<float>(i);
                break;
            case FillRecipe::Kind::uniform:
                fill_uniform_f32(r.seed, d, n, materialize_threads());
                break;
        }
        return;
    }
    int32_t* d = static_cast<int32_t*>(out);
    switch (r.kind) {
        case FillRecipe::Kind::none: std::fill(d, d + n, 0); break;
        case FillRecipe::Kind::constant: std::fill(d, d + n, static_cast<int32_t>(r.constant)); break;
        case FillRecipe::Kind::ramp:
            for (size_t i = 0; i < n; ++i) d[i] = static_cast<int32_t>(i);
            break;
        case FillRecipe::Kind::uniform: {
            Rng rng(r.seed);
            for (size_t i = 0; i < n; ++i) d[i] = static_cast<int32_t>(uniform_index(rng, 1000));
            break;
        }
    }
}

Buffer materialize_argument(const ArgumentSpec& arg) {
    if (arg.type == ElementType::f32) {
        BufferF32 v(arg.length);
        materialize_into(arg, v.data());
        return v;
    }
    BufferI32 v(arg.length);
    materialize_into(arg, v.data());
    return v;
}

uint64_t words_digest(const void* data, size_t n_words) {
    // Little-endian hosts only (x86-64, aarch64): the words' memory bytes
    // are already in the reference's serialization order.
    static_assert(std::endian::native == std::endian::little);
    return fnv1a64(data, n_words * 4);
}

uint64_t buffer_digest(const Buffer& b) {
    return std::visit([](const auto& v) { return words_digest(v.data(), v.size()); }, b);
}

std::string digest_hex(uint64_t d) {
    static const char* hex = "0123456789abcdef";
    std::string s(16, '0');
    for (int i = 15; i >= 0; --i, d >>= 4) s[size_t(i)] = hex[d & 0xf];
    return s;
}

// ---------------------------------------------------------------------------
// Configuration
// ---------------------------------------------------------------------------

Configuration::Configuration(std::shared_ptr<const Names> names, std::vector<Value> values)
    : names_(std::move(names)), values_(std::move(values)) {
    if (!names_ || names_->size() != values_.size())
        throw InvalidConfiguration("name/value count mismatch while constructing configuration");
}

Configuration::Configuration(std::initializer_list<std::pair<std::string, Value>> entries) {
    auto names = std::make_shared<Names>();
    for (const auto& e : entries) {
        names->push_back(e.first);
        values_.push_back(e.second);
    }
    names_ = std::move(names);
}

const Configuration::Names& Configuration::names() const {
    static const Names empty_names;
    return names_ ? *names_ : empty_names;
}

size_t Configuration::find(std::string_view name) const {
    if (!names_) return npos;
    for (size_t i = 0; i < names_->size(); ++i)
        if ((*names_)[i] == name) return i;
    return npos;
}

Value Configuration::at(std::string_view name) const {
    const size_t i = find(name);
    if (i == npos) throw UnknownParameter(std::string(name));
    return values_[i];
}

std::string Configuration::canonical() const {
    const Names& ns = names();
    std::vector<size_t> order(values_.size());
    std::iota(order.begin(), order.end(), size_t{0});
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ns[a] < ns[b]; });
    std::string s;
    s.reserve(order.size() * 10);
    for (size_t k = 0; k < order.size(); ++k) {
        if (k) s += ';';
        s += ns[order[k]];
        s += '=';
        s += std::to_string(values_[order[k]]);
    }
    return s;
}

bool operator==(const Configuration& a, const Configuration& b) {
    if (a.values_ != b.values_) return false;
    return a.names_ == b.names_ || a.names() == b.names();
}

}  // namespace ktb
