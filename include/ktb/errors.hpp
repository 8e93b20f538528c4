// ktb/errors.hpp -- error taxonomy of the ktune API (reference errors.hpp),
// same class names and messages so callers catching ktune exceptions keep
// working.  Per-configuration failures are NOT exceptions (they are
// ktb::Status values); these are harness / input errors.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

namespace ktb {

struct Error : std::runtime_error {
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};

#define KTB_SIMPLE_ERROR(Name, prefix)                                      \
    struct Name : Error {                                                   \
        explicit Name(const std::string& what) : Error(prefix + what) {}    \
    };

KTB_SIMPLE_ERROR(InvalidConfiguration, std::string("invalid configuration: "))
KTB_SIMPLE_ERROR(InvalidProbabilities, std::string("invalid PSO probabilities: "))
KTB_SIMPLE_ERROR(ShapeMismatch, std::string("output shape mismatch: "))
KTB_SIMPLE_ERROR(UnknownParameterSet, std::string("unknown parameter set: "))
KTB_SIMPLE_ERROR(SpawnFailure, std::string("failed to spawn external runner: "))
KTB_SIMPLE_ERROR(ProtocolViolation, std::string("external runner protocol violation: "))
KTB_SIMPLE_ERROR(JobFileError, std::string("job file error: "))
#undef KTB_SIMPLE_ERROR

struct DuplicateParameter : Error {
    explicit DuplicateParameter(const std::string& n)
        : Error("duplicate parameter: \"" + n + "\""), name(n) {}
    std::string name;
};

struct EmptyValueList : Error {
    explicit EmptyValueList(const std::string& n)
        : Error("parameter \"" + n + "\" has an empty value list"), name(n) {}
    std::string name;
};

struct UnknownParameter : Error {
    explicit UnknownParameter(const std::string& n)
        : Error("unknown parameter: \"" + n + "\""), name(n) {}
    std::string name;
};

struct SyntaxError : Error {
    SyntaxError(const std::string& t, size_t off, const std::string& what)
        : Error("syntax error at offset " + std::to_string(off) + " in \"" + t + "\": " + what),
          text(t),
          offset(off) {}
    std::string text;
    size_t offset;
};

struct DivisionByZero : Error {
    explicit DivisionByZero(const std::string& sub)
        : Error("division by zero in subexpression \"" + sub + "\""), subexpression(sub) {}
    std::string subexpression;
};

struct ExplicitEnumerationTooLarge : Error {
    ExplicitEnumerationTooLarge(unsigned long long raw, unsigned long long lim)
        : Error("explicit enumeration refused: raw space size " + std::to_string(raw) +
                " exceeds limit " + std::to_string(lim)),
          raw_size(raw),
          limit(lim) {}
    unsigned long long raw_size, limit;
};

struct EmptySpace : Error {
    EmptySpace() : Error("search space contains no valid configuration") {}
    explicit EmptySpace(const std::string& msg) : Error(msg) {}
};

struct BudgetExceedsSpace : Error {
    BudgetExceedsSpace(size_t req, unsigned long long avail)
        : Error("requested budget of " + std::to_string(req) +
                " unique evaluations exceeds the " + std::to_string(avail) +
                " valid configurations available"),
          requested(req),
          available(avail) {}
    size_t requested;
    unsigned long long available;
};

struct NonPositiveTemperature : Error {
    explicit NonPositiveTemperature(double v)
        : Error("temperature must be > 0, got " + std::to_string(v)), value(v) {}
    double value;
};

struct InexactDivision : Error {
    InexactDivision(size_t d, unsigned long long num, unsigned long long div)
        : Error("thread-size modifier: " + std::to_string(num) + " is not divisible by " +
                std::to_string(div) + " in dimension " + std::to_string(d)),
          dim(d),
          numerator(num),
          divisor(div) {}
    size_t dim;
    unsigned long long numerator, divisor;
};

struct ZeroDivisor : Error {
    explicit ZeroDivisor(size_t d)
        : Error("thread-size modifier: zero divisor in dimension " + std::to_string(d)), dim(d) {}
    size_t dim;
};

struct EmptySpaceAfterConstraints : Error {
    EmptySpaceAfterConstraints()
        : Error("no configuration survives the device-limit constraints") {}
};

struct BackendUnavailable : Error {
    explicit BackendUnavailable(const std::string& n)
        : Error("backend unavailable: \"" + n + "\""), name(n) {}
    std::string name;
};

struct MalformedReplayFile : Error {
    MalformedReplayFile(size_t l, const std::string& what)
        : Error("malformed replay file, line " + std::to_string(l) + ": " + what), line(l) {}
    size_t line;
};

struct NonPositiveTime : Error {
    explicit NonPositiveTime(double v)
        : Error("evaluation time must be > 0, got " + std::to_string(v)), value(v) {}
    double value;
};

struct UnknownDevice : Error {
    explicit UnknownDevice(const std::string& n)
        : Error("unknown device: \"" + n + "\""), name(n) {}
    std::string name;
};

}  // namespace ktb
