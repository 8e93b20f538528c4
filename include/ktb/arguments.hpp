// ktb/arguments.hpp -- kernel argument recipes (reference arguments.hpp).
// Arguments travel as recipes, not data: a backend materializes them itself,
// deterministically, so host and device see the same input bits.
#pragma once

#include <cstdint>
#include <string>
#include <variant>
#include <vector>

#include "ktb/errors.hpp"

namespace ktb {

enum class ArgRole { input, output, scalar };
enum class ElementType { f32, i32 };

const char* to_string(ArgRole role);
const char* to_string(ElementType type);
ArgRole arg_role_from(const std::string& name);
ElementType element_type_from(const std::string& name);

// fill: "none" | "constant:<v>" | "ramp" | "uniform:<seed>" (f32 in [0,1),
// i32 in [0,1000)).
struct ArgumentSpec {
    ArgRole role = ArgRole::input;
    ElementType type = ElementType::f32;
    size_t length = 0;
    double value = 0.0;
    std::string fill = "none";
};

using BufferF32 = std::vector<float>;
using BufferI32 = std::vector<int32_t>;
using Buffer = std::variant<BufferF32, BufferI32>;

size_t buffer_length(const Buffer& b);
ElementType buffer_type(const Buffer& b);

struct FillRecipe {
    enum class Kind { none, constant, ramp, uniform } kind = Kind::none;
    double constant = 0.0;
    uint64_t seed = 0;
};
FillRecipe parse_fill(const std::string& fill);

// Contents of a buffer argument (arguments.hpp:126-180).
Buffer materialize_argument(const ArgumentSpec& arg);
// In-place variant writing `length` elements of 4 bytes into `out`.
void materialize_into(const ArgumentSpec& arg, void* out);

// FNV-1a-64 over 4-byte little-endian words (arguments.hpp:184-205).
uint64_t buffer_digest(const Buffer& b);
uint64_t words_digest(const void* data, size_t n_words);
std::string digest_hex(uint64_t digest);

}  // namespace ktb
