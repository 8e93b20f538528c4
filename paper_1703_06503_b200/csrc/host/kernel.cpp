// kernel.cpp -- launch geometry of a configuration (CLTune's Mul/Div
// Global/Local size modifiers) and the device-limit predicate.
//
// Semantics (reference kernel.hpp:82-163, device.hpp:14-45): modifiers apply
// in order to the base global / local sizes, one factor per dimension (a
// parameter name or a non-negative literal); divisions must be exact.  A
// configuration is launchable on a device when its sizes resolve, every
// local dimension is within the per-dimension limit (and non-zero), their
// product within the work-group limit, no global dimension is zero, and the
// kernel's local-memory expression stays within the device's local memory.
//
// Structure here: the modifier list is compiled once into a GeometryProgram
// whose factors are literals or parameter slots of the space, so the
// predicate evaluated over every raw configuration (2.65 M for the SGEMM
// space) does no name lookups or string parsing.
#include "ktb/kernel.hpp"

#include <algorithm>
#include <cctype>
#include <optional>

namespace ktb {

namespace {

struct PresetRow {
    const char* name;
    size_t wg_total, wg0, wg1, wg2, local_mem;
    double gflops, gbs;
};

// The reference presets plus the B200 (1024 threads; 1024/1024/64;
// 232,448 B opt-in shared memory per block; FP32 SIMT 148 SM x 128 lanes x
// 2 x 1.965 GHz; 8 TB/s HBM3e).
constexpr PresetRow kPresets[] = {
    {"K40m", 1024, 1024, 1024, 64, 49152, 4291.0, 288.0},
    {"GTX480", 1024, 1024, 1024, 64, 49152, 1345.0, 177.0},
    {"HD7970", 256, 256, 256, 256, 32768, 4368.0, 288.0},
    {"Iris5100", 512, 512, 512, 512, 65536, 832.0, 26.0},
    {"B200", 1024, 1024, 1024, 64, 232448, 148.0 * 128 * 2 * 1.965, 8000.0},
};

bool all_digits(const std::string& s) {
    return !s.empty() && std::all_of(s.begin(), s.end(),
                                     [](char c) { return std::isdigit(static_cast<unsigned char>(c)); });
}

// One factor: a literal, or a parameter -- read from its slot when the
// configuration comes from the space the program was bound to (same name
// list), by name otherwise.
struct Factor {
    std::string name;
    std::optional<unsigned long long> literal;
    std::optional<size_t> slot;
    unsigned long long value(const Configuration& c, const Configuration::Names* bound) const {
        if (literal) return *literal;
        if (slot && c.names_ptr().get() == bound) return static_cast<unsigned long long>(c.value_at(*slot));
        return static_cast<unsigned long long>(c.at(name));  // throws UnknownParameter
    }
};

struct GeometryProgram {
    std::vector<size_t> global, local;
    struct Step {
        bool on_global, divide;
        std::vector<Factor> factors;
    };
    std::vector<Step> steps;
    const Configuration::Names* bound = nullptr;

    GeometryProgram(const KernelSpec& k, const SearchSpace* space)
        : global(k.base_global), local(k.base_local),
          bound(space && space->names() ? space->names().get() : nullptr) {
        for (const ThreadSizeModifier& m : k.modifiers) {
            Step s{m.target == SizeTarget::global, m.op == SizeOp::divide, {}};
            const size_t dims = s.on_global ? global.size() : local.size();
            if (m.factors.size() != dims)
                throw Error("thread-size modifier lists " + std::to_string(m.factors.size()) +
                            " factors for " + std::to_string(dims) + " " + to_string(m.target) +
                            " dimensions");
            for (const std::string& f : m.factors) {
                Factor x{f, std::nullopt, std::nullopt};
                if (all_digits(f)) x.literal = std::stoull(f);
                else if (space && space->has_parameter(f)) x.slot = space->parameter_index(f);
                s.factors.push_back(std::move(x));
            }
            steps.push_back(std::move(s));
        }
    }

    ResolvedSizes run(const Configuration& c) const {
        ResolvedSizes r{global, local};
        for (const Step& s : steps) {
            std::vector<size_t>& v = s.on_global ? r.global : r.local;
            for (size_t d = 0; d < v.size(); ++d) {
                const unsigned long long f = s.factors[d].value(c, bound);
                if (!s.divide) {
                    v[d] *= f;
                    continue;
                }
                if (f == 0) throw ZeroDivisor(d);
                if (v[d] % f) throw InexactDivision(d, v[d], f);
                v[d] /= f;
            }
        }
        return r;
    }
};

}  // namespace

DeviceModel device_preset(const std::string& name) {
    for (const PresetRow& p : kPresets)
        if (name == p.name)
            return DeviceModel{p.name, p.wg_total, {p.wg0, p.wg1, p.wg2}, p.local_mem, p.gflops, p.gbs};
    throw UnknownDevice(name);
}

std::vector<std::string> device_preset_names() {
    std::vector<std::string> n;
    for (const PresetRow& p : kPresets) n.emplace_back(p.name);
    return n;
}

const char* to_string(SizeTarget t) { return t == SizeTarget::global ? "global" : "local"; }
const char* to_string(SizeOp o) { return o == SizeOp::multiply ? "multiply" : "divide"; }

ResolvedSizes resolve_thread_sizes(const KernelSpec& k, const Configuration& c) {
    return GeometryProgram(k, nullptr).run(c);
}

Predicate device_constraints(const KernelSpec& kernel, const DeviceModel& device,
                             const SearchSpace& space) {
    auto program = std::make_shared<const GeometryProgram>(kernel, &space);
    std::optional<ConstraintExpr> smem;
    if (!kernel.local_mem_expr.empty()) smem = ConstraintExpr::parse(kernel.local_mem_expr, space.names());
    auto fits = [program, device, smem](const Configuration& c) -> bool {
        std::optional<ResolvedSizes> s;
        try {
            s = program->run(c);
        } catch (const InexactDivision&) {
            return false;
        } catch (const ZeroDivisor&) {
            return false;
        }
        size_t threads = 1;
        for (size_t d = 0; d < s->local.size(); ++d) {
            if (s->local[d] == 0 || s->local[d] > device.max_work_group_dim[d]) return false;
            threads *= s->local[d];
        }
        if (threads > device.max_work_group_total) return false;
        if (std::find(s->global.begin(), s->global.end(), size_t(0)) != s->global.end()) return false;
        if (!smem) return true;
        const Value bytes = smem->evaluate_value(c);
        return bytes >= 0 && static_cast<unsigned long long>(bytes) <= device.local_mem_bytes;
    };
    return Predicate{"device-limits:" + device.name, std::move(fits)};
}

}  // namespace ktb
