// kernel.cpp -- thread-size resolution, device presets and device limits.
#include "ktb/kernel.hpp"

#include <cctype>

namespace ktb {

DeviceModel device_preset(const std::string& name) {
    if (name == "K40m") return DeviceModel{"K40m", 1024, {1024, 1024, 64}, 49152, 4291.0, 288.0};
    if (name == "GTX480")
        return DeviceModel{"GTX480", 1024, {1024, 1024, 64}, 49152, 1345.0, 177.0};
    if (name == "HD7970") return DeviceModel{"HD7970", 256, {256, 256, 256}, 32768, 4368.0, 288.0};
    if (name == "Iris5100")
        return DeviceModel{"Iris5100", 512, {512, 512, 512}, 65536, 832.0, 26.0};
    if (name == "B200")
        return DeviceModel{"B200", 1024, {1024, 1024, 64}, 232448, 148.0 * 128 * 2 * 1.965, 8000.0};
    throw UnknownDevice(name);
}

std::vector<std::string> device_preset_names() {
    return {"K40m", "GTX480", "HD7970", "Iris5100", "B200"};
}

const char* to_string(SizeTarget t) { return t == SizeTarget::global ? "global" : "local"; }
const char* to_string(SizeOp o) { return o == SizeOp::multiply ? "multiply" : "divide"; }

namespace {

bool is_literal(const std::string& s) {
    if (s.empty()) return false;
    for (char c : s)
        if (!std::isdigit(static_cast<unsigned char>(c))) return false;
    return true;
}

unsigned long long factor_of(const std::string& f, const Configuration& c) {
    if (is_literal(f)) return std::stoull(f);
    return static_cast<unsigned long long>(c.at(f));
}

}  // namespace

ResolvedSizes resolve_thread_sizes(const KernelSpec& k, const Configuration& c) {
    ResolvedSizes s{k.base_global, k.base_local};
    for (const ThreadSizeModifier& m : k.modifiers) {
        std::vector<size_t>& t = m.target == SizeTarget::global ? s.global : s.local;
        if (m.factors.size() != t.size())
            throw Error("thread-size modifier lists " + std::to_string(m.factors.size()) +
                        " factors for " + std::to_string(t.size()) + " " + to_string(m.target) +
                        " dimensions");
        for (size_t d = 0; d < t.size(); ++d) {
            const unsigned long long f = factor_of(m.factors[d], c);
            if (m.op == SizeOp::multiply) {
                t[d] *= f;
            } else {
                if (f == 0) throw ZeroDivisor(d);
                if (t[d] % f != 0) throw InexactDivision(d, t[d], f);
                t[d] /= f;
            }
        }
    }
    return s;
}

Predicate device_constraints(const KernelSpec& kernel, const DeviceModel& device,
                             const SearchSpace& space) {
    const bool has_mem = !kernel.local_mem_expr.empty();
    ConstraintExpr mem;
    if (has_mem) mem = ConstraintExpr::parse(kernel.local_mem_expr, space.names());
    auto fn = [kernel, device, mem, has_mem](const Configuration& c) -> bool {
        ResolvedSizes s;
        try {
            s = resolve_thread_sizes(kernel, c);
        } catch (const InexactDivision&) {
            return false;
        } catch (const ZeroDivisor&) {
            return false;
        }
        size_t total = 1;
        for (size_t d = 0; d < s.local.size(); ++d) {
            if (s.local[d] == 0 || s.local[d] > device.max_work_group_dim[d]) return false;
            total *= s.local[d];
        }
        if (total > device.max_work_group_total) return false;
        for (size_t g : s.global)
            if (g == 0) return false;
        if (has_mem) {
            const Value bytes = mem.evaluate_value(c);
            if (bytes < 0 || static_cast<unsigned long long>(bytes) > device.local_mem_bytes)
                return false;
        }
        return true;
    };
    return Predicate{"device-limits:" + device.name, std::move(fn)};
}

}  // namespace ktb
