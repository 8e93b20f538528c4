// ktb/kernel.hpp -- kernel descriptions, launch-geometry arithmetic and the
// device-limit predicate (reference kernel.hpp, device.hpp).
#pragma once

#include <array>
#include <cstddef>
#include <string>
#include <vector>

#include "ktb/arguments.hpp"
#include "ktb/space.hpp"

namespace ktb {

// Device limits a configuration must respect, plus roofline peaks.
struct DeviceModel {
    std::string name = "generic";
    size_t max_work_group_total = 1024;
    std::array<size_t, 3> max_work_group_dim = {1024, 1024, 64};
    size_t local_mem_bytes = 49152;
    double peak_gflops = 0.0;
    double peak_gbs = 0.0;
};

// Presets: the reference's K40m, GTX480, HD7970, Iris5100, plus "B200"
// (1024 threads, 1024/1024/64, 232,448 B opt-in shared memory per block,
// FP32 SIMT peak 148 SM x 128 x 2 x 1.965 GHz, 8 TB/s HBM3e).
DeviceModel device_preset(const std::string& name);
std::vector<std::string> device_preset_names();

enum class SizeTarget { global, local };
enum class SizeOp { multiply, divide };
const char* to_string(SizeTarget t);
const char* to_string(SizeOp o);

// CLTune's Mul/DivGlobalSize and Mul/DivLocalSize: factors are parameter
// names or non-negative integer literals, one per dimension.
struct ThreadSizeModifier {
    SizeTarget target = SizeTarget::global;
    SizeOp op = SizeOp::multiply;
    std::vector<std::string> factors;
};

struct KernelSpec {
    std::string name;
    std::string source_ref;
    std::vector<size_t> base_global;
    std::vector<size_t> base_local;
    std::vector<ThreadSizeModifier> modifiers;
    std::vector<ArgumentSpec> arguments;
    std::string local_mem_expr;  // bytes; empty = none
};

struct ResolvedSizes {
    std::vector<size_t> global;
    std::vector<size_t> local;
};

// Applies the modifiers in order; InexactDivision / ZeroDivisor on bad divides.
ResolvedSizes resolve_thread_sizes(const KernelSpec& kernel, const Configuration& config);

// One predicate for every launchability limit of `device` (kernel.hpp:118-163).
Predicate device_constraints(const KernelSpec& kernel, const DeviceModel& device,
                             const SearchSpace& space);

}  // namespace ktb
