// ktb/landscapes.hpp -- the paper's two case studies (reference
// landscapes.hpp): problem descriptors, search spaces, kernel descriptions
// (argument recipes, launch geometry, shared-memory expressions), throughput
// metrics and the paper's best-known rows.  The CPU oracles live in oracle/
// (test infrastructure); the product verifies against the device reference
// kernels of builtin.cu, which are bit-identical to them.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ktb/kernel.hpp"

namespace ktb {

struct ConvProblem {
    size_t x = 8192;
    size_t y = 4096;
    int filter = 7;
    float weight = 1.0f;
    uint64_t seed = 2026;
    int halo() const { return (filter - 1) / 2; }
    size_t padded_x() const { return x + size_t(filter) - 1; }
    size_t padded_y() const { return y + size_t(filter) - 1; }
    uint64_t filter_seed() const { return seed ^ 0x9e3779b97f4a7c15ull; }
    void validate() const;
};

SearchSpace conv_space();
KernelSpec conv_kernel(const ConvProblem& p);

struct ConvMetrics {
    double gflops = 0.0;
    double gbs = 0.0;
};
ConvMetrics conv_metrics(const ConvProblem& p, double time_ms);

struct GemmProblem {
    size_t m = 2048;
    size_t n = 2048;
    size_t k = 2048;
    float alpha = 1.0f;
    float beta = 0.0f;
    uint64_t seed = 2026;
    uint64_t a_seed() const { return seed; }
    uint64_t b_seed() const { return seed ^ 0x9e3779b97f4a7c15ull; }
    uint64_t c_seed() const { return seed ^ 0xc2b2ae3d27d4eb4full; }
    void validate() const;
};

SearchSpace gemm_space();
KernelSpec gemm_kernel(const GemmProblem& p);
double gemm_gflops(const GemmProblem& p, double time_ms);

// TF32 tcgen05 variant (B200 extension, kernel name "gemm_tf32"): its own
// tile space -- BM x BN output tile per CTA (BM = 128 rows of TMEM lanes),
// BK-deep K stages, STAGES-deep TMA pipeline.  Same argument list and
// problem as gemm_kernel; verified with its own tolerance (rel 1e-3).
SearchSpace gemm_tf32_space();
KernelSpec gemm_tf32_kernel(const GemmProblem& p);

Configuration conv_best_known(const SearchSpace& space, const std::string& device, int filter);
std::vector<std::string> conv_best_known_devices();
Configuration gemm_best_known(const SearchSpace& space, const std::string& device);
std::vector<std::string> gemm_best_known_devices();

}  // namespace ktb
