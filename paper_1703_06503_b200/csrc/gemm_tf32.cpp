// gemm_tf32.cpp -- plan of the TF32 tcgen05 SGEMM variant (kernel name
// "gemm_tf32", reported separately from the fp32 family with its own
// tolerance).  See kernels/gemm_tf32.cu.
#include <string>
#include <vector>

#include "core.hpp"

namespace {
#include "kernel_sources.inc"
}

namespace ktc {

bool plan_tf32(ktc_ctx* ctx, int M, int N, int K, const ktc_request* r, std::string* src_id,
               const std::string** src, std::vector<std::string>* opts, std::string* entry,
               unsigned grid[3], unsigned block[3], unsigned* smem, std::string* why) {
    (void)ctx, (void)M, (void)N, (void)K, (void)r, (void)src_id, (void)src, (void)opts,
        (void)entry, (void)grid, (void)block, (void)smem;
    (void)kConvSource, (void)kGemmSource, (void)kGemmTf32Source;
    *why = "gemm_tf32 family not available in this build";
    return false;
}

}  // namespace ktc
