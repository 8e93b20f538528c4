// core.hpp -- internal state behind the ktc.h device primitives.
#pragma once

#include <cuda.h>

#include <chrono>

#include <cstdint>
#include <string>
#include <vector>

#include "driver.hpp"
#include "ktc.h"

// Mirrors VerifyPartial in builtin.cu (layout must match).
struct KtcVerifyPartial {
    unsigned long long first_fail;
    unsigned long long argmax;
    long long nan_abs;
    long long nan_rel;
    double max_abs;
    double max_rel;
};

struct ktc_ctx {
    int ordinal = -1;
    CUdevice dev = 0;
    CUcontext cu = nullptr;
    CUstream stream = nullptr;
    CUmodule builtin = nullptr;
    CUfunction fn_conv_ref = nullptr, fn_gemm_ref = nullptr;
    CUfunction fn_verify_partial = nullptr, fn_verify_final = nullptr, fn_verify_after = nullptr;
    CUfunction fn_flush = nullptr;
    CUdeviceptr flush_buf = 0;
    size_t flush_bytes = 0;
    CUdeviceptr scratch = 0;  // verify partials + final + flush sink
    int verify_blocks = 0;
    std::vector<CUevent> events;
    // Bound reference (ktc_bind_reference).
    CUdeviceptr ref = 0;
    size_t ref_count = 0;
    int ref_type = KTC_F32;
    double rel_tol = 1e-4, abs_tol = 1e-6;
    ktc_limits limits{};
    bool sticky = false;   // a sticky CUDA error poisoned the context
    long long launches = 0;  // kernels launched through this context
    // Device blocks kept for reuse (exact size match): a new job over the
    // same problem on a pooled context gets its buffers back without
    // cuMemAlloc/cuMemFree (ktc::ctx_alloc / ctx_free).
    std::vector<std::pair<size_t, CUdeviceptr>> free_blocks;
    size_t free_bytes = 0;
    unsigned epoch = 0;  // primary_ctx_epoch() when the resources were made
    // Modules of closed backends, unloaded in bulk (ktc_retire_module):
    // cuModuleUnload costs milliseconds per module, which a fresh job would
    // otherwise pay at the end of every tuning job.
    std::vector<CUmodule> retired;
};

struct ktc_fn {
    ktc_ctx* ctx = nullptr;
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
};

namespace ktc {

// Hands a loaded module to its (pooled) context for deferred unloading; the
// oldest half is unloaded once more than kRetiredCap are waiting, the rest
// when the context is torn down.
void retire_module(ktc_ctx* ctx, CUmodule mod);
constexpr size_t kRetiredCap = 4096;

// Thread-local last-error plumbing shared by every layer.
void set_error(const std::string& msg);
const std::string& last_error();

// Device allocation through the context's block cache.
CUresult ctx_alloc(ktc_ctx* ctx, size_t bytes, CUdeviceptr* p);
void ctx_free(ktc_ctx* ctx, CUdeviceptr p, size_t bytes);

// KTC_TRACE=1: phase timings of job setup / teardown on stderr (diagnostics).
bool trace_on();
void trace_phase(const char* what, std::chrono::steady_clock::time_point since);

// ktc_launch_timed with the prune_factor early-out (see ktc.h).
extern "C" int ktc_launch_timed_pruned(ktc_ctx* ctx, ktc_fn* fn, const unsigned grid[3],
                                       const unsigned block[3], unsigned smem_bytes, void** params,
                                       int warmup, int reps, int flush, double bar,
                                       float* best_ms, float* all_ms, int* reps_done);

// Bumped whenever a primary context is reset (destroyed): host allocations
// tied to the old context (pinned recipe copies) are gone with it.
unsigned primary_ctx_epoch();

// Records `rc` on ctx (marking sticky errors) and returns a ktc.h code.
int fail_cu(ktc_ctx* ctx, CUresult rc, const char* what);
bool is_sticky(CUresult rc);

// Makes ctx current on the calling thread.
int make_current(ktc_ctx* ctx);

// Launch helper on ctx->stream; counts launches.
CUresult launch(ktc_ctx* ctx, CUfunction fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                unsigned by, unsigned bz, unsigned smem, void** params);

// L2 flush on ctx->stream (allocates the flush buffer on first use).
int flush_l2(ktc_ctx* ctx);

// Device verification of count elements (one buffer) -> report.
// had_nan_abs / had_nan_rel (optional) report whether any error was NaN,
// which the cross-buffer merge needs (merge_reports).
int verify_pair(ktc_ctx* ctx, CUdeviceptr cand, CUdeviceptr ref, size_t count, int type,
                double rel, double abs, ktc_verify_report* out, bool* had_nan_abs = nullptr,
                bool* had_nan_rel = nullptr);

// Continues `total` with the report of buffer `k` exactly as the reference's
// record() lambda continues across buffers (tuner.hpp:51-69).
void merge_reports(ktc_verify_report* total, const ktc_verify_report& rep, bool had_nan_abs,
                   bool had_nan_rel, size_t k);

// Waits for an event with a watchdog (seconds); returns CUDA_ERROR_LAUNCH_TIMEOUT on expiry.
CUresult wait_event(ktc_ctx* ctx, CUevent ev, double timeout_s);

}  // namespace ktc
