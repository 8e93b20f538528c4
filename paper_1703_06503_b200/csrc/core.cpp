// core.cpp -- ktc.h layer 1: device primitives over the CUDA driver API.
#include "core.hpp"
#include "ktb/rng.hpp"

#include <atomic>
#include <chrono>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>

namespace {

#include "builtin_cubin.inc"  // const unsigned char ktc_builtin_cubin[]; size_t ktc_builtin_cubin_size

thread_local std::string g_last_error;

}  // namespace

namespace ktc {

void set_error(const std::string& msg) { g_last_error = msg; }
const std::string& last_error() { return g_last_error; }

bool is_sticky(CUresult rc) {
    switch (rc) {
        case CUDA_ERROR_ILLEGAL_ADDRESS:
        case CUDA_ERROR_LAUNCH_FAILED:
        case CUDA_ERROR_ILLEGAL_INSTRUCTION:
        case CUDA_ERROR_MISALIGNED_ADDRESS:
        case CUDA_ERROR_INVALID_ADDRESS_SPACE:
        case CUDA_ERROR_INVALID_PC:
        case CUDA_ERROR_HARDWARE_STACK_ERROR:
        case CUDA_ERROR_ASSERT:
        case CUDA_ERROR_LAUNCH_TIMEOUT:
        case CUDA_ERROR_ECC_UNCORRECTABLE:
        case CUDA_ERROR_CONTEXT_IS_DESTROYED:
            return true;
        default:
            return false;
    }
}

int fail_cu(ktc_ctx* ctx, CUresult rc, const char* what) {
    set_error(cu_error_text(rc, what));
    if (ctx && is_sticky(rc)) ctx->sticky = true;
    if (rc == CUDA_ERROR_OUT_OF_MEMORY) return KTC_ERR_OOM;
    if (is_sticky(rc) || rc == CUDA_ERROR_LAUNCH_OUT_OF_RESOURCES) return KTC_ERR_LAUNCH;
    return KTC_ERR_CUDA;
}

int make_current(ktc_ctx* ctx) {
    if (!ctx) {
        set_error("null context");
        return KTC_ERR_INVALID;
    }
    CUresult rc = driver().cuCtxSetCurrent(ctx->cu);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(ctx, rc, "cuCtxSetCurrent");
}

CUresult launch(ktc_ctx* ctx, CUfunction fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                unsigned by, unsigned bz, unsigned smem, void** params) {
    ++ctx->launches;
    return driver().cuLaunchKernel(fn, gx, gy, gz, bx, by, bz, smem, ctx->stream, params, nullptr);
}

// Longest a configuration's launches may run before it is declared hung
// (runtime_error, context reset): KTC_WATCHDOG_S, default 30 s.
double watchdog_seconds() {
    static const double s = [] {
        const char* e = std::getenv("KTC_WATCHDOG_S");
        const double v = e ? std::atof(e) : 0.0;
        return v > 0.0 ? v : 30.0;
    }();
    return s;
}

CUresult wait_event(ktc_ctx* ctx, CUevent ev, double timeout_s) {
    const Driver& d = driver();
    auto t0 = std::chrono::steady_clock::now();
    int spins = 0;
    for (;;) {
        CUresult rc = d.cuEventQuery(ev);
        if (rc != CUDA_ERROR_NOT_READY) return rc;
        if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
        double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > timeout_s) {
            ctx->sticky = true;  // a hung kernel: only a context reset recovers
            return CUDA_ERROR_LAUNCH_TIMEOUT;
        }
    }
}

int flush_l2(ktc_ctx* ctx) {
    const Driver& d = driver();
    if (!ctx->flush_buf) {
        // Twice the L2, at least 256 MiB: every resident line is displaced.
        size_t bytes = std::max<size_t>(2 * ctx->limits.l2_bytes, size_t(256) << 20);
        CUresult rc = d.cuMemAlloc(&ctx->flush_buf, bytes);
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuMemAlloc(L2 flush buffer)");
        rc = d.cuMemsetD32Async(ctx->flush_buf, 0, bytes / 4, ctx->stream);
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuMemsetD32Async");
        ctx->flush_bytes = bytes;
    }
    unsigned long long n4 = ctx->flush_bytes / 16;
    CUdeviceptr sink = ctx->scratch;
    void* params[] = {&ctx->flush_buf, &n4, &sink};
    CUresult rc = launch(ctx, ctx->fn_flush, unsigned(ctx->limits.sm_count * 4), 1, 1, 512, 1, 1,
                         0, params);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(ctx, rc, "L2 flush launch");
}

void merge_reports(ktc_verify_report* t, const ktc_verify_report& r, bool nan_abs, bool nan_rel,
                   size_t k) {
    if (t->pass) {
        if (!r.pass) {
            t->pass = 0;
            t->buffer_index = k;
            t->element_index = r.element_index;
        } else if (r.max_abs_error > t->max_abs_error) {
            t->buffer_index = k;
            t->element_index = r.element_index;
        }
    }
    // A NaN inside buffer k restarts the running max there (r already holds
    // the post-restart value); a NaN carried in from earlier buffers is
    // replaced by buffer k's first element and so by r's max.
    if (nan_abs || std::isnan(t->max_abs_error)) t->max_abs_error = r.max_abs_error;
    else t->max_abs_error = std::max(t->max_abs_error, r.max_abs_error);
    if (nan_rel || std::isnan(t->max_rel_error)) t->max_rel_error = r.max_rel_error;
    else t->max_rel_error = std::max(t->max_rel_error, r.max_rel_error);
    t->elements_compared += r.elements_compared;
}

int verify_pair(ktc_ctx* ctx, CUdeviceptr cand, CUdeviceptr ref, size_t count, int type, double rel,
                double abs, ktc_verify_report* out, bool* had_nan_abs, bool* had_nan_rel) {
    const Driver& d = driver();
    if (had_nan_abs) *had_nan_abs = false;
    if (had_nan_rel) *had_nan_rel = false;
    std::memset(out, 0, sizeof(*out));
    out->pass = 1;
    out->elements_compared = count;
    if (count == 0) return KTC_OK;
    unsigned long long n = count;
    int is_f32 = type == KTC_F32 ? 1 : 0;
    unsigned blocks =
        static_cast<unsigned>(std::min<size_t>(ctx->verify_blocks, (count + 255) / 256));
    CUdeviceptr partials = ctx->scratch + 256;
    CUdeviceptr result = ctx->scratch + 128;
    void* p1[] = {&cand, &ref, &n, &is_f32, &rel, &abs, &partials};
    CUresult rc = launch(ctx, ctx->fn_verify_partial, blocks, 1, 1, 256, 1, 1, 0, p1);
    if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "verify launch");
    int nb = static_cast<int>(blocks);
    void* p2[] = {&partials, &nb, &result};
    rc = launch(ctx, ctx->fn_verify_final, 1, 1, 1, 256, 1, 1, 0, p2);
    if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "verify launch");
    KtcVerifyPartial vp;
    rc = d.cuMemcpyDtoHAsync(&vp, result, sizeof(vp), ctx->stream);
    if (rc == CUDA_SUCCESS) rc = d.cuStreamSynchronize(ctx->stream);
    if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "verify readback");

    const unsigned long long none = ~0ull;
    out->pass = vp.first_fail == none ? 1 : 0;
    double max_abs = vp.max_abs < 0.0 ? 0.0 : vp.max_abs;
    double max_rel = vp.max_rel < 0.0 ? 0.0 : vp.max_rel;
    // tuner.hpp:53-62: a NaN error replaces the running maximum, and the
    // next element replaces the NaN unconditionally -- so the reported
    // maximum is the max over the suffix after the LAST NaN (NaN if none).
    const long long last = static_cast<long long>(count) - 1;
    if (had_nan_abs) *had_nan_abs = vp.nan_abs >= 0;
    if (had_nan_rel) *had_nan_rel = vp.nan_rel >= 0;
    if (vp.nan_abs >= 0 || vp.nan_rel >= 0) {
        long long abs_start = vp.nan_abs >= 0 ? vp.nan_abs : -1;
        long long rel_start = vp.nan_rel >= 0 ? vp.nan_rel : -1;
        KtcVerifyPartial after{};
        if ((vp.nan_abs >= 0 && vp.nan_abs < last) || (vp.nan_rel >= 0 && vp.nan_rel < last)) {
            void* p3[] = {&cand, &ref, &n, &is_f32, &abs_start, &rel_start, &partials};
            rc = launch(ctx, ctx->fn_verify_after, blocks, 1, 1, 256, 1, 1, 0, p3);
            if (rc == CUDA_SUCCESS) rc = launch(ctx, ctx->fn_verify_final, 1, 1, 1, 256, 1, 1, 0, p2);
            if (rc == CUDA_SUCCESS)
                rc = d.cuMemcpyDtoHAsync(&after, result, sizeof(after), ctx->stream);
            if (rc == CUDA_SUCCESS) rc = d.cuStreamSynchronize(ctx->stream);
            if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "verify (NaN suffix pass)");
        }
        const double qnan = std::numeric_limits<double>::quiet_NaN();
        if (vp.nan_abs >= 0) max_abs = vp.nan_abs == last ? qnan : std::max(0.0, after.max_abs);
        if (vp.nan_rel >= 0) max_rel = vp.nan_rel == last ? qnan : std::max(0.0, after.max_rel);
        // A NaN element after the suffix start... cannot exist (nan_* is the
        // last NaN), so the suffix maxima above are over finite errors only.
    }
    out->max_abs_error = max_abs;
    out->max_rel_error = max_rel;
    if (!out->pass) out->element_index = static_cast<size_t>(vp.first_fail);
    else out->element_index = (max_abs > 0.0 && vp.argmax != none) ? size_t(vp.argmax) : 0;
    out->buffer_index = 0;
    return KTC_OK;
}

}  // namespace ktc

using namespace ktc;

void ktc::retire_module(ktc_ctx* ctx, CUmodule mod) {
    ctx->retired.push_back(mod);
    if (ctx->retired.size() <= kRetiredCap) return;
    const Driver& d = driver();
    d.cuCtxSetCurrent(ctx->cu);
    const size_t half = ctx->retired.size() / 2;
    for (size_t i = 0; i < half; ++i) d.cuModuleUnload(ctx->retired[i]);
    ctx->retired.erase(ctx->retired.begin(), ctx->retired.begin() + long(half));
}

extern "C" {

int ktc_abi_version(void) { return KTC_ABI_VERSION; }

const char* ktc_status_name(int status) {
    switch (status) {
        case KTC_STATUS_SUCCESS: return "ok";
        case KTC_STATUS_COMPILE_ERROR: return "compile_error";
        case KTC_STATUS_RUNTIME_ERROR: return "runtime_error";
        case KTC_STATUS_MISSING: return "missing";
    }
    return "?";
}

const char* ktc_last_error(const void*) { return last_error().c_str(); }

int ktc_device_count(int* count) {
    *count = 0;
    const Driver& d = driver();
    if (!d.ok) {
        set_error(d.error);
        return KTC_ERR_NO_DRIVER;
    }
    CUresult rc = d.cuDeviceGetCount(count);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(nullptr, rc, "cuDeviceGetCount");
}

static int query_limits(ktc_ctx* c) {
    const Driver& d = driver();
    ktc_limits& L = c->limits;
    std::memset(&L, 0, sizeof(L));
    L.ordinal = c->ordinal;
    d.cuDeviceGetName(L.name, sizeof(L.name), c->dev);
    auto attr = [&](CUdevice_attribute a) {
        int v = 0;
        d.cuDeviceGetAttribute(&v, a, c->dev);
        return v;
    };
    L.cc_major = attr(CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR);
    L.cc_minor = attr(CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR);
    L.sm_count = attr(CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT);
    L.max_threads_per_block = attr(CU_DEVICE_ATTRIBUTE_MAX_THREADS_PER_BLOCK);
    L.max_block_dim[0] = attr(CU_DEVICE_ATTRIBUTE_MAX_BLOCK_DIM_X);
    L.max_block_dim[1] = attr(CU_DEVICE_ATTRIBUTE_MAX_BLOCK_DIM_Y);
    L.max_block_dim[2] = attr(CU_DEVICE_ATTRIBUTE_MAX_BLOCK_DIM_Z);
    L.max_grid_dim[0] = attr(CU_DEVICE_ATTRIBUTE_MAX_GRID_DIM_X);
    L.max_grid_dim[1] = attr(CU_DEVICE_ATTRIBUTE_MAX_GRID_DIM_Y);
    L.max_grid_dim[2] = attr(CU_DEVICE_ATTRIBUTE_MAX_GRID_DIM_Z);
    L.smem_per_block_optin = size_t(attr(CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN));
    L.smem_per_sm = size_t(attr(CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_MULTIPROCESSOR));
    L.l2_bytes = size_t(attr(CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE));
    size_t total = 0;
    d.cuDeviceTotalMem(&total, c->dev);
    L.global_mem_bytes = total;
    L.sm_clock_khz = attr(CU_DEVICE_ATTRIBUTE_CLOCK_RATE);
    L.mem_clock_khz = attr(CU_DEVICE_ATTRIBUTE_MEMORY_CLOCK_RATE);
    L.mem_bus_width_bits = attr(CU_DEVICE_ATTRIBUTE_GLOBAL_MEMORY_BUS_WIDTH);
    L.peak_fp32_gflops = double(L.sm_count) * 128.0 * 2.0 * L.sm_clock_khz * 1e-6;
    L.peak_hbm_gbs = 2.0 * L.mem_clock_khz * 1e3 * (L.mem_bus_width_bits / 8.0) * 1e-9;
    return KTC_OK;
}

static int setup_ctx(ktc_ctx* c) {
    const Driver& d = driver();
    CUresult rc = d.cuDevicePrimaryCtxRetain(&c->cu, c->dev);
    if (rc != CUDA_SUCCESS) return fail_cu(c, rc, "cuDevicePrimaryCtxRetain");
    rc = d.cuCtxSetCurrent(c->cu);
    if (rc != CUDA_SUCCESS) return fail_cu(c, rc, "cuCtxSetCurrent");
    rc = d.cuStreamCreate(&c->stream, CU_STREAM_NON_BLOCKING);
    if (rc != CUDA_SUCCESS) return fail_cu(c, rc, "cuStreamCreate");
    rc = d.cuModuleLoadData(&c->builtin, ktc_builtin_cubin);
    if (rc != CUDA_SUCCESS) return fail_cu(c, rc, "cuModuleLoadData(builtin)");
    struct {
        CUfunction* fn;
        const char* name;
    } fns[] = {{&c->fn_conv_ref, "ktc_conv_reference"},
               {&c->fn_gemm_ref, "ktc_gemm_reference"},
               {&c->fn_verify_partial, "ktc_verify_partial"},
               {&c->fn_verify_final, "ktc_verify_final"},
               {&c->fn_verify_after, "ktc_verify_after"},
               {&c->fn_flush, "ktc_l2_flush"}};
    for (auto& f : fns) {
        rc = d.cuModuleGetFunction(f.fn, c->builtin, f.name);
        if (rc != CUDA_SUCCESS) return fail_cu(c, rc, f.name);
    }
    query_limits(c);
    // One full wave of verifier blocks (a partial second wave would run the
    // tail of both HBM streams at a fraction of the bandwidth).
    int per_sm = 0;
    if (d.cuOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c->fn_verify_partial, 256, 0) !=
            CUDA_SUCCESS ||
        per_sm < 1)
        per_sm = 2;
    c->verify_blocks = std::max(1, c->limits.sm_count * per_sm);
    size_t scratch = 256 + sizeof(KtcVerifyPartial) * size_t(c->verify_blocks);
    rc = d.cuMemAlloc(&c->scratch, scratch);
    if (rc != CUDA_SUCCESS) return fail_cu(c, rc, "cuMemAlloc(scratch)");
    c->sticky = false;
    c->epoch = ktc::primary_ctx_epoch();
    return KTC_OK;
}

static std::atomic<unsigned> g_primary_epoch{0};
}  // extern "C"
unsigned ktc::primary_ctx_epoch() { return g_primary_epoch.load(); }
bool ktc::trace_on() {
    static const bool on = [] {
        const char* e = std::getenv("KTC_TRACE");
        return e && std::strcmp(e, "0") != 0;
    }();
    return on;
}
void ktc::trace_phase(const char* what, std::chrono::steady_clock::time_point since) {
    if (!trace_on()) return;
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - since).count();
    std::fprintf(stderr, "ktc-trace %-28s %9.2f ms\n", what, ms);
}
extern "C" {

}  // extern "C"
CUresult ktc::ctx_alloc(ktc_ctx* ctx, size_t bytes, CUdeviceptr* p) {
    if (!bytes) bytes = 4;
    for (size_t i = 0; i < ctx->free_blocks.size(); ++i)
        if (ctx->free_blocks[i].first == bytes) {
            *p = ctx->free_blocks[i].second;
            ctx->free_bytes -= bytes;
            ctx->free_blocks.erase(ctx->free_blocks.begin() + long(i));
            return CUDA_SUCCESS;
        }
    CUresult rc = driver().cuMemAlloc(p, bytes);
    if (rc == CUDA_ERROR_OUT_OF_MEMORY && !ctx->free_blocks.empty()) {
        for (auto& b : ctx->free_blocks) driver().cuMemFree(b.second);
        ctx->free_blocks.clear();
        ctx->free_bytes = 0;
        rc = driver().cuMemAlloc(p, bytes);
    }
    return rc;
}

void ktc::ctx_free(ktc_ctx* ctx, CUdeviceptr p, size_t bytes) {
    if (!p) return;
    if (!bytes) bytes = 4;
    constexpr size_t kCacheCap = size_t(2) << 30;
    if (ctx->sticky) return;  // died with the context
    if (ctx->free_bytes + bytes <= kCacheCap) {
        ctx->free_blocks.emplace_back(bytes, p);
        ctx->free_bytes += bytes;
    } else {
        driver().cuMemFree(p);
    }
}
extern "C" {

static void teardown_ctx(ktc_ctx* c, bool reset) {
    const Driver& d = driver();
    if (!c->cu) return;
    if (!reset) {
        d.cuCtxSetCurrent(c->cu);
        for (CUmodule m : c->retired) d.cuModuleUnload(m);
    }
    c->retired.clear();
    const auto t0 = std::chrono::steady_clock::now();
    if (!reset)
        for (auto& b : c->free_blocks) d.cuMemFree(b.second);
    c->free_blocks.clear();
    c->free_bytes = 0;
    d.cuCtxSetCurrent(c->cu);
    if (!reset) {
        for (CUevent e : c->events) d.cuEventDestroy(e);
        if (c->flush_buf) d.cuMemFree(c->flush_buf);
        if (c->scratch) d.cuMemFree(c->scratch);
        if (c->builtin) d.cuModuleUnload(c->builtin);
        if (c->stream) d.cuStreamDestroy(c->stream);
    }
    c->events.clear();
    c->flush_buf = c->scratch = 0;
    c->flush_bytes = 0;
    c->builtin = nullptr;
    c->stream = nullptr;
    c->ref = 0;
    c->ref_count = 0;
    ktc::trace_phase("teardown: frees", t0);
    if (reset) {
        d.cuDevicePrimaryCtxReset(c->dev);
        g_primary_epoch.fetch_add(1);
    }
    else d.cuDevicePrimaryCtxRelease(c->dev);
    ktc::trace_phase("teardown: + ctx release", t0);
    c->cu = nullptr;
}

// Context pool: a closed context (stream, builtin module, verifier
// scratch, L2-flush buffer, cached device blocks) is kept for the next
// ktc_open of the same device, so a new tuning job pays none of that setup.
// Contexts made before a primary-context reset are dropped (their resources
// died with it).
static std::mutex g_pool_mu;
static std::vector<ktc_ctx*> g_pool;

static ktc_ctx* take_pooled(int ordinal) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (size_t i = 0; i < g_pool.size(); ++i) {
        ktc_ctx* c = g_pool[i];
        if (c->ordinal != ordinal) continue;
        g_pool.erase(g_pool.begin() + long(i));
        if (c->epoch != ktc::primary_ctx_epoch()) {
            driver().cuDevicePrimaryCtxRelease(c->dev);
            delete c;
            return nullptr;
        }
        driver().cuCtxSetCurrent(c->cu);
        c->ref = 0;
        c->ref_count = 0;
        c->launches = 0;
        return c;
    }
    return nullptr;
}

static bool pool_ctx(ktc_ctx* c) {
    if (c->sticky || !c->cu || c->epoch != ktc::primary_ctx_epoch()) return false;
    const char* e = std::getenv("KTC_CTX_POOL");
    if (e && std::strcmp(e, "0") == 0) return false;
    driver().cuCtxSetCurrent(c->cu);
    if (driver().cuStreamSynchronize(c->stream) != CUDA_SUCCESS) return false;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    int same = 0;
    for (ktc_ctx* p : g_pool) same += p->ordinal == c->ordinal;
    if (same >= 2) return false;
    g_pool.push_back(c);
    return true;
}

int ktc_open(int ordinal, ktc_ctx** out) {
    *out = nullptr;
    const Driver& d = driver();
    if (!d.ok) {
        set_error(d.error);
        return KTC_ERR_NO_DRIVER;
    }
    int count = 0;
    d.cuDeviceGetCount(&count);
    if (ordinal < 0 || ordinal >= count) {
        set_error("device ordinal " + std::to_string(ordinal) + " out of range (" +
                  std::to_string(count) + " devices)");
        return KTC_ERR_NO_DEVICE;
    }
    if (ktc_ctx* pooled = take_pooled(ordinal)) {
        *out = pooled;
        return KTC_OK;
    }
    auto* c = new ktc_ctx;
    c->ordinal = ordinal;
    CUresult rc = d.cuDeviceGet(&c->dev, ordinal);
    if (rc != CUDA_SUCCESS) {
        delete c;
        return fail_cu(nullptr, rc, "cuDeviceGet");
    }
    int st = setup_ctx(c);
    if (st != KTC_OK) {
        teardown_ctx(c, false);
        delete c;
        return st;
    }
    *out = c;
    return KTC_OK;
}

void ktc_close(ktc_ctx* ctx) {
    if (!ctx) return;
    if (pool_ctx(ctx)) return;
    teardown_ctx(ctx, false);
    delete ctx;
}

int ktc_query_limits(ktc_ctx* ctx, ktc_limits* out) {
    if (!ctx) return KTC_ERR_INVALID;
    *out = ctx->limits;
    return KTC_OK;
}

int ktc_reset(ktc_ctx* ctx) {
    if (!ctx) return KTC_ERR_INVALID;
    teardown_ctx(ctx, true);
    return setup_ctx(ctx);
}

void ktc_free_host(void* p) { std::free(p); }

int ktc_load(ktc_ctx* ctx, const void* cubin, size_t, const char* kernel_name, ktc_fn** fn) {
    *fn = nullptr;
    int st = make_current(ctx);
    if (st) return st;
    const Driver& d = driver();
    auto* f = new ktc_fn;
    f->ctx = ctx;
    CUresult rc = d.cuModuleLoadData(&f->mod, cubin);
    if (rc != CUDA_SUCCESS) {
        delete f;
        return fail_cu(ctx, rc, "cuModuleLoadData");
    }
    rc = d.cuModuleGetFunction(&f->fn, f->mod, kernel_name);
    if (rc != CUDA_SUCCESS) {
        d.cuModuleUnload(f->mod);
        delete f;
        return fail_cu(ctx, rc, "cuModuleGetFunction");
    }
    *fn = f;
    return KTC_OK;
}

void ktc_unload(ktc_fn* fn) {
    if (!fn) return;
    if (fn->ctx && fn->ctx->cu && !fn->ctx->sticky) {
        driver().cuCtxSetCurrent(fn->ctx->cu);
        driver().cuModuleUnload(fn->mod);
    }
    delete fn;
}

int ktc_set_symbol(ktc_fn* fn, const char* symbol, const void* src, size_t bytes) {
    int st = make_current(fn->ctx);
    if (st) return st;
    const Driver& d = driver();
    CUdeviceptr p = 0;
    size_t size = 0;
    CUresult rc = d.cuModuleGetGlobal(&p, &size, fn->mod, symbol);
    if (rc != CUDA_SUCCESS) return fail_cu(fn->ctx, rc, "cuModuleGetGlobal");
    if (bytes > size) {
        set_error(std::string("symbol ") + symbol + " is smaller than the data");
        return KTC_ERR_INVALID;
    }
    rc = d.cuMemcpyHtoD(p, src, bytes);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(fn->ctx, rc, "cuMemcpyHtoD(symbol)");
}

int ktc_alloc(ktc_ctx* ctx, size_t bytes, ktc_buf* out) {
    int st = make_current(ctx);
    if (st) return st;
    CUdeviceptr p = 0;
    CUresult rc = driver().cuMemAlloc(&p, bytes ? bytes : 4);
    if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuMemAlloc");
    *out = p;
    return KTC_OK;
}

int ktc_free(ktc_ctx* ctx, ktc_buf buf) {
    int st = make_current(ctx);
    if (st) return st;
    CUresult rc = driver().cuMemFree(buf);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(ctx, rc, "cuMemFree");
}

int ktc_upload(ktc_ctx* ctx, ktc_buf dst, const void* src, size_t bytes) {
    int st = make_current(ctx);
    if (st) return st;
    CUresult rc = driver().cuMemcpyHtoD(dst, src, bytes);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(ctx, rc, "cuMemcpyHtoD");
}

int ktc_upload_pitched(ktc_ctx* ctx, ktc_buf dst, size_t dst_pitch, const void* src,
                       size_t src_pitch, size_t width_bytes, size_t rows) {
    int st = make_current(ctx);
    if (st) return st;
    CUDA_MEMCPY2D m;
    std::memset(&m, 0, sizeof(m));
    m.srcMemoryType = CU_MEMORYTYPE_HOST;
    m.srcHost = src;
    m.srcPitch = src_pitch;
    m.dstMemoryType = CU_MEMORYTYPE_DEVICE;
    m.dstDevice = dst;
    m.dstPitch = dst_pitch;
    m.WidthInBytes = width_bytes;
    m.Height = rows;
    CUresult rc = driver().cuMemcpy2D(&m);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(ctx, rc, "cuMemcpy2D");
}

int ktc_download(ktc_ctx* ctx, void* dst, ktc_buf src, size_t bytes) {
    int st = make_current(ctx);
    if (st) return st;
    CUresult rc = driver().cuMemcpyDtoHAsync(dst, src, bytes, ctx->stream);
    if (rc == CUDA_SUCCESS) rc = driver().cuStreamSynchronize(ctx->stream);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(ctx, rc, "cuMemcpyDtoH");
}

int ktc_memset32(ktc_ctx* ctx, ktc_buf dst, uint32_t value, size_t count) {
    int st = make_current(ctx);
    if (st) return st;
    CUresult rc = driver().cuMemsetD32Async(dst, value, count, ctx->stream);
    if (rc == CUDA_SUCCESS) rc = driver().cuStreamSynchronize(ctx->stream);
    return rc == CUDA_SUCCESS ? KTC_OK : fail_cu(ctx, rc, "cuMemsetD32");
}

int ktc_launch_timed(ktc_ctx* ctx, ktc_fn* fn, const unsigned grid[3], const unsigned block[3],
                     unsigned smem_bytes, void** params, int warmup, int reps, int flush,
                     float* best_ms, float* all_ms) {
    int st = make_current(ctx);
    if (st) return st;
    const Driver& d = driver();
    if (reps < 1) reps = 1;
    while (ctx->events.size() < size_t(2 * reps)) {
        CUevent e;
        CUresult rc = d.cuEventCreate(&e, CU_EVENT_DEFAULT);
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuEventCreate");
        ctx->events.push_back(e);
    }
    if (smem_bytes > 48 * 1024) {
        CUresult rc = d.cuFuncSetAttribute(fn->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                           int(smem_bytes));
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuFuncSetAttribute(dynamic smem)");
    }
    CUresult rc = CUDA_SUCCESS;
    for (int w = 0; w < warmup && rc == CUDA_SUCCESS; ++w)
        rc = launch(ctx, fn->fn, grid[0], grid[1], grid[2], block[0], block[1], block[2],
                    smem_bytes, params);
    if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuLaunchKernel (warm-up)");
    if (flush == 2) {
        // Stream timing: the repetitions back to back between ONE event
        // pair (no L2 flushes, no events between launches); every
        // repetition's time is the mean launch duration of the stream.
        rc = d.cuEventRecord(ctx->events[0], ctx->stream);
        for (int r = 0; r < reps && rc == CUDA_SUCCESS; ++r)
            rc = launch(ctx, fn->fn, grid[0], grid[1], grid[2], block[0], block[1], block[2],
                        smem_bytes, params);
        if (rc == CUDA_SUCCESS) rc = d.cuEventRecord(ctx->events[1], ctx->stream);
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuLaunchKernel");
        rc = wait_event(ctx, ctx->events[1], watchdog_seconds());
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "kernel execution");
        float total = 0.0f;
        rc = d.cuEventElapsedTime(&total, ctx->events[0], ctx->events[1]);
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuEventElapsedTime");
        const float mean = total / float(reps);
        if (all_ms)
            for (int r = 0; r < reps; ++r) all_ms[r] = mean;
        *best_ms = mean;
        return KTC_OK;
    }
    for (int r = 0; r < reps; ++r) {
        if (flush) {
            st = flush_l2(ctx);
            if (st) return st;
        }
        rc = d.cuEventRecord(ctx->events[2 * r], ctx->stream);
        if (rc == CUDA_SUCCESS)
            rc = launch(ctx, fn->fn, grid[0], grid[1], grid[2], block[0], block[1], block[2],
                        smem_bytes, params);
        if (rc == CUDA_SUCCESS) rc = d.cuEventRecord(ctx->events[2 * r + 1], ctx->stream);
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuLaunchKernel");
    }
    rc = wait_event(ctx, ctx->events[2 * reps - 1], watchdog_seconds());
    if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "kernel execution");
    float best = std::numeric_limits<float>::infinity();
    for (int r = 0; r < reps; ++r) {
        float ms = 0.0f;
        rc = d.cuEventElapsedTime(&ms, ctx->events[2 * r], ctx->events[2 * r + 1]);
        if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuEventElapsedTime");
        if (all_ms) all_ms[r] = ms;
        best = std::min(best, ms);
    }
    *best_ms = best;
    return KTC_OK;
}

// ktc_launch_timed with an early-out: when `bar` > 0 the first warm-up
// launch is flushed, timed and waited for (the probe); if it took longer
// than `bar` ms that launch is the result (*reps_done = 1).  Otherwise the
// timed repetitions follow with one warm-up fewer (the probe was one).
int ktc_launch_timed_pruned(ktc_ctx* ctx, ktc_fn* fn, const unsigned grid[3],
                            const unsigned block[3], unsigned smem_bytes, void** params, int warmup,
                            int reps, int flush, double bar, float* best_ms, float* all_ms,
                            int* reps_done) {
    *reps_done = reps < 1 ? 1 : reps;
    if (!(bar > 0.0) || reps <= 1)
        return ktc_launch_timed(ctx, fn, grid, block, smem_bytes, params, warmup, reps, flush,
                                best_ms, all_ms);
    // The warm-up launch doubles as the probe: flushed and timed like a
    // repetition.  Over the bar, the configuration is done after one launch
    // (its row time is that launch); otherwise the `reps` timed repetitions
    // follow as usual and the probe only served as the warm-up.
    float probe = 0.0f;
    int st = ktc_launch_timed(ctx, fn, grid, block, smem_bytes, params, 0, 1, flush, &probe, nullptr);
    if (st) return st;
    if (double(probe) > bar) {
        *best_ms = probe;
        if (all_ms) all_ms[0] = probe;
        *reps_done = 1;
        return KTC_OK;
    }
    return ktc_launch_timed(ctx, fn, grid, block, smem_bytes, params, std::max(0, warmup - 1), reps,
                            flush, best_ms, all_ms);
}

int ktc_bind_reference(ktc_ctx* ctx, ktc_buf ref, size_t count, int elem_type, double rel_tol,
                       double abs_tol) {
    if (!ctx) return KTC_ERR_INVALID;
    ctx->ref = ref;
    ctx->ref_count = count;
    ctx->ref_type = elem_type;
    ctx->rel_tol = rel_tol;
    ctx->abs_tol = abs_tol;
    return KTC_OK;
}

int ktc_verify(ktc_ctx* ctx, ktc_buf cand, ktc_verify_report* out) {
    int st = make_current(ctx);
    if (st) return st;
    if (!ctx->ref) {
        set_error("no reference bound (ktc_bind_reference)");
        return KTC_ERR_INVALID;
    }
    return verify_pair(ctx, cand, ctx->ref, ctx->ref_count, ctx->ref_type, ctx->rel_tol,
                       ctx->abs_tol, out);
}

int ktc_verify_pair(ktc_ctx* ctx, ktc_buf cand, ktc_buf ref, size_t count, int elem_type,
                    double rel_tol, double abs_tol, ktc_verify_report* out) {
    int st = make_current(ctx);
    if (st) return st;
    return verify_pair(ctx, cand, ref, count, elem_type, rel_tol, abs_tol, out);
}

uint64_t ktc_digest_words(const void* data, size_t n_words) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    uint64_t h = 0xcbf29ce484222325ull;
    const size_t n = n_words * 4;
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

int ktc_fill_uniform_f32(uint64_t seed, float* out, size_t n, int threads) {
    if (!out && n) return KTC_ERR_INVALID;
    try {
        ktb::fill_uniform_f32(seed, out, n, threads);
    } catch (const std::exception& e) {
        set_error(e.what());
        return KTC_ERR_INVALID;
    }
    return KTC_OK;
}

void ktc_digest_hex(uint64_t digest, char out[17]) {
    static const char* hex = "0123456789abcdef";
    for (int i = 15; i >= 0; --i) {
        out[i] = hex[digest & 0xf];
        digest >>= 4;
    }
    out[16] = '\0';
}

}  // extern "C"
