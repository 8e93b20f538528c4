// backend.cpp -- ktc.h layer 2: ktune::Backend::evaluate on the B200.
//
// One evaluation: cubin from the NVRTC pool (compiled from the
// family source with the configuration as -D defines) -> cuModuleLoadData ->
// launch geometry from the request (grid = ceil(global/local), block =
// local) -> output poisoned with NaN -> 1 warm-up + R timed launches (CUDA
// events, L2 flushed before each) -> device verification of the output
// against the bound reference -> ktc_result.
//
// Inputs are materialized from the request's recipes once per argument list
// (std::mt19937_64, bit-identical to the reference), uploaded in the family's
// device layout, and the family's device reference (builtin.cu, bit-identical
// to the CPU oracle) is computed right after upload.
#include <cuda.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <thread>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "core.hpp"
#include "isolate.hpp"
#include "ktb/arguments.hpp"
#include "compile_service.hpp"

namespace {

#include "kernel_sources.inc"  // kConvSource, kGemmSource, kGemmTf32Source

using namespace ktc;
using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

enum Family { FAM_CONV, FAM_GEMM, FAM_GEMM_TF32, FAM_CUSTOM };

size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

// Device-resident inputs, outputs and reference of one argument list.
struct Inputs {
    std::string sig;
    Family fam = FAM_CUSTOM;
    // conv
    int X = 0, Y = 0, F = 0, ipitch = 0, rows = 0;
    float W = 1.0f;
    std::vector<float> taps;
    // gemm
    int M = 0, N = 0, K = 0;
    float alpha = 1.0f, beta = 0.0f;
    // all: device copy per argument (0 for scalars) and the argument list
    std::vector<ktb::ArgumentSpec> args;
    std::vector<CUdeviceptr> dev;
    std::vector<size_t> bytes;
    // outputs (in argument order): candidate buffer, reference buffer
    std::vector<int> out_arg;
    std::vector<CUdeviceptr> out, ref;
    std::vector<size_t> out_count;
    std::vector<int> out_type;
    bool has_reference = false;
    std::vector<std::string> ref_digest;  // lazily computed
    double best_verified_ms = 0.0;        // prune_factor bar (0 = none yet)
};

struct Plan {
    const KernelSource* ksrc = nullptr;
    Defines problem;  // shared by every configuration of a compile batch
    Defines config;
    unsigned grid[3] = {1, 1, 1}, block[3] = {1, 1, 1};
    unsigned smem = 0;
    int tma_mode = 0;  // 1: conv halo tile box (BW x BH); 2: tf32 A/B operand boxes
    double rel_tol = -1.0;  // family tolerance override (< 0: backend options)
    unsigned box[2] = {0, 0};
    double compile_cost = 1.0;  // relative NVRTC cost estimate (CompileService ordering)
    // SGEMM TAILK: 1-D grid of whole tiles + K-split tail tiles (ptxgen_gemm.cpp)
    bool tailk = false;
    bool sk = false;  // SGEMM stream-K (ptxgen_gemm SK)
    unsigned tiles_x = 0, tiles_y = 0, ktiles = 0, tile_floats = 0, ktile_k = 0, cg = 1;
};

// Relative NVRTC cost of a kernel whose fully unrolled body holds `n` FMAs
// per thread (1 ~ 100 ms on the GPU box).  NVVM's optimizer grows
// super-linearly with the unrolled body (measured: 11x11 taps with 8x8
// outputs/thread, 7,744 FMAs, ~6.9 s; 3x3 with 8x8, 576, ~0.45 s).
double unrolled_cost(double n) { return 1.0 + n / 200.0 + (n / 2000.0) * (n / 2000.0); }

std::string define(const char* name, long long v) {
    return std::string(name) + "=" + std::to_string(v);
}

// The conv family's code path: "ptx" (default) = the direct PTX generator
// (ptxgen_conv.cpp, ptxas only), "nvrtc" = kernels/conv.cu through NVRTC.
// KTC_CONV_CODEGEN overrides; both produce the same kernels.
const KernelSource& conv_source() {
    static const KernelSource s = [] {
        const char* e = std::getenv("KTC_CONV_CODEGEN");
        const std::string mode = e ? e : "ptx";
        KernelSource k = split_source("conv.cu", kConvSource, "conv2d");
        if (mode == "ptx") {
            k.id = "ptxgen-conv#1|" + k.id;
            k.ptx_generator = conv_ptx_module;
        }
        return k;
    }();
    return s;
}
// The SGEMM family's code path: "ptx" (default) = ptxgen_gemm.cpp, "nvrtc"
// = kernels/gemm.cu through NVRTC.  KTC_GEMM_CODEGEN overrides.
const KernelSource& gemm_source() {
    static const KernelSource s = [] {
        const char* e = std::getenv("KTC_GEMM_CODEGEN");
        const std::string mode = e ? e : "ptx";
        KernelSource k = split_source("gemm.cu", kGemmSource, "gemm");
        if (mode == "ptx") {
            k.id = "ptxgen-gemm#1|" + k.id;
            k.ptx_generator = gemm_ptx_module;
        }
        return k;
    }();
    return s;
}
const KernelSource& tf32_source() {
    static const KernelSource s = split_source("gemm_tf32.cu", kGemmTf32Source, "gemm_tf32");
    return s;
}

// Loaded modules, most recently used last (a batch cubin serves several
// configurations; c_taps is set once per module and argument list).
struct ModuleEntry {
    CubinPtr cubin;
    CUmodule mod = nullptr;
    std::string taps_sig;
};

}  // namespace

struct ktc_backend {
    ktc::RemoteBackend* remote = nullptr;  // isolated: every call goes to a worker process
    ktc_ctx* ctx = nullptr;
    ktc_backend_options opts{};
    std::string name;
    std::string cache_dir;
    std::unique_ptr<Inputs> in;
    std::map<std::string, KernelSource> custom_sources;  // path -> source
    std::vector<ModuleEntry> modules;
    // SGEMM TAILK scratch: partial tiles of the split tail and their arrival
    // counters (zeroed on allocation; every tile's last split resets its own).
    CUdeviceptr tail_ws = 0, tail_cnt = 0;
    size_t tail_ws_bytes = 0, tail_cnt_bytes = 0;
    // Host copy of the reference bound by ktc_backend_set_reference, so it
    // survives a context reset (a sticky fault frees every device buffer;
    // the inputs are rebuilt and the reference re-uploaded).
    struct BoundReference {
        std::string sig;
        std::vector<std::vector<unsigned char>> bytes;
        std::vector<size_t> lengths;
        std::vector<int> types;
    } bound;
};

namespace {

// ---------------------------------------------------------------------------
// Request helpers
// ---------------------------------------------------------------------------

struct ParamView {
    const ktc_request* r;
    bool get(const char* name, long long* v) const {
        for (int i = 0; i < r->n_params; ++i)
            if (std::strcmp(r->param_names[i], name) == 0) {
                *v = r->param_values[i];
                return true;
            }
        return false;
    }
};

Family family_of(const char* name) {
    std::string n = name ? name : "";
    if (n == "conv") return FAM_CONV;
    if (n == "gemm") return FAM_GEMM;
    if (n == "gemm_tf32") return FAM_GEMM_TF32;
    return FAM_CUSTOM;
}

std::string signature(const ktc_request* r) {
    std::ostringstream s;
    s << (r->kernel_name ? r->kernel_name : "") << '|' << (r->source_ref ? r->source_ref : "");
    for (int i = 0; i < r->n_args; ++i) {
        const ktc_arg& a = r->args[i];
        s << '|' << a.role << ',' << a.type << ',' << a.length << ',';
        s.precision(17);
        s << a.value << ',' << (a.fill ? a.fill : "none");
    }
    return s.str();
}

ktb::ArgumentSpec to_spec(const ktc_arg& a) {
    ktb::ArgumentSpec s;
    s.role = a.role == KTC_ARG_INPUT ? ktb::ArgRole::input
             : a.role == KTC_ARG_OUTPUT ? ktb::ArgRole::output
                                        : ktb::ArgRole::scalar;
    s.type = a.type == KTC_I32 ? ktb::ElementType::i32 : ktb::ElementType::f32;
    s.length = a.length;
    s.value = a.value;
    s.fill = a.fill ? a.fill : "none";
    return s;
}

void set_msg(ktc_result* out, const std::string& m) {
    std::snprintf(out->message, sizeof(out->message), "%s", m.c_str());
}

void free_inputs(ktc_backend* be) {
    if (!be->in) return;
    const Driver& d = driver();
    if (!be->ctx->sticky) {
        d.cuCtxSetCurrent(be->ctx->cu);
        d.cuStreamSynchronize(be->ctx->stream);  // blocks go back to the cache idle
        const Inputs& I = *be->in;
        for (size_t a = 0; a < I.dev.size(); ++a)
            if (I.dev[a]) ctx_free(be->ctx, I.dev[a], a < I.bytes.size() ? I.bytes[a] : 0);
        for (size_t k = 0; k < I.out.size(); ++k)
            if (I.out[k]) ctx_free(be->ctx, I.out[k], I.out_count[k] * 4);
        for (size_t k = 0; k < I.ref.size(); ++k)
            if (I.ref[k]) ctx_free(be->ctx, I.ref[k], I.out_count[k] * 4);
    }
    be->in.reset();
}

#define CK(call, what)                                               \
    do {                                                             \
        CUresult rc_ = (call);                                       \
        if (rc_ != CUDA_SUCCESS) return fail_cu(be->ctx, rc_, what); \
    } while (0)

// Checks the documented case-study argument layout (the same layout the
// reference's synthetic backend requires, backend.hpp:416-473).
bool check_layout(const ktc_request* r, Family fam, std::string* why) {
    auto scalar = [&](int i) { return i < r->n_args && r->args[i].role == KTC_ARG_SCALAR; };
    auto f32buf = [&](int i, int role) {
        return i < r->n_args && r->args[i].role == role && r->args[i].type == KTC_F32;
    };
    if (fam == FAM_CONV) {
        if (r->n_args == 7 && scalar(0) && scalar(1) && scalar(2) && scalar(3) &&
            f32buf(4, KTC_ARG_INPUT) && f32buf(5, KTC_ARG_INPUT) && f32buf(6, KTC_ARG_OUTPUT))
            return true;
        *why = "expected scalars X, Y, FILTER, W then f32 image, filter and output buffers";
        return false;
    }
    if (r->n_args == 8 && scalar(0) && scalar(1) && scalar(2) && scalar(3) && scalar(4) &&
        f32buf(5, KTC_ARG_INPUT) && f32buf(6, KTC_ARG_INPUT) && f32buf(7, KTC_ARG_OUTPUT))
        return true;
    *why = "expected scalars M, N, K, ALPHA, BETA then f32 A, B and C buffers";
    return false;
}

// Host copies of materialized recipes, in pinned memory, shared by every
// backend of the process: a job's inputs are a pure function of their recipe
// (arguments.hpp:126-180), so a new job over the same problem only pays the
// H2D copy.  Bounded (LRU by insertion) to 4 GiB.  Pinned allocations die
// with the context that made them, so the cache holds its own retain on
// that device's primary context (a job that closes the last backend must
// not free them under the cache) and drops entries made before a
// primary-context reset (primary_ctx_epoch).
// Pinned blocks are pooled by exact size: dropping the recipe cache
// (ktc_drop_caches) forgets the contents, not the page-locked allocations,
// so a fresh job re-materializes into memory that is already pinned.
struct PinnedPool {
    std::mutex mu;
    struct Block {
        size_t bytes;
        void* host;
        unsigned epoch;
    };
    std::vector<Block> free;
    size_t free_bytes = 0;
    static constexpr size_t kCap = size_t(4) << 30;
    void* take(size_t bytes, unsigned epoch) {
        std::lock_guard<std::mutex> lk(mu);
        for (size_t i = 0; i < free.size(); ++i)
            if (free[i].bytes == bytes && free[i].epoch == epoch) {
                void* p = free[i].host;
                free_bytes -= bytes;
                free.erase(free.begin() + long(i));
                return p;
            }
        return nullptr;
    }
    void give(void* host, size_t bytes, unsigned epoch) {
        std::lock_guard<std::mutex> lk(mu);
        free.push_back({bytes, host, epoch});
        free_bytes += bytes;
        while (free_bytes > kCap && !free.empty()) {
            if (free.front().epoch == primary_ctx_epoch()) driver().cuMemFreeHost(free.front().host);
            free_bytes -= free.front().bytes;
            free.erase(free.begin());
        }
    }
};
PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool;  // leaked: outlives static destructors
    return *p;
}

struct PinnedInput {
    void* host = nullptr;
    size_t bytes = 0;
    unsigned epoch = 0;
    ~PinnedInput() {
        if (host && epoch == primary_ctx_epoch()) pinned_pool().give(host, bytes ? bytes : 4, epoch);
    }
};


struct RecipeCache {
    std::mutex mu;
    std::vector<std::pair<std::string, std::shared_ptr<PinnedInput>>> cache;
    std::set<int> retained;  // devices whose primary context the cache keeps alive
};
RecipeCache& recipe_cache() {
    static RecipeCache* rc = new RecipeCache;  // leaked: outlives static destructors
    return *rc;
}

std::shared_ptr<PinnedInput> pinned_recipe(const ktb::ArgumentSpec& a, CUdevice dev) {
    RecipeCache& rc = recipe_cache();
    std::mutex& mu = rc.mu;
    auto& cache = rc.cache;
    auto& retained = rc.retained;
    const std::string key = std::string(ktb::to_string(a.type)) + "|" + a.fill + "|" +
                            std::to_string(a.length);
    std::lock_guard<std::mutex> lk(mu);
    const unsigned epoch = primary_ctx_epoch();
    cache.erase(std::remove_if(cache.begin(), cache.end(),
                               [&](const auto& e) { return e.second->epoch != epoch; }),
                cache.end());
    for (auto& e : cache)
        if (e.first == key) return e.second;
    if (retained.insert(int(dev)).second) {
        CUcontext keep = nullptr;
        driver().cuDevicePrimaryCtxRetain(&keep, dev);  // released at process exit
    }
    auto p = std::make_shared<PinnedInput>();
    p->bytes = a.length * 4;
    p->epoch = epoch;
    p->host = pinned_pool().take(p->bytes ? p->bytes : 4, epoch);
    if (!p->host &&
        driver().cuMemHostAlloc(&p->host, p->bytes ? p->bytes : 4, CU_MEMHOSTALLOC_PORTABLE) !=
            CUDA_SUCCESS) {
        p->host = nullptr;
        throw ktb::Error("cuMemHostAlloc failed for a " + std::to_string(p->bytes) + "-byte input");
    }
    ktb::materialize_into(a, p->host);
    size_t total = p->bytes;
    for (auto& e : cache) total += e.second->bytes;
    while (!cache.empty() && total > (size_t(4) << 30)) {
        total -= cache.front().second->bytes;
        cache.erase(cache.begin());
    }
    cache.emplace_back(key, p);
    return p;
}

// Materializes, uploads and (for the built-in families) computes the device
// reference.  Throws nothing; returns a ktc.h code.
int build_inputs(ktc_backend* be, const ktc_request* r, Family fam) {
    const Driver& d = driver();
    ktc_ctx* ctx = be->ctx;
    auto in = std::make_unique<Inputs>();
    in->sig = signature(r);
    in->fam = fam;
    for (int i = 0; i < r->n_args; ++i) in->args.push_back(to_spec(r->args[i]));
    in->dev.assign(in->args.size(), 0);
    in->bytes.assign(in->args.size(), 0);
    // Ownership: register buffers in `in` as soon as they exist so the
    // error paths below release them via free_inputs.
    be->in = std::move(in);
    Inputs& I = *be->in;
    auto alloc = [&](size_t bytes, CUdeviceptr* p) { return ctx_alloc(ctx, bytes ? bytes : 4, p); };

    if (fam == FAM_CONV) {
        I.X = int(I.args[0].value);
        I.Y = int(I.args[1].value);
        I.F = int(I.args[2].value);
        I.W = float(I.args[3].value);
        if (I.X <= 0 || I.Y <= 0 || I.F < 1 || I.F % 2 == 0) {
            set_error("convolution scalars out of range");
            return KTC_ERR_INVALID;
        }
        const size_t px = size_t(I.X) + I.F - 1, py = size_t(I.Y) + I.F - 1;
        if (I.args[4].length != px * py || I.args[5].length != size_t(I.F) * I.F ||
            I.args[6].length != size_t(I.X) * I.Y) {
            set_error("convolution input sizes do not match the problem dimensions");
            return KTC_ERR_INVALID;
        }
        // HBM layout: padded image re-pitched to a 64-float (256 B) row pitch
        // with slack for the largest tile (512 x 512) and vector over-reads,
        // zero-filled; every tile load of every configuration stays in bounds
        // and every row start is 16-byte aligned for float4 / TMA.
        I.ipitch = int(round_up(round_up(size_t(I.X), 512) + I.F + 8, 64));
        I.rows = int(round_up(size_t(I.Y), 512) + I.F + 32);
        const auto tm = Clock::now();
        std::shared_ptr<PinnedInput> img = pinned_recipe(I.args[4], ctx->dev);
        trace_phase("inputs: image recipe (pinned)", tm);
        I.taps.resize(size_t(I.F) * I.F);
        ktb::materialize_into(I.args[5], I.taps.data());
        I.bytes[4] = size_t(I.ipitch) * I.rows * 4;
        CK(alloc(I.bytes[4], &I.dev[4]), "cuMemAlloc(image)");
        CK(d.cuMemsetD32Async(I.dev[4], 0, I.bytes[4] / 4, ctx->stream), "cuMemset(image)");
        CK(d.cuStreamSynchronize(ctx->stream), "cuStreamSynchronize");
        int st = ktc_upload_pitched(ctx, I.dev[4], size_t(I.ipitch) * 4, img->host, px * 4, px * 4,
                                    py);
        if (st) return st;
        trace_phase("inputs: + H2D image", tm);
        I.bytes[5] = I.taps.size() * 4;
        CK(alloc(I.bytes[5], &I.dev[5]), "cuMemAlloc(taps)");
        CK(d.cuMemcpyHtoD(I.dev[5], I.taps.data(), I.bytes[5]), "cuMemcpyHtoD(taps)");
        I.out_arg = {6};
    } else if (fam == FAM_GEMM || fam == FAM_GEMM_TF32) {
        I.M = int(I.args[0].value);
        I.N = int(I.args[1].value);
        I.K = int(I.args[2].value);
        I.alpha = float(I.args[3].value);
        I.beta = float(I.args[4].value);
        if (I.M <= 0 || I.N <= 0 || I.K <= 0) {
            set_error("matrix dimensions must be positive");
            return KTC_ERR_INVALID;
        }
        if (I.args[5].length != size_t(I.K) * I.M || I.args[6].length != size_t(I.K) * I.N ||
            I.args[7].length != size_t(I.M) * I.N) {
            set_error("matrix sizes do not match the problem dimensions");
            return KTC_ERR_INVALID;
        }
        for (int a = 5; a <= 7; ++a) {  // A, B, C (C pristine: kernels write a separate output)
            std::shared_ptr<PinnedInput> h = pinned_recipe(I.args[a], ctx->dev);
            I.bytes[a] = h->bytes;
            CK(alloc(I.bytes[a], &I.dev[a]), "cuMemAlloc(matrix)");
            CK(d.cuMemcpyHtoD(I.dev[a], h->host, I.bytes[a]), "cuMemcpyHtoD(matrix)");
        }
        I.out_arg = {7};
    } else {
        for (size_t a = 0; a < I.args.size(); ++a) {
            if (I.args[a].role == ktb::ArgRole::scalar) continue;
            I.bytes[a] = I.args[a].length * 4;
            CK(alloc(I.bytes[a], &I.dev[a]), "cuMemAlloc(argument)");
            if (I.args[a].role == ktb::ArgRole::output) I.out_arg.push_back(int(a));
        }
    }
    for (int a : I.out_arg) {
        CUdeviceptr p = 0, q = 0;
        CK(alloc(I.args[a].length * 4, &p), "cuMemAlloc(output)");
        I.out.push_back(p);
        I.ref.push_back(q);
        I.out_count.push_back(I.args[a].length);
        I.out_type.push_back(I.args[a].type == ktb::ElementType::i32 ? KTC_I32 : KTC_F32);
    }
    I.ref_digest.assign(I.out.size(), "");

    // Device reference of the built-in families (bit-identical to the oracle).
    if (fam == FAM_CONV) {
        CK(alloc(I.out_count[0] * 4, &I.ref[0]), "cuMemAlloc(reference)");
        int X = I.X, Y = I.Y, F = I.F, ip = I.ipitch;
        float W = I.W;
        CUdeviceptr img = I.dev[4], taps = I.dev[5], out = I.ref[0];
        void* p[] = {&X, &Y, &F, &W, &img, &ip, &taps, &out};
        CK(launch(ctx, ctx->fn_conv_ref, unsigned((X + 31) / 32), unsigned((Y + 7) / 8), 1, 32, 8, 1,
                  0, p),
           "conv reference launch");
        CK(d.cuStreamSynchronize(ctx->stream), "conv reference");
        I.has_reference = true;
    } else if (fam == FAM_GEMM || fam == FAM_GEMM_TF32) {
        CK(alloc(I.out_count[0] * 4, &I.ref[0]), "cuMemAlloc(reference)");
        int M = I.M, N = I.N, K = I.K;
        float al = I.alpha, bt = I.beta;
        CUdeviceptr A = I.dev[5], B = I.dev[6], C = I.dev[7], out = I.ref[0];
        void* p[] = {&M, &N, &K, &al, &bt, &A, &B, &C, &out};
        CK(launch(ctx, ctx->fn_gemm_ref, unsigned((N + 31) / 32), unsigned((M + 31) / 32), 1, 32, 8,
                  1, 0, p),
           "gemm reference launch");
        CK(d.cuStreamSynchronize(ctx->stream), "gemm reference");
        I.has_reference = true;
    }
    return KTC_OK;
}

int upload_reference(ktc_backend* be, int n_buffers, const void* const* buffers,
                     const size_t* lengths, const int* types) {
    Inputs& I = *be->in;
    if (n_buffers != int(I.out.size())) {
        set_error("reference has " + std::to_string(n_buffers) + " buffers, kernel has " +
                  std::to_string(I.out.size()) + " outputs");
        return KTC_ERR_INVALID;
    }
    const Driver& d = driver();
    for (int k = 0; k < n_buffers; ++k) {
        if (lengths[k] != I.out_count[k] || types[k] != I.out_type[k]) {
            set_error("reference buffer " + std::to_string(k) + " differs in length or type");
            return KTC_ERR_INVALID;
        }
        if (!I.ref[k]) {
            CUresult rc = ctx_alloc(be->ctx, lengths[k] * 4, &I.ref[k]);
            if (rc != CUDA_SUCCESS) return fail_cu(be->ctx, rc, "cuMemAlloc(reference)");
        }
        CUresult rc = d.cuMemcpyHtoD(I.ref[k], buffers[k], lengths[k] * 4);
        if (rc != CUDA_SUCCESS) return fail_cu(be->ctx, rc, "cuMemcpyHtoD(reference)");
        I.ref_digest[k].clear();
    }
    I.has_reference = true;
    return KTC_OK;
}

int ensure_inputs(ktc_backend* be, const ktc_request* r, Family fam) {
    if (be->ctx->sticky) {
        free_inputs(be);
        be->modules.clear();  // died with the context
        be->tail_ws = be->tail_cnt = 0;
        be->tail_ws_bytes = be->tail_cnt_bytes = 0;
        int st = ktc_reset(be->ctx);
        if (st) return st;
    }
    std::string sig = signature(r);
    if (be->in && be->in->sig == sig) return KTC_OK;
    free_inputs(be);
    int st;
    const auto t0 = std::chrono::steady_clock::now();
    try {
        st = build_inputs(be, r, fam);
        trace_phase("build inputs (+reference)", t0);
    } catch (const std::exception& e) {
        set_error(e.what());
        st = KTC_ERR_INVALID;
    }
    if (st) {
        free_inputs(be);  // never leave a half-built argument list cached
        return st;
    }
    if (be->bound.sig == sig) {  // re-bind the host reference after a rebuild
        std::vector<const void*> ptrs;
        for (const auto& b : be->bound.bytes) ptrs.push_back(b.data());
        return upload_reference(be, int(ptrs.size()), ptrs.data(), be->bound.lengths.data(),
                                be->bound.types.data());
    }
    return KTC_OK;
}

// Upload per-evaluation initial contents of custom-kernel buffers (inputs
// and outputs follow their fill recipes, exactly as the reference's
// external runner would receive them).
int refresh_custom_buffers(ktc_backend* be) {
    Inputs& I = *be->in;
    for (size_t a = 0; a < I.args.size(); ++a) {
        if (I.args[a].role == ktb::ArgRole::scalar) continue;
        std::vector<char> h(I.bytes[a]);
        ktb::materialize_into(I.args[a], h.data());
        CK(driver().cuMemcpyHtoD(I.dev[a], h.data(), h.size()), "cuMemcpyHtoD(argument)");
    }
    return KTC_OK;
}

// Problem dimensions straight from the request's scalar arguments (the
// documented layouts of check_layout): plans need nothing else, so compiles
// can be queued before the argument list is materialized and uploaded.
struct Dims {
    int X = 0, Y = 0, F = 0;  // conv
    int M = 0, N = 0, K = 0;  // gemm
};

Dims dims_of(const ktc_request* r, Family fam) {
    Dims d;
    auto iv = [&](int i) { return i < r->n_args ? int(r->args[i].value) : 0; };
    if (fam == FAM_CONV) {
        d.X = iv(0), d.Y = iv(1), d.F = iv(2);
    } else if (fam == FAM_GEMM || fam == FAM_GEMM_TF32) {
        d.M = iv(0), d.N = iv(1), d.K = iv(2);
    }
    return d;
}

bool dims_valid(const Dims& d, Family fam) {
    if (fam == FAM_CONV) return d.X > 0 && d.Y > 0 && d.F >= 1 && d.F % 2 == 1;
    if (fam == FAM_GEMM || fam == FAM_GEMM_TF32) return d.M > 0 && d.N > 0 && d.K > 0;
    return true;
}

// ---------------------------------------------------------------------------
// Plans: configuration -> NVRTC source/defines + launch geometry.
// Returns false with a message for configurations this device cannot run
// (reported as runtime_error, like a launch failure).
// ---------------------------------------------------------------------------

// Row-paired FFMA2 in the unrolled conv (conv.cu CF2); KTC_CONV_F2 overrides.
int conv_f2_policy() {
    static const int v = [] {
        const char* e = std::getenv("KTC_CONV_F2");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// Diagnostic CTA timeline of the conv family (ptxgen_conv TRACE): when
// KTC_CONV_TRACE names a directory, each evaluation's last timed launch
// leaves per-CTA {start ns, end ns, smid, 0} in <dir>/conv_trace_<n>.bin
// (header: grid x, grid y as u32).  Never set in tuning runs.
const char* conv_trace_dir() {
    static const char* v = std::getenv("KTC_CONV_TRACE");
    return v && *v ? v : nullptr;
}

// Conv register budget (ptxgen_conv MINCTA -> .minnctapersm): 0 = ptxas's
// own choice, 1 = the shared-memory-limited CTA count, n > 1 = n CTAs per
// SM.  KTC_CONV_MINCTA overrides.
int conv_mincta_policy() {
    static const int v = [] {
        const char* e = std::getenv("KTC_CONV_MINCTA");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// Single-box TMA halo of exactly TY + 2H rows (else rounded up to 8 rows).
bool conv_bh_exact() {
    static const bool v = [] {
        const char* e = std::getenv("KTC_CONV_BH_EXACT");
        return e ? std::atoi(e) != 0 : false;
    }();
    return v;
}

bool plan_conv(ktc_backend* be, const ktc_request* r, Plan* p, std::string* why) {
    const Dims I = dims_of(r, FAM_CONV);
    ParamView pv{r};
    long long XWG, YWG, XWPT, YWPT, LOCAL, VW, PAD, UNR;
    if (!pv.get("XWG", &XWG) || !pv.get("YWG", &YWG) || !pv.get("XWPT", &XWPT) ||
        !pv.get("YWPT", &YWPT) || !pv.get("LOCAL", &LOCAL) || !pv.get("VW", &VW) ||
        !pv.get("PAD", &PAD) || !pv.get("UNR", &UNR)) {
        *why = "the conv family needs XWG, YWG, XWPT, YWPT, LOCAL, VW, PAD, UNR";
        return false;
    }
    auto pow2 = [](long long v) { return v > 0 && (v & (v - 1)) == 0; };
    if (!pow2(XWG) || !pow2(YWG) || !pow2(XWPT) || !pow2(YWPT) || !(VW == 1 || VW == 2 || VW == 4 || VW == 8) ||
        XWPT % VW != 0 || LOCAL < 0 || LOCAL > 2 || XWG * XWPT < 8 || XWG * XWPT > 512 ||
        YWG * YWPT > 512) {
        *why = "conv configuration outside the family's parameter domain";
        return false;
    }
    const long long H = (I.F - 1) / 2, TX = XWG * XWPT, TY = YWG * YWPT;
    p->ksrc = &conv_source();
    p->problem = {define("FS", I.F)};
    auto& o = p->config;
    o = {define("XWG", XWG), define("YWG", YWG), define("XWPT", XWPT),
         define("YWPT", YWPT), define("LOCAL", LOCAL), define("VW", VW),
         define("PAD", LOCAL >= 1 ? PAD : 0), define("UNR", UNR ? 1 : 0),
         define("GUARD", (I.X % TX != 0 || I.Y % TY != 0) ? 1 : 0),
         define("OUT_VEC", I.X % VW == 0 ? 1 : 0), define("CF2", conv_f2_policy())};
    size_t smem_floats = 0;
    if (LOCAL == 1) {
        const long long SP = TX + 2 * H + PAD;
        o.push_back(define("SP", SP));
        smem_floats = size_t(SP * (TY + 2 * H) + 8);
    } else if (LOCAL == 2) {
        const long long PWO = std::min<long long>(TX, 128);
        const long long BW = (PWO + 2 * H + 3) / 4 * 4 + 4 * PAD;
        const long long TR = TY + 2 * H;
        const long long NB = (TR + 255) / 256;
        const long long NP = TX / PWO;
        // Boxes after the first start 128-B aligned (BH a multiple of 8);
        // a single box may be exactly the halo height (conv_bh_exact()).
        const long long BH = (NB == 1 && NP == 1 && conv_bh_exact()) ? TR
                                                                     : ((TR + NB - 1) / NB + 7) / 8 * 8;
        const long long PF = BW * NB * BH;
        o.insert(o.end(), {define("PWO", PWO), define("BW", BW), define("BH", BH),
                           define("NB", NB), define("NP", NP), define("PF", PF)});
        smem_floats = size_t(NP * PF + 4);
        p->tma_mode = 1;
        p->box[0] = unsigned(BW);
        p->box[1] = unsigned(BH);
    }
    p->smem = unsigned(smem_floats * 4);
    // Register budget: ask ptxas for as many co-resident CTAs as shared
    // memory and the thread limit allow (conv_mincta_policy()).
    if (const int pol = conv_mincta_policy()) {
        const long long per_sm = be->ctx->limits.smem_per_sm ? be->ctx->limits.smem_per_sm : 233472;
        long long n = pol > 1 ? pol
                              : std::min<long long>({32, 2048 / (XWG * YWG),
                                                     per_sm / ((long long)p->smem + 1024)});
        if (n > 1) o.push_back(define("MINCTA", n));
    }
    if (conv_trace_dir()) o.push_back(define("TRACE", 1));
    p->compile_cost = unrolled_cost(double(XWPT * YWPT) * (UNR ? double(I.F) * I.F : 4.0));
    if (p->smem > be->ctx->limits.smem_per_block_optin) {
        *why = "needs " + std::to_string(p->smem) + " bytes of shared memory; the device allows " +
               std::to_string(be->ctx->limits.smem_per_block_optin);
        return false;
    }
    if (r->ndim != 2 || r->local[0] != size_t(XWG) || r->local[1] != size_t(YWG)) {
        *why = "request local size does not match (XWG, YWG)";
        return false;
    }
    for (int k = 0; k < 2; ++k) {
        p->block[k] = unsigned(r->local[k]);
        p->grid[k] = unsigned((r->global[k] + r->local[k] - 1) / r->local[k]);
    }
    // The grid must cover the image (global = (X/XWPT, Y/YWPT) per the
    // reference's modifiers, landscapes.hpp:87-92).
    if ((long long)p->grid[0] * TX < I.X || (long long)p->grid[1] * TY < I.Y) {
        *why = "request global size does not cover the image";
        return false;
    }
    return true;
}

// Upper bound on the double-buffered GEMM tile footprint (bytes).  112 KiB
// keeps two CTAs per SM; KTC_GEMM_DBUF_MAX overrides it (0 disables) for
// A/B experiments.
size_t gemm_dbuf_max_bytes() {
    static const size_t v = [] {
        const char* e = std::getenv("KTC_GEMM_DBUF_MAX");
        return e ? size_t(std::strtoull(e, nullptr, 10)) : size_t(112 * 1024);
    }();
    return v;
}

// Register-budget policy handed to the kernel (gemm.cu OCC): 1 = estimate
// the live registers and ask ptxas for the matching CTAs per SM; 0 = leave
// ptxas the full 255-register budget.  KTC_GEMM_OCC overrides.
int gemm_occ_policy() {
    static const int v = [] {
        const char* e = std::getenv("KTC_GEMM_OCC");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// Split-K tail wave for the PTX-generated SGEMM (TAILK); KTC_GEMM_TAIL=0
// disables it.  The NVRTC build (gemm.cu) has no tail split.
int gemm_tail_policy() {
    static const int v = [] {
        const char* e = std::getenv("KTC_GEMM_TAIL");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// Stream-K for unevenly distributed SGEMM tiles (ptxgen_gemm SK);
// KTC_GEMM_SK=0 disables it.
int gemm_sk_policy() {
    static const int v = [] {
        const char* e = std::getenv("KTC_GEMM_SK");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// Packed FFMA2 outer products (gemm.cu F2); KTC_GEMM_F2 overrides.
int gemm_f2_policy() {
    static const int v = [] {
        const char* e = std::getenv("KTC_GEMM_F2");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

bool plan_gemm(ktc_backend* be, const ktc_request* r, Plan* p, std::string* why) {
    const Dims I = dims_of(r, FAM_GEMM);
    ParamView pv{r};
    static const char* names[] = {"MWG", "NWG",  "KWG",  "MDIMC", "NDIMC", "SA",  "SB",
                                  "MDIMA", "NDIMB", "STRM", "STRN", "VWM",  "VWN", "KWI"};
    long long v[14];
    for (int i = 0; i < 14; ++i)
        if (!pv.get(names[i], &v[i])) {
            *why = std::string("the gemm family needs parameter ") + names[i];
            return false;
        }
    const long long MWG = v[0], NWG = v[1], KWG = v[2], MDIMC = v[3], NDIMC = v[4], SA = v[5],
                    SB = v[6], KWI = v[13], VWM = v[11], VWN = v[12];
    long long MDIMA = v[7], NDIMB = v[8];
    auto pow2 = [](long long x) { return x > 0 && (x & (x - 1)) == 0; };
    for (int i = 0; i < 14; ++i)
        if (i != 5 && i != 6 && i != 9 && i != 10 && !pow2(v[i])) {
            *why = "gemm configuration outside the family's parameter domain";
            return false;
        }
    if (MWG % MDIMC || NWG % NDIMC || (MWG / MDIMC) % VWM || (NWG / NDIMC) % VWN || KWG % KWI ||
        VWM > 8 || VWN > 8 || (MDIMC * NDIMC) % MDIMA || (MDIMC * NDIMC) % NDIMB ||
        KWG % ((MDIMC * NDIMC) / MDIMA) || KWG % ((MDIMC * NDIMC) / NDIMB)) {
        *why = "gemm configuration violates the family's divisibility rules";
        return false;
    }
    if (I.M % MWG || I.N % NWG || I.K % KWG) {
        *why = "problem size (" + std::to_string(I.M) + "x" + std::to_string(I.N) + "x" +
               std::to_string(I.K) + ") is not a multiple of the (MWG, NWG, KWG) tile";
        return false;
    }
    // Code identity: MDIMA / NDIMB only shape the shared-memory copies, so
    // with SA = 0 / SB = 0 they are normalised away and those rows share one
    // cubin (they are still timed as separate rows).
    if (!SA) MDIMA = 8;
    if (!SB) NDIMB = 8;
    p->ksrc = &gemm_source();
    p->config = {define("MWG", MWG),     define("NWG", NWG),     define("KWG", KWG),
               define("MDIMC", MDIMC), define("NDIMC", NDIMC), define("SA", SA ? 1 : 0),
               define("SB", SB ? 1 : 0), define("MDIMA", MDIMA), define("NDIMB", NDIMB),
               define("STRM", v[9] ? 1 : 0), define("STRN", v[10] ? 1 : 0), define("VWM", VWM),
               define("VWN", VWN), define("KWI", KWI)};
    // Double-buffered cp.async tiles when two copies of the staged tiles
    // stay within gemm_dbuf_max_bytes() (so a second CTA still fits per SM);
    // otherwise the single-buffer, register-staged copy.
    const unsigned tile_bytes = unsigned((SA * KWG * MWG + SB * KWG * NWG) * 4);
    const bool dbuf = (SA || SB) && 2 * size_t(tile_bytes) <= gemm_dbuf_max_bytes() &&
                      2 * size_t(tile_bytes) <= be->ctx->limits.smem_per_block_optin;
    p->config.push_back(define("DBUF", dbuf ? 1 : 0));
    p->config.push_back(define("OCC", gemm_occ_policy()));
    p->config.push_back(define("F2", gemm_f2_policy()));
    p->smem = dbuf ? 2 * tile_bytes : tile_bytes;
    // Compiled in only where the launch policy can split: K >= 8192 (every
    // split keeps K/s >= 4096) and at most 16 tiles per SM -- or when a
    // split count is forced (KTC_GEMM_SPLIT, tests and probes).
    const long long tiles = (I.M / MWG) * (I.N / NWG);
    // Stream-K (SK) where whole tiles leave the GPU under-filled: fewer than
    // two tiles per SM on average and K >= 2048 (tools/sk_probe.py: 8192 x
    // 256 x 8192 with 128x128 tiles 48.5 -> 57.1 TFLOP/s, 2048^3 128x128
    // 51.6 -> 54.0; with 3.5 tiles per SM, or K = 1024, dealing K-ranges
    // measured slower).  The launch keeps whole tiles when a CTA's share of
    // K would be under 1024.
    const double per_sm = double(tiles) / double(std::max(be->ctx->limits.sm_count, 1));
    const bool sk = gemm_sk_policy() && gemm_source().ptx_generator && !std::getenv("KTC_GEMM_SPLIT") &&
                    I.K >= 2048 && per_sm < 2.0;
    if (sk) {
        p->config.push_back(define("SK", 1));
        p->sk = true;
    } else if (gemm_tail_policy() && gemm_source().ptx_generator &&
               (I.K >= 8192 || std::getenv("KTC_GEMM_SPLIT")) &&
               tiles <= 16LL * be->ctx->limits.sm_count) {
        p->config.push_back(define("TAILK", 1));
        p->tailk = true;
    }
    if (p->sk || p->tailk) {
        p->smem += 16;  // the arrival flag after the staged tiles
        p->tiles_x = unsigned(I.M / MWG);
        p->tiles_y = unsigned(I.N / NWG);
        p->ktiles = unsigned(I.K / KWG);
        p->ktile_k = unsigned(KWG);
        p->tile_floats = unsigned(MWG * NWG);
    }
    p->compile_cost = unrolled_cost(double((MWG / MDIMC) * (NWG / NDIMC) * KWI) + 64.0);
    if (p->smem > be->ctx->limits.smem_per_block_optin) {
        *why = "needs " + std::to_string(p->smem) + " bytes of shared memory";
        return false;
    }
    if (r->ndim != 2 || r->local[0] != size_t(MDIMC) || r->local[1] != size_t(NDIMC)) {
        *why = "request local size does not match (MDIMC, NDIMC)";
        return false;
    }
    p->block[0] = unsigned(MDIMC);
    p->block[1] = unsigned(NDIMC);
    p->grid[0] = unsigned(I.M / MWG);
    p->grid[1] = unsigned(I.N / NWG);
    // global = (M*MDIMC/MWG, N*NDIMC/NWG) (landscapes.hpp:260-267)
    if (r->global[0] != size_t(p->grid[0]) * MDIMC || r->global[1] != size_t(p->grid[1]) * NDIMC) {
        *why = "request global size does not match the (MWG, NWG) tiling";
        return false;
    }
    return true;
}


bool plan_custom(ktc_backend* be, const ktc_request* r, Plan* p, std::string* why) {
    const std::string path = r->source_ref ? r->source_ref : "";
    const std::string entry = r->kernel_name ? r->kernel_name : "";
    auto it = be->custom_sources.find(path + "|" + entry);
    if (it == be->custom_sources.end()) {
        std::ifstream f(path, std::ios::binary);
        if (!f) {
            *why = "cannot read kernel source \"" + path + "\"";
            return false;
        }
        std::ostringstream s;
        s << f.rdbuf();
        KernelSource ks = split_source(path, s.str(), entry);
        ks.prelude.clear();
        ks.body = s.str();
        ks.batchable = false;
        ks.fixed_entry = entry;
        it = be->custom_sources.emplace(path + "|" + entry, ks).first;
    }
    p->ksrc = &it->second;
    for (int i = 0; i < r->n_params; ++i)
        p->config.push_back(define(r->param_names[i], r->param_values[i]));
    if (r->ndim < 1 || r->ndim > 3) {
        *why = "thread sizes must have 1 to 3 dimensions";
        return false;
    }
    for (int k = 0; k < r->ndim; ++k) {
        if (r->local[k] == 0) {
            *why = "zero local size";
            return false;
        }
        p->block[k] = unsigned(r->local[k]);
        p->grid[k] = unsigned((r->global[k] + r->local[k] - 1) / r->local[k]);
    }
    return true;
}



// TF32 stream-K (gemm_tf32.cu SK); KTC_TF32_SK=0 disables it.
int tf32_sk_policy() {
    static const int v = [] {
        const char* e = std::getenv("KTC_TF32_SK");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// TF32 tcgen05 variant (kernels/gemm_tf32.cu): one 128-thread CTA per
// 128 x BN tile, TMA tensor maps for A (M-major) and B (N-major), SWIZZLE_128B.
bool plan_gemm_tf32(ktc_backend* be, const ktc_request* r, Plan* p, std::string* why) {
    const Dims I = dims_of(r, FAM_GEMM_TF32);
    ParamView pv{r};
    long long BN, BK, STAGES, CG = 1;
    if (!pv.get("BN", &BN) || !pv.get("BK", &BK) || !pv.get("STAGES", &STAGES)) {
        *why = "the gemm_tf32 family needs BN, BK, STAGES";
        return false;
    }
    pv.get("CG", &CG);  // optional: 1 (one CTA per tile) unless given
    if (!(BN == 64 || BN == 128 || BN == 256) || !(BK == 32 || BK == 64) || STAGES < 2 ||
        STAGES > 8 || !(CG == 1 || CG == 2)) {
        *why = "gemm_tf32 configuration outside the family's parameter domain";
        return false;
    }
    if (I.M % (128 * CG) || I.N % BN || I.K % BK) {
        *why = "problem size (" + std::to_string(I.M) + "x" + std::to_string(I.N) + "x" +
               std::to_string(I.K) + ") is not a multiple of the (" + std::to_string(128 * CG) +
               ", BN, BK) tile";
        return false;
    }
    p->ksrc = &tf32_source();
    // Stream-K (SK host switch) for long-K problems whose (pair-)tiles fill
    // less than one wave of one CTA per SM: the tiles x K-blocks units are
    // dealt to the resident clusters (1024 x 1024 x 8192: 86 -> 63 us with
    // 256 x 256 pair tiles).  With K = 2048 the partial-tile reductions cost
    // more than the idle SMs (2048^3: 32.7 -> 50 us), so it stays off there.
    const long long tiles = (I.M / (128 * CG)) * (I.N / BN);
    const bool sk = tf32_sk_policy() && (I.K >= 4096 || tf32_sk_policy() == 2) && I.K / BK >= 8 &&
                    tiles * CG < (long long)be->ctx->limits.sm_count;
    p->config = {define("BN", BN), define("BK", BK), define("STAGES", STAGES), define("CG", CG),
                 define("SK", sk ? 1 : 0)};
    if (sk && std::getenv("KTC_TF32_SK_TRACE")) p->config.push_back(define("SKTRACE", 1));
    p->smem = unsigned(STAGES * 4 * BK * (128 + BN / CG) + 2048);
    if (p->smem > be->ctx->limits.smem_per_block_optin) {
        *why = "needs " + std::to_string(p->smem) + " bytes of shared memory";
        return false;
    }
    p->block[0] = sk ? 192 : 128;
    p->grid[0] = unsigned(I.M / 128);
    p->grid[1] = unsigned(I.N / BN);
    if (sk) {
        p->sk = true;
        p->tiles_x = unsigned(I.M / (128 * CG));  // tile rows (pairs for CG = 2)
        p->tiles_y = unsigned(I.N / BN);
        p->ktiles = unsigned(I.K / BK);
        p->ktile_k = unsigned(BK);
        p->tile_floats = unsigned(128 * BN);
        p->cg = unsigned(CG);
    }
    p->tma_mode = 2;
    p->box[0] = 32;
    p->box[1] = unsigned(BK);
    return true;
}

int evaluate(ktc_backend* be, const ktc_request* r, ktc_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->status = KTC_STATUS_RUNTIME_ERROR;
    out->verification = KTC_VERIFY_SKIPPED;
    const Driver& d = driver();
    ktc_ctx* ctx = be->ctx;
    const Family fam = family_of(r->kernel_name);
    std::string why;
    if (fam != FAM_CUSTOM && !check_layout(r, fam, &why)) {
        set_msg(out, "runtime_error: " + why);
        return KTC_OK;
    }
    int st = make_current(ctx);
    if (st) return st;
    st = ensure_inputs(be, r, fam);
    if (st) return st;
    Inputs& I = *be->in;

    Plan plan;
    bool ok = fam == FAM_CONV   ? plan_conv(be, r, &plan, &why)
              : fam == FAM_GEMM ? plan_gemm(be, r, &plan, &why)
              : fam == FAM_GEMM_TF32 ? plan_gemm_tf32(be, r, &plan, &why)
                                     : plan_custom(be, r, &plan, &why);
    if (!ok) {
        set_msg(out, why);
        return KTC_OK;
    }

    // 1. cubin
    auto t0 = Clock::now();
    bool hit = false;
    KernelPtr kern =
        CompileService::instance().get(*plan.ksrc, plan.problem, plan.config, &hit, plan.compile_cost);
    out->compile_ms = hit ? 0.0 : ms_since(t0);
    out->compile_cache_hit = hit ? 1 : 0;
    if (!kern->ok()) {
        out->status = KTC_STATUS_COMPILE_ERROR;
        set_msg(out, "NVRTC: " + kern->log.substr(0, 480));
        return KTC_OK;
    }

    // 2. module (cached per cubin: a compile batch serves several configs)
    t0 = Clock::now();
    ModuleEntry* me = nullptr;
    for (size_t i = 0; i < be->modules.size(); ++i)
        if (be->modules[i].cubin.get() == kern->cubin.get()) {
            std::rotate(be->modules.begin() + long(i), be->modules.begin() + long(i) + 1,
                        be->modules.end());
            me = &be->modules.back();
            break;
        }
    if (!me) {
        if (be->modules.size() >= 24) {
            driver().cuModuleUnload(be->modules.front().mod);
            be->modules.erase(be->modules.begin());
        }
        ModuleEntry e;
        e.cubin = kern->cubin;
        CUresult rc = driver().cuModuleLoadData(&e.mod, kern->cubin->image.data());
        if (rc != CUDA_SUCCESS) {
            st = fail_cu(ctx, rc, "cuModuleLoadData");
            set_msg(out, last_error());
            return ctx->sticky ? st : KTC_OK;
        }
        be->modules.push_back(e);
        me = &be->modules.back();
    }
    ktc_fn fn_storage;
    fn_storage.ctx = ctx;
    fn_storage.mod = me->mod;
    {
        CUresult rc = driver().cuModuleGetFunction(&fn_storage.fn, me->mod, kern->entry.c_str());
        if (rc != CUDA_SUCCESS) {
            st = fail_cu(ctx, rc, "cuModuleGetFunction");
            set_msg(out, last_error());
            return ctx->sticky ? st : KTC_OK;
        }
    }
    ktc_fn* fn = &fn_storage;

    alignas(64) CUtensorMap tmap, tmap2, tmap3;
    std::memset(&tmap, 0, sizeof(tmap));
    std::memset(&tmap2, 0, sizeof(tmap2));
    std::vector<void*> params;
    // Scalar storage must outlive the launches.
    int iX = 0, iY = 0, iP = 0, iM = 0, iN = 0, iK = 0;
    float fW = 0, fA = 0, fB = 0;
    CUdeviceptr pImg = 0, pOut = 0, pA = 0, pB = 0, pC = 0;
    CUdeviceptr tk_ws = 0, tk_cnt = 0, trace_buf = 0;
    size_t sk_trace_off = 0;
    unsigned sk_trace_ctas = 0;
    unsigned tk_full = 0, tk_splits = 1, tk_gx = 1, tk_kt = 1;
    std::vector<long long> scal_i;  // custom scalars
    std::vector<float> scal_f;
    std::vector<CUdeviceptr> ptrs;
    if (fam == FAM_CONV) {
        if (me->taps_sig != I.sig) {
            if (ktc_set_symbol(fn, "c_taps", I.taps.data(), I.taps.size() * 4) != KTC_OK) {
                set_msg(out, last_error());
                return ctx->sticky ? KTC_ERR_LAUNCH : KTC_OK;
            }
            // Row-paired taps (conv.cu c_tpair), when the module kept the symbol.
            CUdeviceptr tp = 0;
            size_t tp_size = 0;
            if (d.cuModuleGetGlobal(&tp, &tp_size, fn->mod, "c_tpair") == CUDA_SUCCESS) {
                std::vector<float> pairs(size_t(2) * I.F * I.F, 0.0f);
                for (int jj = 1; jj < I.F; ++jj)
                    for (int i = 0; i < I.F; ++i) {
                        pairs[2 * size_t(jj * I.F + i)] = I.taps[size_t(jj * I.F + i)];
                        pairs[2 * size_t(jj * I.F + i) + 1] = I.taps[size_t((jj - 1) * I.F + i)];
                    }
                if (tp_size < pairs.size() * 4 ||
                    d.cuMemcpyHtoD(tp, pairs.data(), pairs.size() * 4) != CUDA_SUCCESS) {
                    set_msg(out, "cannot set c_tpair");
                    return ctx->sticky ? KTC_ERR_LAUNCH : KTC_OK;
                }
            }
            me->taps_sig = I.sig;
        }
        if (plan.tma_mode == 1) {
            cuuint64_t dims[2] = {cuuint64_t(I.ipitch), cuuint64_t(I.rows)};
            cuuint64_t strides[1] = {cuuint64_t(I.ipitch) * 4};
            cuuint32_t box[2] = {plan.box[0], plan.box[1]};
            cuuint32_t estr[2] = {1, 1};
            CUresult rc = d.cuTensorMapEncodeTiled(
                &tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, reinterpret_cast<void*>(I.dev[4]), dims,
                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (rc != CUDA_SUCCESS) {
                set_msg(out, cu_error_text(rc, "cuTensorMapEncodeTiled"));
                return KTC_OK;
            }
        }
        iX = I.X;
        iY = I.Y;
        fW = I.W;
        pImg = I.dev[4];
        iP = I.ipitch;
        pOut = I.out[0];
        params = {&iX, &iY, &fW, &pImg, &iP, &pOut, &tmap};
        if (conv_trace_dir()) {
            const size_t tb = size_t(plan.grid[0]) * plan.grid[1] * 32;
            if (d.cuMemAlloc(&trace_buf, tb) != CUDA_SUCCESS) {
                set_msg(out, "cannot allocate the conv trace buffer");
                return KTC_OK;
            }
            params.push_back(&trace_buf);
        }
    } else if (fam == FAM_GEMM || fam == FAM_GEMM_TF32) {
        if (plan.tma_mode == 2) {
            auto encode = [&](CUtensorMap* m, CUdeviceptr base, int inner, int outer) {
                cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
                cuuint64_t strides[1] = {cuuint64_t(inner) * 4};
                cuuint32_t box[2] = {plan.box[0], plan.box[1]};
                cuuint32_t estr[2] = {1, 1};
                return d.cuTensorMapEncodeTiled(
                    m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, reinterpret_cast<void*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    // MN-major TF32 operands need UMMA's SW128_32B layout:
                    // 128-byte rows, 32-byte swizzle atoms (4-row groups).
                    CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            };
            CUresult rc = encode(&tmap, I.dev[5], I.M, I.K);
            if (rc == CUDA_SUCCESS) rc = encode(&tmap2, I.dev[6], I.N, I.K);
            if (rc == CUDA_SUCCESS) {
                // output C (M x N, N contiguous) for the TMA-store epilogue:
                // 32-column x 128-row boxes, 128-byte swizzle
                cuuint64_t dims[2] = {cuuint64_t(I.N), cuuint64_t(I.M)};
                cuuint64_t strides[1] = {cuuint64_t(I.N) * 4};
                cuuint32_t box[2] = {32, 128};
                cuuint32_t estr[2] = {1, 1};
                rc = d.cuTensorMapEncodeTiled(&tmap3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                              reinterpret_cast<void*>(I.out[0]), dims, strides, box,
                                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_128B,
                                              CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
            if (rc != CUDA_SUCCESS) {
                set_msg(out, cu_error_text(rc, "cuTensorMapEncodeTiled"));
                return KTC_OK;
            }
        }
        iM = I.M;
        iN = I.N;
        iK = I.K;
        fA = I.alpha;
        fB = I.beta;
        pA = I.dev[5];
        pB = I.dev[6];
        pC = I.dev[7];
        pOut = I.out[0];
        params = {&iM, &iN, &iK, &fA, &fB, &pA, &pB, &pC, &pOut};
        if (plan.sk) {
            // Stream-K: G = resident CTAs (occupancy x SMs) share the
            // tiles x K-tiles units evenly; MAXSEG = most segments of a tile.
            int occ = 0;
            d.cuOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn->fn,
                                                          int(plan.block[0] * plan.block[1]),
                                                          size_t(plan.smem));
            const unsigned tiles = plan.tiles_x * plan.tiles_y;
            const unsigned long long U = (unsigned long long)tiles * plan.ktiles;
            // G = resident CTAs (SGEMM) or resident clusters of cg CTAs (TF32)
            unsigned G = unsigned(std::min<unsigned long long>(
                U, (unsigned long long)std::max(occ, 1) * unsigned(ctx->limits.sm_count) / plan.cg));
            // a CTA's share of K under 1024 -> one whole tile per CTA
            if (U / G * plan.ktile_k < 1024) G = tiles;
            auto cv = [&](unsigned long long v) { return ((v + 1) * G - 1) / U; };
            unsigned maxseg = 1;
            for (unsigned t = 0; t < tiles; ++t)
                maxseg = std::max(maxseg, unsigned(cv((unsigned long long)(t + 1) * plan.ktiles - 1) -
                                                   cv((unsigned long long)t * plan.ktiles) + 1));
            // TF32: one partial / counter per CTA of a pair (its 128 rows)
            // (+ a diagnostic timeline of 16 u64 per CTA when KTC_TF32_SK_TRACE is set)
            const size_t ws_part = size_t(tiles) * plan.cg * maxseg * plan.tile_floats * 4;
            const size_t ws = ws_part + size_t(G) * plan.cg * 128;
            sk_trace_off = ws_part;
            sk_trace_ctas = G * plan.cg;
            const size_t cn = size_t(tiles) * plan.cg * 4;
            if (ws > be->tail_ws_bytes) {
                if (be->tail_ws) d.cuMemFree(be->tail_ws);
                be->tail_ws = 0;
                be->tail_ws_bytes = 0;
                if (d.cuMemAlloc(&be->tail_ws, ws) != CUDA_SUCCESS) {
                    set_msg(out, "cannot allocate the stream-K workspace");
                    return KTC_OK;
                }
                be->tail_ws_bytes = ws;
            }
            if (cn > be->tail_cnt_bytes) {
                if (be->tail_cnt) d.cuMemFree(be->tail_cnt);
                be->tail_cnt = 0;
                be->tail_cnt_bytes = 0;
                if (d.cuMemAlloc(&be->tail_cnt, cn) != CUDA_SUCCESS ||
                    d.cuMemsetD32Async(be->tail_cnt, 0, cn / 4, ctx->stream) != CUDA_SUCCESS) {
                    set_msg(out, "cannot allocate the stream-K counters");
                    return KTC_OK;
                }
                be->tail_cnt_bytes = cn;
            }
            tk_ws = be->tail_ws;
            tk_cnt = be->tail_cnt;
            tk_full = unsigned(U);   // SK: p11 = units, p12 = MAXSEG, p13 = tiles_x, p14 = K-tiles
            tk_splits = maxseg;
            tk_gx = plan.tiles_x;
            tk_kt = plan.ktiles;
            if (fam == FAM_GEMM_TF32) {
                // gemm_tf32.cu SK: (..., tmap_a, tmap_b, tmap_c, W, cnt, U, MAXSEG, tile rows, K-blocks)
                params.insert(params.end(), {&tmap, &tmap2, &tmap3});
                plan.tma_mode = 0;  // tensor maps already passed
            }
            params.insert(params.end(), {&tk_ws, &tk_cnt, &tk_full, &tk_splits, &tk_gx, &tk_kt});
            plan.grid[0] = G * plan.cg;
            plan.grid[1] = 1;
        }
        if (plan.tailk) {
            // Split-K launch policy (tools/split_probe.py, DESIGN 4): per-SM
            // balance.  The tiles land ~evenly on the SMs, so a launch of c
            // CTAs per SM runs ceil(c) rounds on the busiest SM; cutting every
            // tile's K range into s CTAs (each K/s >= 4096) is worth it when
            // it evens the rounds out by more than the partial-tile reduction
            // costs (~3%).  8192x256x8192: 3.46 -> 6.92/7 tiles per SM, +14%;
            // with K/s = 1024 (2048^3, 64x128 tiles) the same rebalancing
            // measured 3% slower, so short splits are not offered.
            const unsigned tiles = plan.tiles_x * plan.tiles_y;
            const unsigned sms = unsigned(std::max(ctx->limits.sm_count, 1));
            const unsigned smax = std::min({8u, plan.ktiles, std::max(unsigned(I.K) / 4096u, 1u)});
            unsigned splits = 1;
            double best = -1.0;
            for (unsigned s = 1; s <= smax; ++s) {
                const double c = double(tiles) * s / sms;
                const double eff = c / std::ceil(c) * (s > 1 ? 0.97 : 1.0);
                if (eff > best + 1e-9) {
                    best = eff;
                    splits = s;
                }
            }
            if (const char* e = std::getenv("KTC_GEMM_SPLIT"))
                splits = std::min(unsigned(std::max(std::atoi(e), 1)), plan.ktiles);
            if (splits < 2) splits = 1;
            tk_full = splits > 1 ? 0 : tiles;
            tk_splits = splits;
            tk_gx = plan.tiles_x;
            tk_kt = plan.ktiles;
            const size_t ws = size_t(tiles - tk_full) * splits * plan.tile_floats * 4;
            const size_t cn = size_t(tiles - tk_full) * 4;
            if (ws > be->tail_ws_bytes) {
                if (be->tail_ws) d.cuMemFree(be->tail_ws);
                be->tail_ws = 0;
                be->tail_ws_bytes = 0;
                if (d.cuMemAlloc(&be->tail_ws, ws) != CUDA_SUCCESS) {
                    set_msg(out, "cannot allocate the split-K tail workspace");
                    return KTC_OK;
                }
                be->tail_ws_bytes = ws;
            }
            if (cn > be->tail_cnt_bytes) {
                if (be->tail_cnt) d.cuMemFree(be->tail_cnt);
                be->tail_cnt = 0;
                be->tail_cnt_bytes = 0;
                if (d.cuMemAlloc(&be->tail_cnt, cn) != CUDA_SUCCESS ||
                    d.cuMemsetD32Async(be->tail_cnt, 0, cn / 4, ctx->stream) != CUDA_SUCCESS) {
                    set_msg(out, "cannot allocate the split-K tail counters");
                    return KTC_OK;
                }
                be->tail_cnt_bytes = cn;
            }
            tk_ws = be->tail_ws ? be->tail_ws : pOut;  // never read without a tail
            tk_cnt = be->tail_cnt ? be->tail_cnt : pOut;
            params.insert(params.end(), {&tk_ws, &tk_cnt, &tk_full, &tk_splits, &tk_gx, &tk_kt});
            plan.grid[0] = tk_full + (tiles - tk_full) * splits;
            plan.grid[1] = 1;
        }
        if (plan.tma_mode == 2) {
            params.push_back(&tmap);
            params.push_back(&tmap2);
            if (fam == FAM_GEMM_TF32) params.push_back(&tmap3);
        }
    } else {
        st = refresh_custom_buffers(be);
        if (st) return st;
        scal_i.resize(I.args.size());
        scal_f.resize(I.args.size());
        ptrs.resize(I.args.size());
        size_t oi = 0;
        for (size_t a = 0; a < I.args.size(); ++a) {
            const auto& s = I.args[a];
            if (s.role == ktb::ArgRole::scalar) {
                if (s.type == ktb::ElementType::i32) {
                    scal_i[a] = (long long)(int)s.value;
                    params.push_back(&scal_i[a]);  // little-endian: low 4 bytes = int
                } else {
                    scal_f[a] = float(s.value);
                    params.push_back(&scal_f[a]);
                }
            } else if (s.role == ktb::ArgRole::output) {
                ptrs[a] = I.out[oi++];
                params.push_back(&ptrs[a]);
            } else {
                ptrs[a] = I.dev[a];
                params.push_back(&ptrs[a]);
            }
        }
        // outputs start from their recipe contents
        for (size_t k = 0; k < I.out_arg.size(); ++k) {
            CUresult rc = d.cuMemcpyDtoDAsync(I.out[k], I.dev[I.out_arg[k]],
                                              I.out_count[k] * 4, ctx->stream);
            if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuMemcpyDtoD(output init)");
        }
    }
    out->load_ms = ms_since(t0);

    // 3. run: outputs poisoned with NaN so a configuration that skips
    // elements can never pass on a previous configuration's results.
    t0 = Clock::now();
    if (fam != FAM_CUSTOM) {
        for (size_t k = 0; k < I.out.size(); ++k) {
            CUresult rc = d.cuMemsetD32Async(I.out[k], 0xFFFFFFFFu, I.out_count[k], ctx->stream);
            if (rc != CUDA_SUCCESS) return fail_cu(ctx, rc, "cuMemsetD32(output)");
        }
    }
    const long long launches0 = ctx->launches;
    float best = 0.0f;
    const int reps = r->repetitions > 0 ? r->repetitions : 1;
    std::vector<float> all(size_t(reps), 0.0f);
    const double bar = be->opts.prune_factor > 0.0 && I.best_verified_ms > 0.0
                           ? be->opts.prune_factor * I.best_verified_ms
                           : 0.0;
    int reps_done = reps;
    st = ktc_launch_timed_pruned(ctx, fn, plan.grid, plan.block, plan.smem, params.data(),
                                 be->opts.warmup, reps, be->opts.flush_l2, bar, &best, all.data(),
                                 &reps_done);
    if (sk_trace_ctas && std::getenv("KTC_TF32_SK_TRACE") && fam == FAM_GEMM_TF32 && !st) {
        // TF32 stream-K timeline of the last launch (diagnostic)
        static std::atomic<int> sk_n{0};
        std::vector<unsigned long long> host(size_t(sk_trace_ctas) * 16);
        if (d.cuCtxSynchronize() == CUDA_SUCCESS &&
            d.cuMemcpyDtoH(host.data(), be->tail_ws + sk_trace_off, host.size() * 8) == CUDA_SUCCESS) {
            const std::string path = std::string(std::getenv("KTC_TF32_SK_TRACE")) + "/sk_trace_" +
                                     std::to_string(sk_n++) + ".bin";
            if (FILE* f = std::fopen(path.c_str(), "wb")) {
                std::fwrite(host.data(), 8, host.size(), f);
                std::fclose(f);
            }
        }
    }
    if (trace_buf) {
        static std::atomic<int> trace_n{0};
        const size_t n = size_t(plan.grid[0]) * plan.grid[1];
        std::vector<unsigned long long> host(n * 4);
        if (!st && d.cuCtxSynchronize() == CUDA_SUCCESS &&
            d.cuMemcpyDtoH(host.data(), trace_buf, n * 32) == CUDA_SUCCESS) {
            const std::string path = std::string(conv_trace_dir()) + "/conv_trace_" +
                                     std::to_string(trace_n++) + ".bin";
            if (FILE* f = std::fopen(path.c_str(), "wb")) {
                const unsigned hdr[2] = {plan.grid[0], plan.grid[1]};
                std::fwrite(hdr, sizeof(hdr), 1, f);
                std::fwrite(host.data(), 32, n, f);
                std::fclose(f);
            }
        }
        d.cuMemFree(trace_buf);
    }
    double sum = 0.0;
    for (int k = 0; k < reps_done; ++k) sum += all[size_t(k)];
    out->mean_ms = sum / double(std::max(1, reps_done));
    out->run_ms = ms_since(t0);
    if (st) {
        set_msg(out, last_error());
        out->kernel_launches = int(ctx->launches - launches0);
        // Sticky faults poison the context: reset now so the next
        // configuration starts clean (inputs are rebuilt lazily).
        if (ctx->sticky && !ktc::g_isolated_worker) {
            be->modules.clear();  // modules died with the context
            be->tail_ws = be->tail_cnt = 0;
            be->tail_ws_bytes = be->tail_cnt_bytes = 0;
            free_inputs(be);
            int rs = ktc_reset(ctx);
            if (rs) return rs;
        }
        return KTC_OK;
    }
    if (!(best > 0.0f) || !std::isfinite(best)) {
        set_msg(out, "non-positive kernel time");
        return KTC_OK;
    }
    out->status = KTC_STATUS_SUCCESS;
    out->time_ms = double(best);
    out->n_outputs = int(I.out.size());

    // 4. verification on the device
    t0 = Clock::now();
    if (be->opts.verify && r->want_outputs && I.has_reference) {
        ktc_verify_report total{};
        total.pass = 1;
        for (size_t k = 0; k < I.out.size(); ++k) {
            ktc_verify_report rep;
            bool nan_abs = false, nan_rel = false;
            const double rel = fam == FAM_GEMM_TF32 ? std::max(be->opts.rel_tol, 1e-3)
                                                    : be->opts.rel_tol;
            st = verify_pair(ctx, I.out[k], I.ref[k], I.out_count[k], I.out_type[k], rel,
                             be->opts.abs_tol, &rep, &nan_abs, &nan_rel);
            if (st) return st;
            merge_reports(&total, rep, nan_abs, nan_rel, k);
        }
        out->report = total;
        out->verification = total.pass ? KTC_VERIFY_PASS : KTC_VERIFY_FAIL;
        if (total.pass && reps_done == reps &&
            (I.best_verified_ms <= 0.0 || out->time_ms < I.best_verified_ms))
            I.best_verified_ms = out->time_ms;  // the prune_factor bar: full best-of-N only
    }
    out->verify_ms = ms_since(t0);

    // 5. digests (adapter use: the reference tuner's digest comparison)
    if (be->opts.digest_outputs) {
        for (size_t k = 0; k < I.out.size() && k < KTC_MAX_OUTPUTS; ++k) {
            std::vector<uint32_t> h(I.out_count[k]);
            st = ktc_download(ctx, h.data(), I.out[k], h.size() * 4);
            if (st) return st;
            ktc_digest_hex(ktc_digest_words(h.data(), h.size()), out->output_digests[k]);
        }
    }
    out->kernel_launches = int(ctx->launches - launches0);
    return KTC_OK;
}

}  // namespace

using namespace ktc;

extern "C" {

void ktc_backend_default_options(ktc_backend_options* o) {
    std::memset(o, 0, sizeof(*o));
    o->warmup = 1;
    o->flush_l2 = 1;
    o->verify = 1;
    o->rel_tol = 1e-4;
    o->abs_tol = 1e-6;
    o->compile_threads = 0;
    o->cache_dir = nullptr;
    o->digest_outputs = 0;
    o->prune_factor = 0.0;
}

int ktc_backend_open(int ordinal, const ktc_backend_options* opts, ktc_backend** out) {
    *out = nullptr;
    bool isolate = opts && opts->isolate;
    if (const char* e = std::getenv("KTC_ISOLATE")) isolate = std::atoi(e) != 0;
    if (isolate && !ktc::g_isolated_worker) {
        ktc_backend_options o;
        if (opts) o = *opts;
        else ktc_backend_default_options(&o);
        std::string name, err;
        ktc::RemoteBackend* rb =
            ktc::remote_open(ordinal, o, o.cache_dir ? o.cache_dir : "", &name, &err);
        if (!rb) {
            set_error(err);
            return KTC_ERR_CUDA;
        }
        auto* be = new ktc_backend;
        be->remote = rb;
        be->opts = o;
        be->opts.cache_dir = nullptr;
        be->name = name + " (isolated)";
        *out = be;
        return KTC_OK;
    }
    ktc_ctx* ctx = nullptr;
    int st = ktc_open(ordinal, &ctx);
    if (st) return st;
    auto* be = new ktc_backend;
    be->ctx = ctx;
    if (opts) be->opts = *opts;
    else ktc_backend_default_options(&be->opts);
    if (be->opts.cache_dir) be->cache_dir = be->opts.cache_dir;
    be->opts.cache_dir = nullptr;
    CompileService::instance().configure(be->opts.compile_threads, be->cache_dir);
    be->name = std::string("cuda:sm_100a:") + ctx->limits.name;
    *out = be;
    return KTC_OK;
}

void ktc_backend_close(ktc_backend* be) {
    if (!be) return;
    if (be->remote) {
        ktc::remote_close(be->remote);
        delete be;
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    free_inputs(be);
    trace_phase("close: free inputs", t0);
    if (!be->ctx->sticky) {
        driver().cuCtxSetCurrent(be->ctx->cu);
        if (be->tail_ws) driver().cuMemFree(be->tail_ws);
        if (be->tail_cnt) driver().cuMemFree(be->tail_cnt);
        // Deferred to the pooled context (bulk unload): unloading here cost
        // 2-67 ms per closed job, and a background unloader stalled the next
        // job's 134 MB H2D copy by up to 0.8 s (driver serialization).
        for (ModuleEntry& m : be->modules) retire_module(be->ctx, m.mod);
    }
    trace_phase("close: + modules retired", t0);
    be->modules.clear();
    ktc_close(be->ctx);
    trace_phase("close: + context", t0);
    delete be;
}

const char* ktc_backend_name(ktc_backend* be) { return be ? be->name.c_str() : ""; }
ktc_ctx* ktc_backend_ctx(ktc_backend* be) { return be && !be->remote ? be->ctx : nullptr; }

int ktc_backend_evaluate(ktc_backend* be, const ktc_request* req, ktc_result* out) {
    if (!be || !req || !out) return KTC_ERR_INVALID;
    if (be->remote) return ktc::remote_evaluate(be->remote, req, out);
    try {
        return evaluate(be, req, out);
    } catch (const std::exception& e) {
        set_error(e.what());
        return KTC_ERR_INVALID;
    }
}

int ktc_backend_prefetch(ktc_backend* be, const ktc_request* req) {
    if (!be || !req) return KTC_ERR_INVALID;
    if (be->remote) return ktc::remote_prefetch(be->remote, req);
    try {
        const Family fam = family_of(req->kernel_name);
        std::string why;
        if (fam != FAM_CUSTOM && !check_layout(req, fam, &why)) return KTC_OK;
        // Plans need the problem scalars only (dims_of), not the inputs.
        if (!dims_valid(dims_of(req, fam), fam)) return KTC_OK;
        Plan plan;
        bool ok = fam == FAM_CONV   ? plan_conv(be, req, &plan, &why)
                  : fam == FAM_GEMM ? plan_gemm(be, req, &plan, &why)
                  : fam == FAM_GEMM_TF32 ? plan_gemm_tf32(be, req, &plan, &why)
                                         : plan_custom(be, req, &plan, &why);
        if (ok)
            CompileService::instance().prefetch(*plan.ksrc, plan.problem, plan.config,
                                                plan.compile_cost);
        return KTC_OK;
    } catch (const std::exception& e) {
        set_error(e.what());
        return KTC_ERR_INVALID;
    }
}

int ktc_drop_caches(int flags) {
    // (isolated backends: the worker processes keep their own caches)
    if (flags & KTC_DROP_COMPILED) CompileService::instance().drop_cache();
    if (flags & KTC_DROP_HOST_INPUTS) {
        RecipeCache& rc = recipe_cache();
        std::lock_guard<std::mutex> lk(rc.mu);
        rc.cache.clear();  // pinned blocks are freed when their last job releases them
    }
    return KTC_OK;
}

int ktc_backend_begin_search(ktc_backend* be) {
    if (!be) return KTC_ERR_INVALID;
    if (be->remote) return ktc::remote_begin_search(be->remote);
    if (be->in) be->in->best_verified_ms = 0.0;
    return KTC_OK;
}

size_t ktc_backend_prefetch_depth(ktc_backend* be) {
    if (!be) return 0;
    if (be->remote) return ktc::remote_prefetch_depth(be->remote);
    // Two configurations per pool thread in flight: a deeper window lets the
    // pool's longest-first ordering compile far-ahead configurations while
    // the evaluator compiles the one it needs itself (bench value 808-817
    // configs/s at 2 x threads, 626-639 at 2 x threads x 8 on one box).
    CompileService& cs = CompileService::instance();
    return size_t(2) * size_t(cs.threads()) * size_t(std::min(cs.batch(), 2));
}

int ktc_backend_set_reference(ktc_backend* be, const ktc_request* req, int n_buffers,
                              const void* const* buffers, const size_t* lengths, const int* types) {
    if (!be || !req) return KTC_ERR_INVALID;
    if (be->remote)
        return ktc::remote_set_reference(be->remote, req, n_buffers, buffers, lengths, types);
    int st = make_current(be->ctx);
    if (st) return st;
    const Family fam = family_of(req->kernel_name);
    be->bound = {};
    st = ensure_inputs(be, req, fam);
    if (st) return st;
    st = upload_reference(be, n_buffers, buffers, lengths, types);
    if (st) return st;
    be->bound.sig = be->in->sig;
    for (int k = 0; k < n_buffers; ++k) {
        const auto* b = static_cast<const unsigned char*>(buffers[k]);
        be->bound.bytes.emplace_back(b, b + lengths[k] * 4);
        be->bound.lengths.push_back(lengths[k]);
        be->bound.types.push_back(types[k]);
    }
    return KTC_OK;
}



int ktc_backend_read_output(ktc_backend* be, int index, void* dst, size_t bytes) {
    if (be && be->remote) return ktc::remote_read_output(be->remote, index, dst, bytes);
    if (!be || !be->in || index < 0 || index >= int(be->in->out.size())) return KTC_ERR_INVALID;
    size_t n = std::min(bytes, be->in->out_count[index] * 4);
    return ktc_download(be->ctx, dst, be->in->out[index], n);
}

int ktc_backend_read_reference(ktc_backend* be, const ktc_request* req, int index, void* dst,
                               size_t bytes, char digest_hex[17]) {
    if (!be || !req) return KTC_ERR_INVALID;
    if (be->remote)
        return ktc::remote_read_reference(be->remote, req, index, dst, bytes, digest_hex);
    int st = make_current(be->ctx);
    if (st) return st;
    st = ensure_inputs(be, req, family_of(req->kernel_name));
    if (st) return st;
    Inputs& I = *be->in;
    if (index < 0 || index >= int(I.out.size()) || !I.ref[index]) {
        set_error("no reference output " + std::to_string(index));
        return KTC_ERR_INVALID;
    }
    std::vector<uint32_t> h(I.out_count[index]);
    st = ktc_download(be->ctx, h.data(), I.ref[index], h.size() * 4);
    if (st) return st;
    if (dst) std::memcpy(dst, h.data(), std::min(bytes, h.size() * 4));
    if (digest_hex) ktc_digest_hex(ktc_digest_words(h.data(), h.size()), digest_hex);
    return KTC_OK;
}

}  // extern "C"
