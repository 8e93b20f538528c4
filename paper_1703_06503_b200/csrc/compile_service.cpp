// compile_service.cpp -- see compile_service.hpp.
#include "compile_service.hpp"

#include <nvPTXCompiler.h>
#include <nvrtc.h>
#include <sys/stat.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>

#include "core.hpp"

namespace ktc {

namespace {

const char* kMarker = "//@@KTC_BODY@@";
const char* kDefaultFastCompile = "0";

uint64_t fnv(const std::string& s, uint64_t h = 0xcbf29ce484222325ull) {
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    return h;
}

std::string hex64(uint64_t v) {
    char buf[17];
    std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(v));
    return buf;
}

std::string hash_name(const std::string& key) {
    return hex64(fnv(key)) + hex64(fnv(key, 0x84222325cbf29ce4ull));
}

// Options every tuning-time compile gets.  KTC_LINEINFO=1 adds -lineinfo
// (profiling runs: ncu source page); KTC_FAST_COMPILE=<0|min|mid|max>
// selects NVRTC's --Ofast-compile level.  Both are part of the cache key.
const std::vector<std::string>& base_options() {
    // Leaked on purpose: pool workers may still read it while static
    // destructors run (the atexit quiesce is registered before this static
    // would be constructed, so a destructible vector would die first).
    static const std::vector<std::string>* opts = [] {
        auto* o_ = new std::vector<std::string>();
        std::vector<std::string>& o = *o_;
        o = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=true"};
        const char* li = std::getenv("KTC_LINEINFO");
        if (li && std::strcmp(li, "0") != 0) o.push_back("-lineinfo");
        const char* fc = std::getenv("KTC_FAST_COMPILE");
        const std::string level = fc ? fc : kDefaultFastCompile;
        if (!level.empty() && level != "0") o.push_back("--Ofast-compile=" + level);
        return o_;
    }();
    return *opts;
}

std::string define_name(const std::string& d) { return d.substr(0, d.find('=')); }
std::string define_value(const std::string& d) {
    const size_t eq = d.find('=');
    return eq == std::string::npos ? "1" : d.substr(eq + 1);
}

// One NVRTC program holding every configuration of the batch.
std::string assemble(const KernelSource& src, const std::vector<const Defines*>& configs) {
    std::ostringstream s;
    s << src.prelude << "\n";
    for (size_t i = 0; i < configs.size(); ++i) {
        s << "namespace ktc_k" << i << " {\n";
        for (const std::string& d : *configs[i])
            s << "#define " << define_name(d) << " " << define_value(d) << "\n";
        s << "#define KTC_ENTRY " << src.entry_base << "_k" << i << "\n";
        s << src.body << "\n";
        for (const std::string& d : *configs[i]) s << "#undef " << define_name(d) << "\n";
        s << "#undef KTC_ENTRY\n}\n";
    }
    return s.str();
}

std::vector<std::string> problem_options(const Defines& problem) {
    std::vector<std::string> o;
    for (const std::string& d : problem) o.push_back("-D" + d);
    return o;
}

}  // namespace

KernelSource split_source(const std::string& name, const std::string& text,
                          const std::string& entry_base) {
    KernelSource s;
    const size_t at = text.find(kMarker);
    s.prelude = at == std::string::npos ? std::string() : text.substr(0, at);
    s.body = at == std::string::npos ? text : text.substr(at);
    s.entry_base = entry_base;
    s.id = name + "#" + hex64(fnv(text));
    return s;
}

CubinPtr nvrtc_compile(const std::string& src, const std::vector<std::string>& opts) {
    auto out = std::make_shared<Cubin>();
    auto t0 = std::chrono::steady_clock::now();
    nvrtcProgram prog = nullptr;
    nvrtcResult rc = nvrtcCreateProgram(&prog, src.c_str(), "ktc_kernel.cu", 0, nullptr, nullptr);
    if (rc != NVRTC_SUCCESS) {
        out->log = std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(rc);
        return out;
    }
    std::vector<const char*> argv;
    for (const auto& o : base_options()) argv.push_back(o.c_str());
    for (const auto& o : opts) argv.push_back(o.c_str());
    rc = nvrtcCompileProgram(prog, int(argv.size()), argv.data());
    size_t log_size = 0;
    nvrtcGetProgramLogSize(prog, &log_size);
    if (log_size > 1) {
        std::string log(log_size, '\0');
        nvrtcGetProgramLog(prog, log.data());
        while (!log.empty() && (log.back() == '\0' || log.back() == '\n')) log.pop_back();
        out->log = log;
    }
    if (rc == NVRTC_SUCCESS) {
        size_t n = 0;
        nvrtcGetCUBINSize(prog, &n);
        out->image.resize(n);
        nvrtcGetCUBIN(prog, out->image.data());
    } else if (out->log.empty()) {
        out->log = nvrtcGetErrorString(rc);
    }
    nvrtcDestroyProgram(&prog);
    out->compile_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

CubinPtr ptx_compile(const std::string& ptx) {
    auto out = std::make_shared<Cubin>();
    auto t0 = std::chrono::steady_clock::now();
    nvPTXCompilerHandle h = nullptr;
    if (nvPTXCompilerCreate(&h, ptx.size(), ptx.c_str()) != NVPTXCOMPILE_SUCCESS) {
        out->log = "nvPTXCompilerCreate failed";
        return out;
    }
    std::vector<const char*> argv = {"--gpu-name=sm_100a", "-O3"};
    const char* li = std::getenv("KTC_LINEINFO");
    if (li && std::strcmp(li, "0") != 0) argv.push_back("--generate-line-info");
    const nvPTXCompileResult rc = nvPTXCompilerCompile(h, int(argv.size()), argv.data());
    size_t n = 0;
    if (rc == NVPTXCOMPILE_SUCCESS) {
        nvPTXCompilerGetCompiledProgramSize(h, &n);
        out->image.resize(n);
        nvPTXCompilerGetCompiledProgram(h, out->image.data());
    } else {
        nvPTXCompilerGetErrorLogSize(h, &n);
        std::string log(n, '\0');
        if (n) nvPTXCompilerGetErrorLog(h, log.data());
        while (!log.empty() && (log.back() == '\0' || log.back() == '\n')) log.pop_back();
        out->log = "ptxas: " + (log.empty() ? std::string("error ") + std::to_string(int(rc)) : log);
    }
    nvPTXCompilerDestroy(&h);
    out->compile_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

CompileService& CompileService::instance() {
    // Intentionally leaked (workers outlive statics); quiesced at exit.
    static CompileService* svc = [] {
        auto* s = new CompileService;
        (void)base_options();  // construct before the quiesce handler is registered
        std::atexit([] { CompileService::instance().quiesce(); });
        return s;
    }();
    return *svc;
}

void CompileService::drop_cache() {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto it = cache_.begin(); it != cache_.end();) {
        if (it->second.wait_for(std::chrono::seconds(0)) == std::future_status::ready)
            it = cache_.erase(it);
        else
            ++it;
    }
}

void CompileService::quiesce() {
    std::unique_lock<std::mutex> lk(mu_);
    exiting_ = true;
    queues_.clear();
    queued_cost_ = 0.0;
    idle_cv_.wait_for(lk, std::chrono::seconds(60), [&] { return running_ == 0; });
}

void CompileService::configure(int threads, const std::string& cache_dir, int batch) {
    std::lock_guard<std::mutex> lk(mu_);
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    want_threads_ = threads;
    if (const char* env = std::getenv("KTC_COMPILE_BATCH")) batch = std::atoi(env);
    batch_ = std::max(1, std::min(batch, 32));
    if (const char* env = std::getenv("KTC_PTX_BATCH")) ptx_batch_ = std::max(1, std::min(std::atoi(env), 32));
    cache_dir_ = cache_dir;
    if (!cache_dir_.empty()) ::mkdir(cache_dir_.c_str(), 0755);
    ensure_workers_locked();
}

void CompileService::ensure_workers_locked() {
    if (want_threads_ <= 0) want_threads_ = int(std::max(1u, std::thread::hardware_concurrency()));
    while (int(workers_.size()) < want_threads_) workers_.emplace_back([this] { worker(); });
}

std::string CompileService::batch_key_of(const KernelSource& src, const Defines& problem) const {
    int major = 0, minor = 0;
    nvrtcVersion(&major, &minor);
    std::string k = src.id + "|nvrtc" + std::to_string(major) + "." + std::to_string(minor);
    for (const auto& o : base_options()) k += "|" + o;
    for (const auto& d : problem) k += "|P" + d;
    return k;
}

std::string CompileService::key_of(const KernelSource& src, const Defines& problem,
                                   const Defines& config) const {
    std::string k = batch_key_of(src, problem);
    for (const auto& d : config) k += "|C" + d;
    return k;
}

KernelPtr CompileService::load_disk(const std::string& key) {
    if (cache_dir_.empty()) return nullptr;
    std::ifstream ref(cache_dir_ + "/" + hash_name(key) + ".ref");
    std::string file, entry;
    if (!(ref >> file >> entry)) return nullptr;
    std::ifstream in(cache_dir_ + "/" + file, std::ios::binary);
    if (!in) return nullptr;
    auto c = std::make_shared<Cubin>();
    c->image.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    if (c->image.empty()) return nullptr;
    auto k = std::make_shared<CompiledKernel>();
    k->cubin = c;
    k->entry = entry;
    return k;
}

void CompileService::store_disk(const std::string& key, const CompiledKernel& k) {
    if (cache_dir_.empty() || !k.ok()) return;
    const std::string file = hash_name(std::to_string(reinterpret_cast<uintptr_t>(k.cubin.get())) +
                                       key) + ".cubin";
    const std::string tid = std::to_string(std::hash<std::thread::id>()(std::this_thread::get_id()));
    {
        std::ofstream out(cache_dir_ + "/" + file + ".tmp" + tid, std::ios::binary);
        out.write(k.cubin->image.data(), std::streamsize(k.cubin->image.size()));
    }
    std::rename((cache_dir_ + "/" + file + ".tmp" + tid).c_str(), (cache_dir_ + "/" + file).c_str());
    {
        std::ofstream ref(cache_dir_ + "/" + hash_name(key) + ".ref.tmp" + tid);
        ref << file << " " << k.entry << "\n";
    }
    std::rename((cache_dir_ + "/" + hash_name(key) + ".ref.tmp" + tid).c_str(),
                (cache_dir_ + "/" + hash_name(key) + ".ref").c_str());
}

void CompileService::run_batch(Batch b) {
    // Disk hits first.
    std::vector<Item> todo;
    for (Item& it : b.items) {
        if (KernelPtr k = load_disk(it.key)) it.promise->set_value(k);
        else todo.push_back(std::move(it));
    }
    if (todo.empty()) return;
    const std::vector<std::string> popts = problem_options(b.problem);
    if (!b.src->batchable) {
        for (Item& it : todo) {
            std::vector<std::string> o = popts;
            for (const std::string& d : problem_options(it.config)) o.push_back(d);
            CubinPtr c = nvrtc_compile(b.src->body, o);
            {
                std::lock_guard<std::mutex> lk(mu_);
                compile_ms_ += c->compile_ms;
                ++programs_;
            }
            auto k = std::make_shared<CompiledKernel>();
            k->cubin = c;
            k->entry = b.src->fixed_entry;
            k->log = c->log;
            k->compile_ms = c->compile_ms;
            store_disk(it.key, *k);
            it.promise->set_value(k);
        }
        return;
    }
    auto compile_group = [&](const std::vector<Item*>& group) -> bool {
        std::vector<const Defines*> cfgs;
        for (Item* it : group) cfgs.push_back(&it->config);
        CubinPtr c;
        if (b.src->ptx_generator) {
            std::string ptx;
            try {
                ptx = b.src->ptx_generator(b.problem, cfgs, b.src->entry_base);
            } catch (const std::exception& e) {
                auto bad = std::make_shared<Cubin>();
                bad->log = std::string("ptx generator: ") + e.what();
                c = bad;
            }
            if (!c) c = ptx_compile(ptx);
        } else {
            c = nvrtc_compile(assemble(*b.src, cfgs), popts);
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            compile_ms_ += c->compile_ms;
            ++programs_;
        }
        if (!c->ok() && group.size() > 1) return false;
        for (size_t i = 0; i < group.size(); ++i) {
            auto k = std::make_shared<CompiledKernel>();
            k->cubin = c;
            k->entry = b.src->entry_base + "_k" + std::to_string(i);
            k->log = c->log;
            k->compile_ms = c->compile_ms;
            k->batch = int(group.size());
            store_disk(group[i]->key, *k);
            group[i]->promise->set_value(k);
        }
        return true;
    };
    std::vector<Item*> all;
    for (Item& it : todo) all.push_back(&it);
    if (!compile_group(all))
        for (Item* it : all) compile_group({it});  // attribute errors to their configuration
}

int CompileService::threads() {
    std::lock_guard<std::mutex> lk(mu_);
    return want_threads_ > 0 ? want_threads_ : int(std::max(1u, std::thread::hardware_concurrency()));
}

int CompileService::batch() {
    std::lock_guard<std::mutex> lk(mu_);
    return batch_;
}

// Program formation (under mu_).  Configurations wait as items in one queue
// per (source, problem); a thread that picks work forms its NVRTC program
// then, from the queue of the oldest item:
//   * the most expensive queued item first (longest-processing-time-first:
//     the makespan of a burst -- a fresh job, the end of a search -- is set
//     by its slowest compile, so that one must not start last);
//   * then further items, cheapest first, while the program stays within
//     this thread's fair share of the queued cost (total / pool threads)
//     and `batch_` items.
// A backlogged pool therefore builds full programs (NVRTC's fixed ~50 ms per
// program amortized); an under-loaded one spreads the work evenly.  Items
// the evaluator needs before a pool thread took them are compiled by the
// evaluator itself (get()), so nothing waits behind the ordering.
bool CompileService::take_program_locked(Batch* out) {
    auto qit = queues_.end();
    for (auto it = queues_.begin(); it != queues_.end(); ++it)
        if (!it->second.items.empty() &&
            (qit == queues_.end() || it->second.oldest() < qit->second.oldest()))
            qit = it;
    if (qit == queues_.end()) return false;
    Queue& q = qit->second;
    out->src = q.src;
    out->problem = q.problem;
    out->items.clear();
    auto take = [&](size_t i) {
        queued_cost_ -= q.items[i].cost;
        out->items.push_back(std::move(q.items[i]));
        q.items.erase(q.items.begin() + long(i));
    };
    if (!q.src->batchable) {
        size_t oldest = 0;
        for (size_t i = 1; i < q.items.size(); ++i)
            if (q.items[i].born < q.items[oldest].born) oldest = i;
        take(oldest);
    } else {
        size_t big = 0;
        for (size_t i = 1; i < q.items.size(); ++i)
            if (q.items[i].cost > q.items[big].cost) big = i;
        double total = q.items[big].cost;
        const double share = (queued_cost_ + total_inflight_) / double(std::max(1, want_threads_));
        // PTX-generator families: ptxas has no NVVM-style fixed cost to
        // amortise, and multi-entry modules measured slower (bench value
        // ~800 configs/s with one configuration per program vs ~700 with 8),
        // so they compile one configuration per program unless KTC_PTX_BATCH.
        const int cap = q.src->ptx_generator ? ptx_batch_ : batch_;
        take(big);
        while (!q.items.empty() && int(out->items.size()) < cap) {
            size_t small = 0;
            for (size_t i = 1; i < q.items.size(); ++i)
                if (q.items[i].cost < q.items[small].cost) small = i;
            if (total + q.items[small].cost > share) break;
            total += q.items[small].cost;
            take(small);
        }
    }
    if (q.items.empty()) queues_.erase(qit);
    return true;
}

void CompileService::worker() {
    for (;;) {
        Batch b;
        double cost = 0.0;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return !queues_.empty() && !exiting_; });
            take_program_locked(&b);
            for (const Item& it : b.items) cost += it.cost;
            total_inflight_ += cost;
            ++running_;
        }
        run_batch(std::move(b));
        std::lock_guard<std::mutex> lk(mu_);
        total_inflight_ -= cost;
        if (--running_ == 0) idle_cv_.notify_all();
    }
}

std::shared_future<KernelPtr> CompileService::enlist_locked(const KernelSource& src,
                                                            const Defines& problem,
                                                            const Defines& config, double cost,
                                                            bool* created) {
    const std::string key = key_of(src, problem, config);
    auto it = cache_.find(key);
    if (it != cache_.end()) {
        *created = false;
        return it->second;
    }
    *created = true;
    auto promise = std::make_shared<std::promise<KernelPtr>>();
    std::shared_future<KernelPtr> fut = promise->get_future().share();
    if (cache_.size() > 50000) cache_.clear();  // bound host memory
    cache_.emplace(key, fut);
    const std::string qkey = src.batchable ? batch_key_of(src, problem) : key;
    auto& sp = sources_[src.id];
    if (!sp) sp = std::make_shared<const KernelSource>(src);
    Queue& q = queues_[qkey];
    if (!q.src) {
        q.src = sp;
        q.problem = problem;
    }
    q.items.push_back(Item{config, key, promise, std::max(cost, 1e-3),
                           std::chrono::steady_clock::now()});
    queued_cost_ += q.items.back().cost;
    cv_.notify_one();
    return fut;
}

void CompileService::prefetch(const KernelSource& src, const Defines& problem,
                              const Defines& config, double cost) {
    std::lock_guard<std::mutex> lk(mu_);
    ensure_workers_locked();
    bool created = false;
    enlist_locked(src, problem, config, cost, &created);
}

KernelPtr CompileService::get(const KernelSource& src, const Defines& problem,
                              const Defines& config, bool* hit, double cost) {
    std::shared_future<KernelPtr> fut;
    Batch mine;
    bool run_here = false;
    {
        std::lock_guard<std::mutex> lk(mu_);
        ensure_workers_locked();
        bool created = false;
        fut = enlist_locked(src, problem, config, cost, &created);
        if (hit) *hit = !created && fut.wait_for(std::chrono::seconds(0)) == std::future_status::ready;
        // Still queued (no pool thread took it yet): compile it right here,
        // alone -- the caller is waiting for exactly this configuration.
        const std::string key = key_of(src, problem, config);
        const std::string qkey = src.batchable ? batch_key_of(src, problem) : key;
        auto qit = queues_.find(qkey);
        if (qit != queues_.end()) {
            Queue& q = qit->second;
            for (size_t i = 0; i < q.items.size(); ++i)
                if (q.items[i].key == key) {
                    mine.src = q.src;
                    mine.problem = q.problem;
                    queued_cost_ -= q.items[i].cost;
                    mine.items.push_back(std::move(q.items[i]));
                    q.items.erase(q.items.begin() + long(i));
                    if (q.items.empty()) queues_.erase(qit);
                    run_here = true;
                    break;
                }
        }
    }
    if (run_here) run_batch(std::move(mine));
    return fut.get();
}

double CompileService::total_compile_ms() {
    std::lock_guard<std::mutex> lk(mu_);
    return compile_ms_;
}

size_t CompileService::programs_compiled() {
    std::lock_guard<std::mutex> lk(mu_);
    return programs_;
}

void CompileService::reset_stats() {
    std::lock_guard<std::mutex> lk(mu_);
    compile_ms_ = 0.0;
    programs_ = 0;
}

}  // namespace ktc

using namespace ktc;

extern "C" int ktc_compile(const char* src, const char* const* opts, int nopts, void** cubin,
                           size_t* cubin_size, char* log, size_t log_cap) {
    std::vector<std::string> o;
    for (int i = 0; i < nopts; ++i) o.emplace_back(opts[i]);
    // Family sources need an entry name when compiled stand-alone.
    std::string text = src;
    if (text.find("KTC_ENTRY") != std::string::npos) o.push_back("-DKTC_ENTRY=ktc_entry");
    CubinPtr c = nvrtc_compile(text, o);
    if (log && log_cap) std::snprintf(log, log_cap, "%s", c->log.c_str());
    if (!c->ok()) {
        set_error("NVRTC: " + c->log.substr(0, 2000));
        *cubin = nullptr;
        *cubin_size = 0;
        return KTC_ERR_NVRTC;
    }
    *cubin = std::malloc(c->image.size());
    std::memcpy(*cubin, c->image.data(), c->image.size());
    *cubin_size = c->image.size();
    return KTC_OK;
}

static int codegen(bool gemm, const char* const* defines, int ndefines, void** cubin,
                   size_t* cubin_size, char** ptx, char* log, size_t log_cap) {
    Defines problem, config;
    for (int i = 0; i < ndefines; ++i) {
        std::string d = defines[i];
        if (d.rfind("-D", 0) == 0) d = d.substr(2);
        (d.rfind("FS=", 0) == 0 ? problem : config).push_back(d);
    }
    std::string text;
    try {
        text = gemm ? gemm_ptx_module(problem, {&config}, "gemm")
                    : conv_ptx_module(problem, {&config}, "conv2d");
    } catch (const std::exception& e) {
        if (log && log_cap) std::snprintf(log, log_cap, "%s", e.what());
        set_error(e.what());
        return KTC_ERR_INVALID;
    }
    if (ptx) {
        *ptx = static_cast<char*>(std::malloc(text.size() + 1));
        std::memcpy(*ptx, text.c_str(), text.size() + 1);
    }
    CubinPtr c = ptx_compile(text);
    if (log && log_cap) std::snprintf(log, log_cap, "%s", c->log.c_str());
    if (!c->ok()) {
        set_error(c->log.substr(0, 2000));
        *cubin = nullptr;
        *cubin_size = 0;
        return KTC_ERR_NVRTC;
    }
    *cubin = std::malloc(c->image.size());
    std::memcpy(*cubin, c->image.data(), c->image.size());
    *cubin_size = c->image.size();
    return KTC_OK;
}

extern "C" int ktc_codegen_conv(const char* const* defines, int ndefines, void** cubin,
                                size_t* cubin_size, char** ptx, char* log, size_t log_cap) {
    return codegen(false, defines, ndefines, cubin, cubin_size, ptx, log, log_cap);
}

extern "C" int ktc_codegen_gemm(const char* const* defines, int ndefines, void** cubin,
                                size_t* cubin_size, char** ptx, char* log, size_t log_cap) {
    return codegen(true, defines, ndefines, cubin, cubin_size, ptx, log, log_cap);
}
