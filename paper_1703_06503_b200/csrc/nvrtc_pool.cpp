// nvrtc_pool.cpp -- see nvrtc_pool.hpp.
#include "nvrtc_pool.hpp"

#include <nvrtc.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sys/stat.h>

#include "core.hpp"

namespace ktc {

namespace {

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

const std::vector<std::string>& base_options() {
    static const std::vector<std::string> opts = {
        "--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true",
        "-default-device"};
    return opts;
}

}  // namespace

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

CompileService& CompileService::instance() {
    static CompileService* svc = new CompileService;  // never destroyed: workers outlive statics
    return *svc;
}

CompileService::~CompileService() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}

void CompileService::configure(int threads, const std::string& cache_dir) {
    std::lock_guard<std::mutex> lk(mu_);
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    want_threads_ = threads;
    cache_dir_ = cache_dir;
    if (!cache_dir_.empty()) ::mkdir(cache_dir_.c_str(), 0755);
    ensure_workers_locked();
}

void CompileService::ensure_workers_locked() {
    if (want_threads_ <= 0) want_threads_ = int(std::max(1u, std::thread::hardware_concurrency()));
    while (int(workers_.size()) < want_threads_) workers_.emplace_back([this] { worker(); });
}

std::string CompileService::make_key(const std::string& src_id,
                                     const std::vector<std::string>& opts) const {
    int major = 0, minor = 0;
    nvrtcVersion(&major, &minor);
    std::string k = src_id + "|nvrtc" + std::to_string(major) + "." + std::to_string(minor);
    for (const auto& o : base_options()) k += "|" + o;
    for (const auto& o : opts) k += "|" + o;
    return k;
}

CubinPtr CompileService::load_disk(const std::string& key) {
    if (cache_dir_.empty()) return nullptr;
    std::string path = cache_dir_ + "/" + hex64(fnv(key)) + hex64(fnv(key, 0x84222325cbf29ce4ull)) +
                       ".cubin";
    std::ifstream in(path, std::ios::binary);
    if (!in) return nullptr;
    auto c = std::make_shared<Cubin>();
    c->image.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    if (c->image.empty()) return nullptr;
    return c;
}

void CompileService::store_disk(const std::string& key, const Cubin& c) {
    if (cache_dir_.empty() || !c.ok()) return;
    std::string path = cache_dir_ + "/" + hex64(fnv(key)) + hex64(fnv(key, 0x84222325cbf29ce4ull)) +
                       ".cubin";
    std::string tmp = path + ".tmp" + std::to_string(std::hash<std::thread::id>()(
                                          std::this_thread::get_id()));
    {
        std::ofstream out(tmp, std::ios::binary);
        out.write(c.image.data(), std::streamsize(c.image.size()));
    }
    std::rename(tmp.c_str(), path.c_str());
}

CubinPtr CompileService::run(const Job& job) {
    CubinPtr c = load_disk(job.key);
    if (!c) {
        c = nvrtc_compile(job.src, job.opts);
        store_disk(job.key, *c);
        std::lock_guard<std::mutex> lk(mu_);
        compile_ms_ += c->compile_ms;
    }
    return c;
}

void CompileService::worker() {
    for (;;) {
        Job job;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || !queue_.empty(); });
            if (stop_) return;
            job = std::move(queue_.front());
            queue_.pop_front();
        }
        job.promise->set_value(run(job));
    }
}

CubinPtr CompileService::get(const std::string& src_id, const std::string& src,
                             const std::vector<std::string>& opts, bool* hit) {
    const std::string key = make_key(src_id, opts);
    std::shared_future<CubinPtr> fut;
    std::shared_ptr<std::promise<CubinPtr>> mine;
    {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = cache_.find(key);
        if (it != cache_.end()) {
            fut = it->second;
        } else {
            mine = std::make_shared<std::promise<CubinPtr>>();
            fut = mine->get_future().share();
            if (cache_.size() > 20000) cache_.clear();  // bound host memory
            cache_.emplace(key, fut);
        }
    }
    if (mine) {
        if (hit) *hit = false;
        CubinPtr c = run(Job{key, src, opts, mine});
        mine->set_value(c);
        return c;
    }
    if (hit) *hit = fut.wait_for(std::chrono::seconds(0)) == std::future_status::ready;
    return fut.get();
}

void CompileService::prefetch(const std::string& src_id, const std::string& src,
                              const std::vector<std::string>& opts) {
    const std::string key = make_key(src_id, opts);
    std::lock_guard<std::mutex> lk(mu_);
    if (cache_.count(key)) return;
    ensure_workers_locked();
    auto promise = std::make_shared<std::promise<CubinPtr>>();
    if (cache_.size() > 20000) cache_.clear();
    cache_.emplace(key, promise->get_future().share());
    queue_.push_back(Job{key, src, opts, promise});
    cv_.notify_one();
}

double CompileService::total_compile_ms() {
    std::lock_guard<std::mutex> lk(mu_);
    return compile_ms_;
}

void CompileService::reset_stats() {
    std::lock_guard<std::mutex> lk(mu_);
    compile_ms_ = 0.0;
}

}  // namespace ktc

using namespace ktc;

extern "C" int ktc_compile(const char* src, const char* const* opts, int nopts, void** cubin,
                           size_t* cubin_size, char* log, size_t log_cap) {
    std::vector<std::string> o;
    for (int i = 0; i < nopts; ++i) o.emplace_back(opts[i]);
    CubinPtr c = nvrtc_compile(src, o);
    if (log && log_cap) {
        std::snprintf(log, log_cap, "%s", c->log.c_str());
    }
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
