// compile_service.hpp -- tuning-time compilation for sm_100a: a shared host
// thread pool, cost-aware program formation and a cubin cache.
//
// Compilation is the throughput limiter of tuning (SURVEY 7 "Hard parts" 1).
// Levers:
//   * no NVVM for the built-in families: their KernelSource carries a PTX
//     generator (ptxgen_conv.cpp / ptxgen_gemm.cpp) and programs go straight
//     to ptxas (nvPTXCompiler, in process); NVRTC compiles the rest (TF32,
//     custom kernels) from source;
//   * ahead-of-time: callers prefetch() the configurations they will evaluate
//     next, so the pool compiles while the device runs;
//   * program formation (take_program_locked): longest estimated compile
//     first, then cheap configurations up to the thread's fair share of the
//     queued cost and `batch` entries (each configuration its own entry
//     _k<i>; in NVRTC sources, its own namespace and macro block).  A
//     program that fails is split back into single compilations so errors
//     land on the configuration that caused them.
// NVRTC sources carry a `//@@KTC_BODY@@` marker: the text above it (helpers,
// problem-level symbols) appears once per program, the text below it once per
// configuration with KTC_ENTRY naming the kernel.
#pragma once

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace ktc {

struct Cubin {
    std::vector<char> image;  // empty on failure
    std::string log;
    double compile_ms = 0.0;
    bool ok() const { return !image.empty(); }
};
using CubinPtr = std::shared_ptr<const Cubin>;

// A family's source split at the body marker.
// Defines are "NAME=VALUE" strings.
using Defines = std::vector<std::string>;

struct KernelSource {
    std::string id;          // identity (name + content hash)
    std::string prelude;
    std::string body;
    std::string entry_base;  // kernel entry = entry_base + "_k<i>"
    // Custom (user) kernels: compiled alone, whole text, own entry name,
    // configuration passed as -D options.
    bool batchable = true;
    std::string fixed_entry;
    // Direct code generation (no NVRTC): emits the PTX module of a batch
    // (entries entry_base_k<i>), compiled by ptxas in process.
    std::function<std::string(const Defines& problem, const std::vector<const Defines*>& configs,
                              const std::string& entry_base)>
        ptx_generator;
};
KernelSource split_source(const std::string& name, const std::string& text,
                          const std::string& entry_base);

struct CompiledKernel {
    CubinPtr cubin;     // shared by every configuration of the batch
    std::string entry;  // this configuration's kernel symbol
    std::string log;
    double compile_ms = 0.0;  // wall time of the (batch) compilation
    int batch = 1;
    bool ok() const { return cubin && cubin->ok(); }
};
using KernelPtr = std::shared_ptr<const CompiledKernel>;


// Raw NVRTC compile of `src` with extra options (fixed arch/std options added).
CubinPtr nvrtc_compile(const std::string& src, const std::vector<std::string>& opts);

// ptxas (nvPTXCompiler, in process) of a PTX module for sm_100a.
CubinPtr ptx_compile(const std::string& ptx);

// PTX generators of the convolution and SGEMM families (ptxgen_*.cpp).
std::string conv_ptx_module(const Defines& problem, const std::vector<const Defines*>& configs,
                            const std::string& entry_base);
std::string gemm_ptx_module(const Defines& problem, const std::vector<const Defines*>& configs,
                            const std::string& entry_base);

class CompileService {
  public:
    static CompileService& instance();

    // Pool size (0 = hardware threads), disk cache dir ("" = memory only),
    // configurations per NVRTC program (1 disables batching).
    void configure(int threads, const std::string& cache_dir, int batch = 8);

    // `cost`: relative compile-cost estimate (1 ~ a small configuration),
    // used to order and size programs (see take_program_locked).
    KernelPtr get(const KernelSource& src, const Defines& problem, const Defines& config,
                  bool* hit, double cost = 1.0);
    void prefetch(const KernelSource& src, const Defines& problem, const Defines& config,
                  double cost = 1.0);
    int threads();
    int batch();
    double total_compile_ms();
    size_t programs_compiled();
    void reset_stats();
    // Forgets every finished compile (in-memory cache); in-flight ones finish.
    void drop_cache();

    // Process exit (atexit): drops every queued (speculative) compile and
    // waits for the programs already in ptxas/NVRTC to finish, so no worker
    // is inside the compiler while static destructors run.
    void quiesce();

  private:
    CompileService() = default;
    struct Item {
        Defines config;
        std::string key;
        std::shared_ptr<std::promise<KernelPtr>> promise;
        double cost = 1.0;
        std::chrono::steady_clock::time_point born;
    };
    struct Batch {  // one NVRTC program
        std::shared_ptr<const KernelSource> src;
        Defines problem;
        std::vector<Item> items;
    };
    struct Queue {  // waiting configurations of one (source, problem)
        std::shared_ptr<const KernelSource> src;
        Defines problem;
        std::vector<Item> items;
        std::chrono::steady_clock::time_point oldest() const {
            auto t = items.front().born;
            for (const Item& it : items) t = std::min(t, it.born);
            return t;
        }
    };
    std::string key_of(const KernelSource& src, const Defines& problem, const Defines& config) const;
    std::string batch_key_of(const KernelSource& src, const Defines& problem) const;
    void run_batch(Batch b);
    bool take_program_locked(Batch* out);
    void worker();
    void ensure_workers_locked();
    // Registers `config` (if new) in its queue; returns the future and
    // whether this call created it.
    std::shared_future<KernelPtr> enlist_locked(const KernelSource& src, const Defines& problem,
                                                const Defines& config, double cost, bool* created);
    KernelPtr load_disk(const std::string& key);
    void store_disk(const std::string& key, const CompiledKernel& k);

    std::mutex mu_;
    std::condition_variable cv_;
    std::map<std::string, Queue> queues_;  // by batch key (source, problem)
    double queued_cost_ = 0.0;               // sum of queued item costs
    double total_inflight_ = 0.0;            // cost of programs being compiled
    int running_ = 0;                        // batches inside run_batch
    bool exiting_ = false;
    std::condition_variable idle_cv_;
    std::unordered_map<std::string, std::shared_future<KernelPtr>> cache_;
    std::map<std::string, std::shared_ptr<const KernelSource>> sources_;
    std::vector<std::thread> workers_;
    int want_threads_ = 0;
    int batch_ = 8;
    int ptx_batch_ = 1;  // configurations per program for the PTX-generator families
    std::string cache_dir_;
    double compile_ms_ = 0.0;
    size_t programs_ = 0;
};

}  // namespace ktc
