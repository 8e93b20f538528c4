// nvrtc_pool.hpp -- NVRTC compilation for sm_100a with a shared host thread
// pool and a cubin cache keyed by (source, options, arch, NVRTC version).
//
// Compilation is the throughput limiter of tuning (SURVEY 7 "Hard parts" 1:
// ~60-150 ms per configuration per core).  Evaluation on the GPU takes a few
// milliseconds, so the pool compiles ahead of the device: callers prefetch()
// the next configurations while the current one runs.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace ktc {

struct Cubin {
    std::vector<char> image;  // empty on failure
    std::string log;          // NVRTC log (errors)
    double compile_ms = 0.0;  // 0 for cache hits loaded from disk
    bool ok() const { return !image.empty(); }
};

using CubinPtr = std::shared_ptr<const Cubin>;

// Compiles `src` with `opts` (+ the fixed arch/std options) synchronously.
CubinPtr nvrtc_compile(const std::string& src, const std::vector<std::string>& opts);

class CompileService {
  public:
    static CompileService& instance();

    // Sets the pool size (0 = hardware threads) and the disk cache dir.
    void configure(int threads, const std::string& cache_dir);

    // Returns the cubin, compiling on the calling thread unless it is cached
    // or already being compiled by the pool.  `hit` reports a cache hit.
    CubinPtr get(const std::string& src_id, const std::string& src,
                 const std::vector<std::string>& opts, bool* hit);

    // Queues a background compilation (no-op if cached or in flight).
    void prefetch(const std::string& src_id, const std::string& src,
                  const std::vector<std::string>& opts);

    size_t threads() const { return workers_.size(); }
    double total_compile_ms();
    void reset_stats();

  private:
    CompileService() = default;
    ~CompileService();
    struct Job {
        std::string key, src;
        std::vector<std::string> opts;
        std::shared_ptr<std::promise<CubinPtr>> promise;
    };
    std::string make_key(const std::string& src_id, const std::vector<std::string>& opts) const;
    CubinPtr load_disk(const std::string& key);
    void store_disk(const std::string& key, const Cubin& c);
    CubinPtr run(const Job& job);
    void worker();
    void ensure_workers_locked();

    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Job> queue_;
    std::unordered_map<std::string, std::shared_future<CubinPtr>> cache_;
    std::vector<std::thread> workers_;
    int want_threads_ = 0;
    std::string cache_dir_;
    bool stop_ = false;
    double compile_ms_ = 0.0;
};

}  // namespace ktc
