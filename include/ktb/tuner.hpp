// ktb/tuner.hpp -- tuning orchestration (reference tuner.hpp): host output
// verification, the job description, the outcome record, compose_space and
// run_tuning -- plus run_tuning_sharded, which spreads the order-independent
// strategies (full, random) over several devices and merges the rows back
// into exactly the outcome a sequential run_tuning would produce on the same
// per-configuration results.
#pragma once

#include <chrono>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "ktb/backend.hpp"
#include "ktb/kernel.hpp"
#include "ktb/search.hpp"

namespace ktb {

VerificationReport verify_outputs(const std::vector<Buffer>& candidate,
                                  const std::vector<Buffer>& reference, double rel_tol = 1e-4,
                                  double abs_tol = 1e-6);

enum class Verification { skipped, pass, fail };
const char* to_string(Verification v);

struct TuningRow {
    size_t step = 0;
    Configuration config;
    Status status = Status::missing;
    std::optional<double> time_ms;
    ResolvedSizes sizes;
    Verification verification = Verification::skipped;
    std::optional<double> best_so_far;
    std::string message;
    // B200 additions
    std::optional<VerificationReport> report;  // device verification details
    uint64_t space_index = 0;                  // enumeration index (sharded runs)
    int device = -1;                           // ordinal that evaluated the row
};

struct TuningJob {
    KernelSpec kernel;
    SearchSpace space;
    DeviceModel device;
    StrategySpec strategy;
    uint64_t seed = 1;
    int repetitions = 1;
    bool verify = false;
    double rel_tol = 1e-4;
    double abs_tol = 1e-6;
    // Host reference outputs (CLTune SetReference).  Built-in families on a
    // CudaBackend verify against their device reference instead.
    std::function<std::vector<Buffer>()> reference;
};

struct TuningOutcome {
    std::vector<TuningRow> rows;
    std::optional<size_t> best_index;
    std::optional<Configuration> best_config;
    std::optional<double> best_time_ms;
    size_t budget = 0;
    size_t unique_evaluations = 0;
    size_t failed_evaluations = 0;
    size_t total_steps = 0;
    unsigned long long space_size = 0;
    std::string kernel_name, device_name, backend_name;
    StrategySpec strategy;
    uint64_t seed = 0;
    std::chrono::system_clock::time_point started_at, finished_at;
    const TuningRow* best_row() const { return best_index ? &rows[*best_index] : nullptr; }
};

SearchSpace compose_space(const KernelSpec& kernel, const DeviceModel& device,
                          const SearchSpace& user_space);

TuningOutcome run_tuning(const TuningJob& job, Backend& backend, const SearchSpace& effective);
TuningOutcome run_tuning(const TuningJob& job, Backend& backend);

// Full / random search sharded over `backends` (one host thread each, a
// dynamic chunk queue over the unit list, NVRTC compiles prefetched into the
// shared pool).  `subset`, when non-empty, replaces the unit list with those
// enumeration indices (fixed throughput samples).  Other strategies (and a
// single backend) fall back to run_tuning on backends[0].
// Checkpoint of a long search: a replay table (`config,time_ms`, the format
// of ReplayBackend) that already-evaluated successful configurations are
// served from and new successful rows are appended to as they complete, so
// an interrupted full search resumes where it stopped.
//
// The checkpoint is bound to the job that wrote it: `<path>.job` holds
// job_signature(job) (kernel, source, argument recipes and problem scalars,
// launch geometry, device, repetitions, verification rule).  Resuming with a
// different job (e.g. GEMM 4096^3 on a 2048^3 checkpoint -- identical
// configuration keys) throws instead of serving the other problem's times.
std::string job_signature(const TuningJob& job);

class ResultLog {
  public:
    explicit ResultLog(const std::string& path, const std::string& signature = "");
    bool lookup(const std::string& key, double* time_ms) const;
    void append(const std::string& key, double time_ms);
    size_t known() const { return table_.size(); }

  private:
    std::map<std::string, double> table_;
    std::string path_;
    std::mutex mu_;
};

TuningOutcome run_tuning_sharded(const TuningJob& job, const std::vector<Backend*>& backends,
                                 const SearchSpace& effective,
                                 const std::vector<uint64_t>& subset = {},
                                 ResultLog* log = nullptr);

// Row bookkeeping shared by both drivers: turns a backend result into a row
// (applying the verification rule of tuner.hpp:256-289) and returns the
// time the search sees (nullopt = failed evaluation).
std::optional<double> finish_row(const TuningJob& job, EvaluationResult& result, TuningRow& row,
                                 const std::vector<Buffer>* reference,
                                 const std::vector<std::string>* reference_digests);

// RFC 4180 results CSV (CRLF), byte-compatible with write_results_csv.
void write_results_csv(std::ostream& out, const TuningOutcome& outcome);
std::string format_double(double v);
// One RFC 4180 record (fields quoted when needed, CRLF), as every report uses.
void write_csv_row(std::ostream& out, const std::vector<std::string>& fields);

}  // namespace ktb
