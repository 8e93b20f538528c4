// ktb/backend.hpp -- the evaluation boundary (reference backend.hpp:21-80)
// and its implementations:
//   CudaBackend    NVRTC + CUDA driver on one B200, via libktc's C ABI
//   ReplayBackend  recorded `config,time_ms` tables (backend.hpp:485-592)
#pragma once

#include <istream>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "ktb/arguments.hpp"
#include "ktb/config.hpp"
#include "ktc.h"

namespace ktb {

enum class Status { success, compile_error, runtime_error, missing };
const char* to_string(Status s);
Status status_from(const std::string& name);

// Field-for-field ktune::VerificationReport (tuner.hpp:30-37).
struct VerificationReport {
    bool pass = true;
    double max_abs_error = 0.0;
    double max_rel_error = 0.0;
    size_t buffer_index = 0;
    size_t element_index = 0;
    size_t elements_compared = 0;
};

struct EvaluationRequest {
    std::string kernel_name;
    std::string source_ref;
    Configuration config;
    std::vector<size_t> global;
    std::vector<size_t> local;
    std::vector<ArgumentSpec> arguments;
    std::string device_name;
    int repetitions = 1;
    bool want_outputs = false;
};

struct EvaluationResult {
    Status status = Status::missing;
    double time_ms = 0.0;
    std::vector<std::string> output_digests;
    std::vector<Buffer> outputs;
    std::string message;
    // Additive over ktune: set by backends that verify on the device; the
    // tuner consumes it before the outputs / digest paths.
    std::optional<VerificationReport> device_verification;
    bool ok() const { return status == Status::success; }
};

class Backend {
  public:
    virtual ~Backend() = default;
    virtual EvaluationResult evaluate(const EvaluationRequest& request) = 0;
    virtual bool concurrency_safe() const { return false; }
    virtual std::string name() const = 0;
    // Hint: `request` will be evaluated soon (compile ahead).  Optional.
    virtual void prefetch(const EvaluationRequest&) {}
    // How many requests ahead prefetch() is worth calling (0 = no preference).
    virtual size_t prefetch_depth() const { return 0; }
    // Device ordinal behind this backend, -1 if none.
    virtual int device() const { return -1; }
    // A new search starts on this backend (drops per-search state such as
    // the prune_factor bar).  Called by run_tuning / run_tuning_sharded.
    virtual void begin_search() {}
    // CLTune SetReference: binds host reference outputs so the backend can
    // verify on its own (device-side).  Returns false when unsupported, in
    // which case the tuner verifies returned outputs on the host.
    virtual bool bind_reference(const EvaluationRequest&, const std::vector<Buffer>&) {
        return false;
    }
};

class ReplayBackend : public Backend {
  public:
    explicit ReplayBackend(std::map<std::string, double> table) : table_(std::move(table)) {}
    static ReplayBackend load(const std::string& path);
    static ReplayBackend parse(std::istream& in);
    static void save(const std::string& path, const std::map<std::string, double>& table);
    std::string name() const override { return "replay"; }
    bool concurrency_safe() const override { return true; }
    EvaluationResult evaluate(const EvaluationRequest& r) override;
    const std::map<std::string, double>& table() const { return table_; }

  private:
    std::map<std::string, double> table_;
};

// One B200 (one CUDA context).  evaluate() compiles the configuration with
// NVRTC for sm_100a, launches it with the request's geometry, times it with
// CUDA events (best of `repetitions`, L2 flushed before each) and verifies
// the output on the device against the family's device reference.  Not
// concurrency-safe by itself: give each thread its own CudaBackend.
class CudaBackend : public Backend {
  public:
    explicit CudaBackend(int ordinal, const ktc_backend_options* opts = nullptr);
    ~CudaBackend() override;
    CudaBackend(const CudaBackend&) = delete;
    CudaBackend& operator=(const CudaBackend&) = delete;

    EvaluationResult evaluate(const EvaluationRequest& r) override;
    void prefetch(const EvaluationRequest& r) override;
    size_t prefetch_depth() const override;
    std::string name() const override;
    int device() const override { return ordinal_; }
    void begin_search() override { ktc_backend_begin_search(be_); }
    bool bind_reference(const EvaluationRequest& r, const std::vector<Buffer>& outputs) override;
    ktc_backend* handle() { return be_; }
    // Accounting of the last evaluate() and running totals.
    const ktc_result& last_result() const { return last_; }
    struct Totals {
        double compile_ms = 0, load_ms = 0, run_ms = 0, verify_ms = 0;
        size_t evaluations = 0, cache_hits = 0, launches = 0;
    };
    const Totals& totals() const { return totals_; }
    void reset_totals() { totals_ = Totals{}; }

  private:
    int ordinal_;
    ktc_backend* be_ = nullptr;
    ktc_result last_{};
    Totals totals_{};
};

}  // namespace ktb
