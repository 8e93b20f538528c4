// tuner.cpp -- run_tuning, the multi-device sharded executor, host output
// verification and the results CSV.
#include "ktb/tuner.hpp"

#include <atomic>
#include <charconv>
#include <cmath>
#include <fstream>
#include <mutex>
#include <iterator>
#include <ostream>
#include <sstream>
#include <thread>

#include "ktb/landscapes.hpp"

namespace ktc {
void trace_phase(const char* what, std::chrono::steady_clock::time_point since);
}

namespace ktb {

std::string format_double(double v) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, r.ptr);
}

const char* to_string(Verification v) {
    switch (v) {
        case Verification::skipped: return "";
        case Verification::pass: return "pass";
        case Verification::fail: return "fail";
    }
    return "?";
}

// Host verification (tuner.hpp:39-106); the device path is builtin.cu.
VerificationReport verify_outputs(const std::vector<Buffer>& cand, const std::vector<Buffer>& ref,
                                  double rel_tol, double abs_tol) {
    if (cand.size() != ref.size())
        throw ShapeMismatch("candidate has " + std::to_string(cand.size()) +
                            " output buffers, reference has " + std::to_string(ref.size()));
    VerificationReport rep;
    auto record = [&](size_t b, size_t e, double abs_err, double rel_err, bool ok) {
        if (!(abs_err <= rep.max_abs_error)) {
            rep.max_abs_error = abs_err;
            if (rep.pass) rep.buffer_index = b, rep.element_index = e;
        }
        if (!(rel_err <= rep.max_rel_error)) rep.max_rel_error = rel_err;
        if (!ok && rep.pass) rep.pass = false, rep.buffer_index = b, rep.element_index = e;
        ++rep.elements_compared;
    };
    for (size_t b = 0; b < cand.size(); ++b) {
        if (cand[b].index() != ref[b].index())
            throw ShapeMismatch("output buffer " + std::to_string(b) + " differs in element type");
        if (buffer_length(cand[b]) != buffer_length(ref[b]))
            throw ShapeMismatch("output buffer " + std::to_string(b) + " has length " +
                                std::to_string(buffer_length(cand[b])) + ", reference has " +
                                std::to_string(buffer_length(ref[b])));
        if (const auto* c = std::get_if<BufferF32>(&cand[b])) {
            const auto& r = std::get<BufferF32>(ref[b]);
            for (size_t i = 0; i < c->size(); ++i) {
                const double ae = std::abs(double((*c)[i]) - double(r[i]));
                const double mag = std::abs(double(r[i]));
                record(b, i, ae, mag > 0.0 ? ae / mag : 0.0, ae <= abs_tol + rel_tol * mag);
            }
        } else {
            const auto& c32 = std::get<BufferI32>(cand[b]);
            const auto& r32 = std::get<BufferI32>(ref[b]);
            for (size_t i = 0; i < c32.size(); ++i) {
                const double ae = std::abs(double(c32[i]) - double(r32[i]));
                record(b, i, ae, ae, c32[i] == r32[i]);
            }
        }
    }
    return rep;
}

SearchSpace compose_space(const KernelSpec& kernel, const DeviceModel& device,
                          const SearchSpace& user_space) {
    SearchSpace eff = user_space;
    eff.add_predicate(device_constraints(kernel, device, user_space));
    return eff;
}

namespace {

EvaluationRequest make_request(const TuningJob& job, const Configuration& c, ResolvedSizes* sizes) {
    *sizes = resolve_thread_sizes(job.kernel, c);
    EvaluationRequest r;
    r.kernel_name = job.kernel.name;
    r.source_ref = job.kernel.source_ref;
    r.config = c;
    r.global = sizes->global;
    r.local = sizes->local;
    r.arguments = job.kernel.arguments;
    r.device_name = job.device.name;
    r.repetitions = job.repetitions;
    r.want_outputs = job.verify;
    return r;
}

void check_nonempty(const TuningJob& job, const SearchSpace& eff) {
    if (job.verify && !job.reference && job.kernel.name != "conv" && job.kernel.name != "gemm" &&
        job.kernel.name != "gemm_tf32")
        throw Error("verification requested but the job has no reference");
    if (eff.valid_count() == 0) {
        if (job.space.valid_count() == 0) throw EmptySpace();
        throw EmptySpaceAfterConstraints();
    }
}

// Binds the job's host reference to a device backend once (custom kernels).
bool bind_host_reference(const TuningJob& job, Backend& be, const SearchSpace& eff,
                         std::vector<Buffer>* ref) {
    if (!job.verify || !job.reference) return false;
    if (ref->empty()) *ref = job.reference();
    ResolvedSizes s;
    EvaluationRequest proto = make_request(job, eff.config_at(0), &s);
    return be.bind_reference(proto, *ref);
}

void fill_header(TuningOutcome& o, const TuningJob& job, Backend& be, const SearchSpace& eff) {
    o.started_at = std::chrono::system_clock::now();
    o.kernel_name = job.kernel.name;
    o.device_name = job.device.name;
    o.backend_name = be.name();
    o.strategy = job.strategy;
    o.seed = job.seed;
    o.space_size = eff.valid_count();
}

}  // namespace

std::optional<double> finish_row(const TuningJob& job, EvaluationResult& res, TuningRow& row,
                                 const std::vector<Buffer>* reference,
                                 const std::vector<std::string>* reference_digests) {
    row.status = res.status;
    row.message = res.message;
    if (!res.ok()) return std::nullopt;
    row.time_ms = res.time_ms;
    if (job.verify) {
        if (res.device_verification) {
            const VerificationReport& rep = *res.device_verification;
            row.report = rep;
            row.verification = rep.pass ? Verification::pass : Verification::fail;
            if (!rep.pass)
                row.message = "verification failed: max abs error " +
                              format_double(rep.max_abs_error) + " at buffer " +
                              std::to_string(rep.buffer_index) + " element " +
                              std::to_string(rep.element_index);
        } else if (!res.outputs.empty() && reference && !reference->empty()) {
            VerificationReport rep =
                verify_outputs(res.outputs, *reference, job.rel_tol, job.abs_tol);
            row.report = rep;
            row.verification = rep.pass ? Verification::pass : Verification::fail;
            if (!rep.pass)
                row.message = "verification failed: max abs error " +
                              format_double(rep.max_abs_error) + " at buffer " +
                              std::to_string(rep.buffer_index) + " element " +
                              std::to_string(rep.element_index);
        } else if (!res.output_digests.empty() && reference_digests) {
            row.verification =
                res.output_digests == *reference_digests ? Verification::pass : Verification::fail;
            if (row.verification == Verification::fail)
                row.message = "verification failed: output digest mismatch";
        } else {
            row.verification = Verification::fail;
            row.message = "verification failed: the backend returned no outputs to compare";
        }
        if (row.verification == Verification::fail) return std::nullopt;
    }
    return *row.time_ms;
}

TuningOutcome run_tuning(const TuningJob& job, Backend& backend, const SearchSpace& eff) {
    check_nonempty(job, eff);
    backend.begin_search();
    TuningOutcome out;
    fill_header(out, job, backend, eff);
    std::vector<Buffer> reference;
    std::vector<std::string> digests;
    bool ready = false;
    const bool bound = bind_host_reference(job, backend, eff, &reference);
    auto ensure = [&]() {
        if (ready || !job.reference) return;
        if (reference.empty()) reference = job.reference();
        for (const Buffer& b : reference) digests.push_back(digest_hex(buffer_digest(b)));
        ready = true;
    };
    (void)bound;
    Evaluator ev = [&](const Configuration& c) -> std::optional<double> {
        TuningRow row;
        row.config = c;
        EvaluationRequest req = make_request(job, c, &row.sizes);
        row.device = backend.device();
        EvaluationResult res = backend.evaluate(req);
        if (job.verify && res.ok() && !res.device_verification) ensure();
        std::optional<double> t = finish_row(job, res, row, &reference, &digests);
        out.rows.push_back(std::move(row));
        return t;
    };
    Prefetcher pf = [&](const Configuration& c) {
        ResolvedSizes sz;
        backend.prefetch(make_request(job, c, &sz));
    };
    SearchOutcome s = run_search(eff, ev, job.strategy, job.seed, pf);
    for (size_t i = 0; i < out.rows.size(); ++i) {
        out.rows[i].step = s.trace[i].step;
        out.rows[i].best_so_far = s.trace[i].best_so_far;
    }
    out.best_config = s.best_config;
    out.best_time_ms = s.best_time_ms;
    out.budget = s.budget;
    out.unique_evaluations = s.unique_evaluations;
    out.failed_evaluations = s.failed_evaluations;
    out.total_steps = s.total_steps;
    if (out.best_config) {
        for (size_t i = 0; i < out.rows.size(); ++i) {
            const TuningRow& r = out.rows[i];
            if (r.status == Status::success && r.verification != Verification::fail &&
                r.config == *out.best_config) {
                out.best_index = i;
                break;
            }
        }
    }
    out.finished_at = std::chrono::system_clock::now();
    return out;
}

TuningOutcome run_tuning(const TuningJob& job, Backend& backend) {
    return run_tuning(job, backend, compose_space(job.kernel, job.device, job.space));
}

// ---------------------------------------------------------------------------
// Sharded executor.  Units (enumeration indices) are handed out in chunks
// from one atomic cursor; a second cursor keeps NVRTC compiles a window
// ahead of the slowest device.  Each unit's row lands at its unit position,
// so the merged outcome is a pure function of the per-unit results: the
// same rows, steps, running bests and best index as the sequential
// run_tuning on the same results (CachedEvaluator semantics: strict <,
// earliest wins, search.hpp:203-208).
// ---------------------------------------------------------------------------

std::string job_signature(const TuningJob& job) {
    std::ostringstream s;
    s.precision(17);
    const KernelSpec& k = job.kernel;
    s << "kernel=" << k.name << "\nsource=" << k.source_ref << "\nglobal=";
    for (size_t g : k.base_global) s << g << ' ';
    s << "\nlocal=";
    for (size_t l : k.base_local) s << l << ' ';
    s << "\nlocal_mem=" << k.local_mem_expr << "\nargs=";
    for (const ArgumentSpec& a : k.arguments)
        s << int(a.role) << ':' << int(a.type) << ':' << a.length << ':' << a.value << ':'
          << a.fill << ' ';
    s << "\ndevice=" << job.device.name << "\nrepetitions=" << job.repetitions
      << "\nverify=" << job.verify << ' ' << job.rel_tol << ' ' << job.abs_tol << "\n";
    return s.str();
}

ResultLog::ResultLog(const std::string& path, const std::string& signature) : path_(path) {
    const std::string sig_path = path + ".job";
    std::ifstream probe(path, std::ios::binary);
    if (probe) {
        table_ = ReplayBackend::load(path).table();
        if (!signature.empty() && !table_.empty()) {
            std::ifstream sf(sig_path, std::ios::binary);
            std::string recorded((std::istreambuf_iterator<char>(sf)),
                                 std::istreambuf_iterator<char>());
            if (recorded != signature)
                throw Error("checkpoint " + path + " was written by a different job (" +
                            (sf ? "signature mismatch in " + sig_path : "no " + sig_path) +
                            "); refusing to resume from it");
        }
    } else {
        ReplayBackend::save(path, {});  // header only
    }
    if (!signature.empty()) {
        std::ofstream sf(sig_path, std::ios::binary | std::ios::trunc);
        sf << signature;
    }
}

bool ResultLog::lookup(const std::string& key, double* t) const {
    auto it = table_.find(key);
    if (it == table_.end()) return false;
    *t = it->second;
    return true;
}

void ResultLog::append(const std::string& key, double t) {
    std::lock_guard<std::mutex> lk(mu_);
    if (!table_.emplace(key, t).second) return;
    std::ofstream out(path_, std::ios::binary | std::ios::app);
    out << key << ',' << format_double(t) << '\n';
}

TuningOutcome run_tuning_sharded(const TuningJob& job, const std::vector<Backend*>& backends,
                                 const SearchSpace& eff, const std::vector<uint64_t>& subset,
                                 ResultLog* log) {
    if (backends.empty()) throw Error("run_tuning_sharded: no backends");
    const bool ordered = job.strategy.kind == StrategyKind::full ||
                         job.strategy.kind == StrategyKind::random;
    // Order-dependent strategies (annealing, PSO) are sequential chains: one
    // device, speculative compile-ahead of their candidate moves.
    if (!ordered) return run_tuning(job, *backends[0], eff);
    // Above the enumeration limit there is no index table to shard: the
    // sequential run_tuning samples by rejection (space.hpp sample_unique's
    // large-space branch), as the reference does.
    if (subset.empty() && eff.raw_size() > SearchSpace::kEnumerationLimit)
        return run_tuning(job, *backends[0], eff);
    check_nonempty(job, eff);
    for (Backend* b : backends) b->begin_search();

    TuningOutcome out;
    fill_header(out, job, *backends[0], eff);
    std::vector<uint64_t> units = subset;
    size_t budget_n = 0;
    if (units.empty()) units = planned_indices(eff, job.strategy, job.seed, &budget_n);
    else budget_n = units.size();

    std::vector<Buffer> reference;
    std::vector<std::string> digests;
    if (job.verify && job.reference) {
        reference = job.reference();
        for (const Buffer& b : reference) digests.push_back(digest_hex(buffer_digest(b)));
        for (Backend* be : backends) bind_host_reference(job, *be, eff, &reference);
    }

    const size_t n = units.size();
    const auto t_start = std::chrono::steady_clock::now();
    std::vector<TuningRow> rows(n);
    std::vector<std::optional<double>> times(n);
    std::atomic<size_t> next{0}, prefetched{0};
    const size_t chunk = 4;
    // Deep enough that every compile-pool thread has a program in flight.
    size_t window = 64;
    for (Backend* be : backends) window = std::max(window, be->prefetch_depth());
    std::vector<std::string> errors(backends.size());

    auto worker = [&](size_t w) {
        Backend& be = *backends[w];
        try {
            for (;;) {
                const size_t i0 = next.fetch_add(chunk);
                if (i0 >= n) break;
                const size_t i1 = std::min(n, i0 + chunk);
                // Keep the compile pool `window` units ahead.
                for (size_t p = prefetched.load(); p < std::min(n, i1 + window);
                     p = prefetched.load()) {
                    if (!prefetched.compare_exchange_weak(p, p + 1)) continue;
                    ResolvedSizes s;
                    be.prefetch(make_request(job, eff.config_at(size_t(units[p])), &s));
                }
                for (size_t i = i0; i < i1; ++i) {
                    TuningRow& row = rows[i];
                    row.config = eff.config_at(size_t(units[i]));
                    row.space_index = units[i];
                    row.device = be.device();
                    EvaluationRequest req = make_request(job, row.config, &row.sizes);
                    double known = 0.0;
                    if (log && log->lookup(row.config.canonical(), &known)) {
                        // Checkpointed: only verified successes are logged.
                        row.status = Status::success;
                        row.time_ms = known;
                        row.verification = job.verify ? Verification::pass : Verification::skipped;
                        row.message = "resumed from checkpoint";
                        times[i] = known;
                        continue;
                    }
                    EvaluationResult res = be.evaluate(req);
                    if (i == 0) ktc::trace_phase("sharded: first unit", t_start);
                    times[i] = finish_row(job, res, row, &reference, &digests);
                    if (log && times[i]) log->append(row.config.canonical(), *times[i]);
                }
            }
        } catch (const std::exception& e) {
            errors[w] = e.what();
            next.store(n);  // stop the others
        }
    };
    std::vector<std::thread> pool;
    for (size_t w = 0; w < backends.size(); ++w) pool.emplace_back(worker, w);
    for (auto& t : pool) t.join();
    ktc::trace_phase("sharded: all units", t_start);
    for (const std::string& e : errors)
        if (!e.empty()) throw Error(e);

    // Merge in unit order.
    out.budget = budget_n;
    std::optional<double> best;
    for (size_t i = 0; i < n; ++i) {
        rows[i].step = i + 1;
        if (times[i]) {
            if (!best || *times[i] < *best) {
                best = times[i];
                out.best_config = rows[i].config;
                out.best_index = i;
            }
        } else {
            ++out.failed_evaluations;
        }
        rows[i].best_so_far = best;
    }
    out.best_time_ms = best;
    out.unique_evaluations = n;
    out.total_steps = n;
    out.rows = std::move(rows);
    out.finished_at = std::chrono::system_clock::now();
    return out;
}

// ---------------------------------------------------------------------------
// Results CSV (report.hpp:62-77): RFC 4180 quoting, CRLF rows, shortest
// round-trip doubles.
// ---------------------------------------------------------------------------

namespace {

std::string csv_field(const std::string& t) {
    if (t.find_first_of(",\"\r\n") == std::string::npos) return t;
    std::string o = "\"";
    for (char c : t) {
        if (c == '"') o += '"';
        o += c;
    }
    return o + "\"";
}

void csv_row(std::ostream& out, const std::vector<std::string>& f) {
    for (size_t i = 0; i < f.size(); ++i) {
        if (i) out << ',';
        out << csv_field(f[i]);
    }
    out << "\r\n";
}

std::string join_sizes(const std::vector<size_t>& s) {
    std::string o;
    for (size_t i = 0; i < s.size(); ++i) {
        if (i) o += 'x';
        o += std::to_string(s[i]);
    }
    return o;
}

}  // namespace

void write_csv_row(std::ostream& out, const std::vector<std::string>& fields) {
    csv_row(out, fields);
}

void write_results_csv(std::ostream& out, const TuningOutcome& o) {
    csv_row(out, {"step", "config", "status", "time_ms", "global", "local", "best_so_far",
                  "verified"});
    for (const TuningRow& r : o.rows)
        csv_row(out, {std::to_string(r.step), r.config.canonical(), to_string(r.status),
                      r.time_ms ? format_double(*r.time_ms) : "", join_sizes(r.sizes.global),
                      join_sizes(r.sizes.local), r.best_so_far ? format_double(*r.best_so_far) : "",
                      to_string(r.verification)});
}

}  // namespace ktb
