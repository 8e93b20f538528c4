// ktune_ref_capi.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// /root/reference/proj/include (read in place, never copied) into
// oracle/_ref/libktune_ref.so.  Used by tests/ (golden vectors, parity of the
// search layer), by bench.py's cpu_baseline leg and by `bench.py --impl
// reference` (the reference's own CPU tuner loop).  The product never loads
// it.
//
// Every function forwards to the reference's own code path:
//   kr_conv_reference   -> ktune::conv_reference      (landscapes.hpp:146)
//   kr_gemm_reference   -> ktune::gemm_reference      (landscapes.hpp:315)
//   kr_conv_apply       -> ktune::conv_apply          (landscapes.hpp:120)
//   kr_gemm_apply       -> ktune::gemm_apply          (landscapes.hpp:293)
//   kr_materialize_*    -> ktune::materialize_argument (arguments.hpp:126)
//   kr_digest_f32       -> ktune::buffer_digest        (arguments.hpp:184)
//   kr_verify_f32       -> ktune::verify_outputs       (tuner.hpp:39)
//   kr_job_*            -> ktune::parse_job + compose_space + run_tuning
//                          + write_results_csv         (jobfile.hpp:614,
//                          tuner.hpp:181/194, report.hpp:62)
//   kr_job_stats        -> the `ktune stats` sequence (tools/ktune.cpp:120-258:
//                          run_tuning per seed, make_experiment_stats,
//                          write_stats_csv / write_runs_csv); the CLI itself
//                          needs CLI11, which is absent, so its body is
//                          restated here over the same library calls
#include <atomic>
#include <chrono>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>

#include "ktune/jobfile.hpp"
#include "ktune/landscapes.hpp"
#include "ktune/report.hpp"
#include "ktune/stats.hpp"
#include "ktune/tuner.hpp"

namespace {

thread_local std::string g_error;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::exception& err) {
        g_error = err.what();
        return 1;
    }
}

void copy_out(const ktune::BufferF32& src, float* dst) {
    std::memcpy(dst, src.data(), src.size() * sizeof(float));
}

}  // namespace

extern "C" {

const char* kr_last_error() { return g_error.c_str(); }

int kr_materialize_f32(const char* fill, size_t length, float* out) {
    return guarded([&] {
        ktune::ArgumentSpec arg{ktune::ArgRole::input, ktune::ElementType::f32, length, 0.0,
                                fill};
        copy_out(std::get<ktune::BufferF32>(ktune::materialize_argument(arg)), out);
    });
}

int kr_materialize_i32(const char* fill, size_t length, int32_t* out) {
    return guarded([&] {
        ktune::ArgumentSpec arg{ktune::ArgRole::input, ktune::ElementType::i32, length, 0.0,
                                fill};
        auto buf = std::get<ktune::BufferI32>(ktune::materialize_argument(arg));
        std::memcpy(out, buf.data(), buf.size() * sizeof(int32_t));
    });
}

int kr_conv_reference(size_t x, size_t y, int filter, float weight, uint64_t seed, float* out) {
    return guarded([&] {
        ktune::ConvProblem p;
        p.x = x;
        p.y = y;
        p.filter = filter;
        p.weight = weight;
        p.seed = seed;
        copy_out(ktune::conv_reference(p), out);
    });
}

int kr_gemm_reference(size_t m, size_t n, size_t k, float alpha, float beta, uint64_t seed,
                      float* out) {
    return guarded([&] {
        ktune::GemmProblem p;
        p.m = m;
        p.n = n;
        p.k = k;
        p.alpha = alpha;
        p.beta = beta;
        p.seed = seed;
        copy_out(ktune::gemm_reference(p), out);
    });
}

int kr_conv_apply(const float* image, const float* taps, size_t x, size_t y, int f, float w,
                  float* out) {
    return guarded([&] {
        ktune::BufferF32 img(image, image + (x + f - 1) * (y + f - 1));
        ktune::BufferF32 tp(taps, taps + f * f);
        copy_out(ktune::conv_apply(img, tp, x, y, f, w), out);
    });
}

int kr_gemm_apply(const float* a, const float* b, const float* c, size_t m, size_t n, size_t k,
                  float alpha, float beta, float* out) {
    return guarded([&] {
        ktune::BufferF32 av(a, a + k * m), bv(b, b + k * n), cv(c, c + m * n);
        copy_out(ktune::gemm_apply(av, bv, cv, m, n, k, alpha, beta), out);
    });
}

uint64_t kr_digest_f32(const float* data, size_t n) {
    ktune::Buffer buf(ktune::BufferF32(data, data + n));
    return ktune::buffer_digest(buf);
}

// Report layout identical to ko_verify_report / ktc_verify_report.
struct kr_verify_report {
    int pass;
    double max_abs_error;
    double max_rel_error;
    size_t buffer_index;
    size_t element_index;
    size_t elements_compared;
};

int kr_verify_f32(const float* cand, const float* ref, size_t n, double rel_tol, double abs_tol,
                  kr_verify_report* out) {
    return guarded([&] {
        std::vector<ktune::Buffer> c{ktune::BufferF32(cand, cand + n)};
        std::vector<ktune::Buffer> r{ktune::BufferF32(ref, ref + n)};
        ktune::VerificationReport rep = ktune::verify_outputs(c, r, rel_tol, abs_tol);
        out->pass = rep.pass ? 1 : 0;
        out->max_abs_error = rep.max_abs_error;
        out->max_rel_error = rep.max_rel_error;
        out->buffer_index = rep.buffer_index;
        out->element_index = rep.element_index;
        out->elements_compared = rep.elements_compared;
    });
}

// ---------------------------------------------------------------------------
// Job-level entry points (the reference's own tuner on its own job format).
// ---------------------------------------------------------------------------

// Space funnel of a job: raw, constraint-only, valid after device limits.
int kr_job_counts(const char* job_json, unsigned long long* raw, unsigned long long* constrained,
                  unsigned long long* valid) {
    return guarded([&] {
        ktune::LoadedJob loaded = ktune::parse_job(std::string(job_json));
        ktune::SearchSpace eff =
            ktune::compose_space(loaded.job.kernel, loaded.job.device, loaded.job.space);
        *raw = eff.raw_size();
        *constrained = eff.constraint_only_count();
        *valid = eff.valid_count();
    });
}

// Writes the composed space's valid configurations, in enumeration order,
// one canonical string per line.
int kr_job_enumerate(const char* job_json, const char* out_path) {
    return guarded([&] {
        ktune::LoadedJob loaded = ktune::parse_job(std::string(job_json));
        ktune::SearchSpace eff =
            ktune::compose_space(loaded.job.kernel, loaded.job.device, loaded.job.space);
        std::ofstream out(out_path, std::ios::binary);
        for (const ktune::Configuration& c : eff.enumerate_valid()) out << c.canonical() << '\n';
    });
}

// Prices every valid configuration of the composed space with the job's own
// backend (e.g. synthetic) and saves a replay table (failures omitted, so
// they replay as `missing`).
int kr_job_price_table(const char* job_json, const char* out_path) {
    return guarded([&] {
        ktune::LoadedJob loaded = ktune::parse_job(std::string(job_json));
        ktune::SearchSpace eff =
            ktune::compose_space(loaded.job.kernel, loaded.job.device, loaded.job.space);
        std::map<std::string, double> table;
        for (const ktune::Configuration& c : eff.enumerate_valid()) {
            ktune::EvaluationRequest req;
            req.kernel_name = loaded.job.kernel.name;
            req.config = c;
            req.arguments = loaded.job.kernel.arguments;
            ktune::EvaluationResult res = loaded.backend->evaluate(req);
            if (res.ok()) table.emplace(c.canonical(), res.time_ms);
        }
        ktune::ReplayBackend::save(out_path, table);
    });
}

// Runs the job through the reference tuner and writes its results CSV.
// `base_dir` anchors relative replay paths.  Returns the best row index
// (-1 when nothing succeeded) through *best_index.
int kr_job_run(const char* job_json, const char* base_dir, const char* out_csv,
               long long* best_index, double* best_time_ms) {
    return guarded([&] {
        ktune::LoadedJob loaded =
            ktune::parse_job(std::string(job_json), std::filesystem::path(base_dir));
        ktune::TuningOutcome outcome = ktune::run_tuning(loaded.job, *loaded.backend);
        ktune::save_report(out_csv, [&](std::ostream& out) {
            ktune::write_results_csv(out, outcome);
        });
        *best_index = outcome.best_index ? static_cast<long long>(*outcome.best_index) : -1;
        *best_time_ms = outcome.best_time_ms ? *outcome.best_time_ms : 0.0;
    });
}

// `ktune stats <job> --runs R --base-seed S --out <out_csv>`, serial
// (tools/ktune.cpp:120-258).  Writes out_csv, <stem>_runs and, for spaces of
// at most 100,000 configurations, <stem>_space.
int kr_job_stats(const char* job_json, const char* base_dir, size_t runs, uint64_t base_seed,
                 const char* out_csv) {
    return guarded([&] {
        ktune::LoadedJob loaded =
            ktune::parse_job(std::string(job_json), std::filesystem::path(base_dir));
        ktune::SearchSpace effective =
            ktune::compose_space(loaded.job.kernel, loaded.job.device, loaded.job.space);
        if (effective.valid_count() == 0) throw ktune::EmptySpaceAfterConstraints();
        std::vector<ktune::RunSummary> summaries;
        std::vector<double> bests;
        for (size_t i = 0; i < runs; ++i) {
            ktune::TuningJob job = loaded.job;
            job.seed = base_seed + i;
            ktune::TuningOutcome o = ktune::run_tuning(job, *loaded.backend, effective);
            if (!o.best_time_ms) throw ktune::Error("run found no successful configuration");
            summaries.push_back({i, job.seed, *o.best_time_ms, o.best_config->canonical()});
            bests.push_back(*o.best_time_ms);
        }
        const std::filesystem::path out(out_csv);
        auto derived = [&](const char* suffix) {
            std::filesystem::path name = out.stem();
            name += suffix;
            name += out.extension();
            return (out.parent_path() / name).string();
        };
        ktune::ExperimentStats stats = ktune::make_experiment_stats(bests);
        ktune::save_report(out_csv, [&](std::ostream& o) { ktune::write_stats_csv(o, stats); });
        ktune::save_report(derived("_runs"),
                           [&](std::ostream& o) { ktune::write_runs_csv(o, summaries); });
        if (effective.valid_count() <= 100000) {
            ktune::TuningJob job = loaded.job;
            job.strategy = ktune::StrategySpec{};
            job.seed = base_seed;
            ktune::TuningOutcome o = ktune::run_tuning(job, *loaded.backend, effective);
            std::vector<double> times;
            for (const ktune::TuningRow& row : o.rows)
                if (row.status == ktune::Status::success &&
                    row.verification != ktune::Verification::fail && row.time_ms)
                    times.push_back(*row.time_ms);
            if (!times.empty()) {
                ktune::ExperimentStats space = ktune::make_experiment_stats(times);
                ktune::save_report(derived("_space"),
                                   [&](std::ostream& o) { ktune::write_stats_csv(o, space); });
            }
        }
    });
}

// The reference CPU tuner loop on a bounded sample: `threads` independent
// run_tuning() calls (seeds seed..seed+threads-1), each a random search of
// `per_thread` configurations over the job's composed space, with the job's
// own backend and verify flag (synthetic + verify=true prices every config
// with the CPU oracle, tuner.hpp:256-289).  Reports configurations per
// second of wall time.
int kr_job_throughput(const char* job_json, int threads, size_t per_thread, double* configs_per_s,
                      double* wall_s, size_t* evaluated) {
    return guarded([&] {
        ktune::LoadedJob proto = ktune::parse_job(std::string(job_json));
        ktune::SearchSpace eff =
            ktune::compose_space(proto.job.kernel, proto.job.device, proto.job.space);
        const double count = static_cast<double>(eff.valid_count());
        std::atomic<size_t> done{0};
        std::vector<std::string> errors(threads);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    ktune::LoadedJob loaded = ktune::parse_job(std::string(job_json));
                    loaded.job.strategy.kind = ktune::StrategyKind::random;
                    loaded.job.strategy.fraction = (static_cast<double>(per_thread) + 0.5) / count;
                    loaded.job.seed = proto.job.seed + static_cast<uint64_t>(t);
                    ktune::TuningOutcome out = ktune::run_tuning(loaded.job, *loaded.backend, eff);
                    done += out.rows.size();
                } catch (const std::exception& err) {
                    errors[t] = err.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        for (const auto& e : errors)
            if (!e.empty()) throw ktune::Error(e);
        *wall_s = std::chrono::duration<double>(t1 - t0).count();
        *evaluated = done.load();
        *configs_per_s = static_cast<double>(*evaluated) / *wall_s;
    });
}

}  // extern "C"
