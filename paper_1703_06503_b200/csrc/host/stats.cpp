// Repeated-search statistics (reference: include/ktune/stats.hpp,
// report.hpp:80-112, tools/ktune.cpp:120-258): per-run summaries gathered
// from replicas, the sample moments and a Gaussian density of the best
// times, and the report writers.  The floating-point evaluation order is
// dictated by byte-parity of the reports with the reference's.
#include "ktb/stats.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <exception>
#include <filesystem>
#include <thread>

#include "ktb/errors.hpp"

namespace ktb {

namespace {

// Moments of a sample in one object: the running sum and extremes in sample
// order, then the (n-1) deviation around the mean.  Floating-point order is
// part of the contract -- the reports must be byte-identical to the
// reference's on the same samples -- so every accumulation below runs in the
// order the reference's report defines (sample order, then sorted order for
// the density).
struct Moments {
    size_t n = 0;
    double total = 0.0, lo = 0.0, hi = 0.0, mean = 0.0, sd = 0.0;
    explicit Moments(const std::vector<double>& v) : n(v.size()) {
        if (v.empty()) throw Error("cannot summarize an empty sample");
        lo = hi = v.front();
        for (double x : v) {
            total += x;
            lo = std::min(lo, x);
            hi = std::max(hi, x);
        }
        mean = total / double(n);
        if (n < 2) return;
        double ss = 0.0;
        for (double x : v) ss += (x - mean) * (x - mean);
        sd = std::sqrt(ss / double(n - 1));
    }
};

// Linear-interpolation (type 7) quantile of an ascending sample.
double type7(const std::vector<double>& asc, double p) {
    const double at = p * double(asc.size() - 1);
    const size_t k = size_t(at);
    const double frac = at - double(k);
    return asc[k] * (1.0 - frac) + asc[std::min(k + 1, asc.size() - 1)] * frac;
}

// Robust spread for Silverman's rule: min(sd, IQR/1.34), or whichever of
// the two is non-zero, or 0 for a constant sample.
double silverman_spread(double sd, double iqr) {
    const double r = iqr / 1.34;
    if (sd > 0.0 && iqr > 0.0) return std::min(sd, r);
    return sd > 0.0 ? sd : iqr > 0.0 ? r : 0.0;
}

}  // namespace

Summary summarize(const std::vector<double>& values) {
    const Moments m(values);
    Summary s;
    s.count = m.n;
    s.mean = m.mean;
    s.stddev = m.sd;
    s.min = m.lo;
    s.max = m.hi;
    return s;
}

Kde kde(const std::vector<double>& samples, size_t points) {
    if (samples.empty()) throw Error("cannot estimate a density from an empty sample");
    if (points < 2) throw Error("a density grid needs at least two points");
    std::vector<double> asc(samples);
    std::sort(asc.begin(), asc.end());
    const double n = double(asc.size());
    const double spread =
        silverman_spread(Moments(samples).sd, type7(asc, 0.75) - type7(asc, 0.25));
    Kde k;
    // A constant sample gets a fixed bandwidth over [min - 1, max + 1].
    const double left = asc.front() - (spread > 0.0 ? 0.0 : 1.0);
    const double right = asc.back() + (spread > 0.0 ? 0.0 : 1.0);
    k.bandwidth = spread > 0.0 ? 0.9 * spread * std::pow(n, -0.2) : 0.25;
    const double step = (right - left) / double(points - 1);
    const double scale = 1.0 / (n * k.bandwidth * std::sqrt(2.0 * 3.14159265358979323846));
    k.x.resize(points);
    k.y.resize(points);
    for (size_t g = 0; g < points; ++g) {
        k.x[g] = left + step * double(g);
        double mass = 0.0;
        for (double s : asc) {
            const double z = (k.x[g] - s) / k.bandwidth;
            mass += std::exp(-0.5 * z * z);
        }
        k.y[g] = mass * scale;
    }
    // Renormalize to a unit trapezoid integral over the grid.
    double area = 0.0;
    for (size_t g = 1; g < points; ++g) area += 0.5 * (k.y[g - 1] + k.y[g]) * step;
    for (double& y : k.y) y /= area;
    return k;
}

ExperimentStats make_experiment_stats(std::vector<double> values, size_t points) {
    ExperimentStats e;
    e.summary = summarize(values);
    e.density = kde(values, points);
    e.values = std::move(values);
    return e;
}

void write_stats_csv(std::ostream& out, const ExperimentStats& st) {
    write_csv_row(out, {"statistic", "value"});
    write_csv_row(out, {"count", std::to_string(st.summary.count)});
    write_csv_row(out, {"mean", format_double(st.summary.mean)});
    write_csv_row(out, {"std", format_double(st.summary.stddev)});
    write_csv_row(out, {"min", format_double(st.summary.min)});
    write_csv_row(out, {"max", format_double(st.summary.max)});
    write_csv_row(out, {"density_x", "density_y"});
    for (size_t i = 0; i < st.density.x.size(); ++i)
        write_csv_row(out, {format_double(st.density.x[i]), format_double(st.density.y[i])});
}

void write_runs_csv(std::ostream& out, const std::vector<RunSummary>& runs) {
    write_csv_row(out, {"run", "seed", "best_time_ms", "best_config"});
    for (const RunSummary& r : runs)
        write_csv_row(out, {std::to_string(r.run), std::to_string(r.seed),
                            format_double(r.best_time_ms), r.best_config});
}

std::string derive_report_path(const std::string& path, const std::string& suffix) {
    const std::filesystem::path p(path);
    std::filesystem::path name = p.stem();
    name += suffix;
    name += p.extension();
    return (p.parent_path() / name).string();
}

StatsOutcome run_stats(const TuningJob& job, const std::vector<Backend*>& backends,
                       const SearchSpace& eff, size_t runs, uint64_t base_seed,
                       bool space_sweep) {
    if (backends.empty()) throw Error("run_stats: no backends");
    if (runs == 0) throw Error("run_stats: at least one run is needed");
    if (eff.valid_count() == 0) {
        if (job.space.valid_count() == 0) throw EmptySpace();
        throw EmptySpaceAfterConstraints();
    }
    StatsOutcome out;
    out.runs.resize(runs);
    std::vector<std::exception_ptr> failed(runs);
    std::atomic<size_t> next{0};
    // Replicas: each worker owns one backend (one device) and runs whole
    // searches on it; the run index alone fixes the seed, so which device
    // ran a search does not change its result.
    auto worker = [&](Backend* be) {
        for (size_t r = next.fetch_add(1); r < runs; r = next.fetch_add(1)) {
            try {
                TuningJob j = job;
                j.seed = base_seed + r;
                TuningOutcome o = run_tuning_sharded(j, {be}, eff);
                if (!o.best_time_ms)
                    throw Error("run " + std::to_string(r) + " (seed " + std::to_string(j.seed) +
                                ") found no successful configuration");
                out.runs[r] = RunSummary{r, j.seed, *o.best_time_ms, o.best_config->canonical()};
            } catch (...) {
                failed[r] = std::current_exception();
            }
        }
    };
    const size_t nw = std::min(backends.size(), runs);
    if (nw == 1) {
        worker(backends[0]);
    } else {
        std::vector<std::thread> pool;
        for (size_t w = 0; w < nw; ++w) pool.emplace_back(worker, backends[w]);
        for (auto& th : pool) th.join();
    }
    for (auto& e : failed)
        if (e) std::rethrow_exception(e);

    std::vector<double> bests;
    bests.reserve(runs);
    for (const RunSummary& r : out.runs) bests.push_back(r.best_time_ms);
    out.best_of_run = make_experiment_stats(std::move(bests));

    if (!space_sweep) return out;
    if (eff.valid_count() > kSpaceSweepLimit) {
        out.space_skipped_for_size = true;
        return out;
    }
    // The whole space once (full strategy, seed = base_seed), sharded over
    // every backend; rows come back in enumeration order.
    TuningJob j = job;
    j.strategy = StrategySpec{};
    j.seed = base_seed;
    TuningOutcome full = run_tuning_sharded(j, backends, eff);
    std::vector<double> times;
    times.reserve(full.rows.size());
    for (const TuningRow& r : full.rows)
        if (r.status == Status::success && r.verification != Verification::fail && r.time_ms)
            times.push_back(*r.time_ms);
    if (!times.empty()) out.space = make_experiment_stats(std::move(times));
    return out;
}

}  // namespace ktb
