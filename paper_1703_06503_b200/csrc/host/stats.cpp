// Repeated-search statistics (reference: include/ktune/stats.hpp,
// report.hpp:80-112, tools/ktune.cpp:120-258).  The arithmetic follows the
// reference operation for operation (same summation orders, same grid, same
// renormalization) so the reports are byte-identical on the same samples.
#include "ktb/stats.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <exception>
#include <filesystem>
#include <thread>

#include "ktb/errors.hpp"

namespace ktb {

Summary summarize(const std::vector<double>& values) {
    if (values.empty()) throw Error("cannot summarize an empty sample");
    Summary s;
    s.count = values.size();
    s.min = s.max = values.front();
    double sum = 0.0;
    for (double v : values) {
        sum += v;
        s.min = std::min(s.min, v);
        s.max = std::max(s.max, v);
    }
    s.mean = sum / double(values.size());
    if (values.size() > 1) {
        double sq = 0.0;
        for (double v : values) sq += (v - s.mean) * (v - s.mean);
        s.stddev = std::sqrt(sq / double(values.size() - 1));
    }
    return s;
}

namespace {

// Type-7 (linear interpolation) quantile of a sorted sample.
double quantile7(const std::vector<double>& sorted, double p) {
    const double pos = p * double(sorted.size() - 1);
    const size_t lo = size_t(pos);
    const size_t hi = std::min(lo + 1, sorted.size() - 1);
    const double w = pos - double(lo);
    return sorted[lo] * (1.0 - w) + sorted[hi] * w;
}

}  // namespace

Kde kde(const std::vector<double>& samples, size_t points) {
    if (samples.empty()) throw Error("cannot estimate a density from an empty sample");
    if (points < 2) throw Error("a density grid needs at least two points");
    std::vector<double> sorted(samples);
    std::sort(sorted.begin(), sorted.end());
    const double n = double(sorted.size());
    const Summary sum = summarize(samples);
    const double iqr = quantile7(sorted, 0.75) - quantile7(sorted, 0.25);
    double spread = 0.0;
    if (sum.stddev > 0.0 && iqr > 0.0) spread = std::min(sum.stddev, iqr / 1.34);
    else if (sum.stddev > 0.0) spread = sum.stddev;
    else if (iqr > 0.0) spread = iqr / 1.34;

    Kde k;
    double left = sorted.front(), right = sorted.back();
    if (spread > 0.0) {
        k.bandwidth = 0.9 * spread * std::pow(n, -0.2);
    } else {
        k.bandwidth = 0.25;
        left -= 1.0;
        right += 1.0;
    }
    const double dx = (right - left) / double(points - 1);
    const double norm = 1.0 / (n * k.bandwidth * std::sqrt(2.0 * 3.14159265358979323846));
    k.x.resize(points);
    k.y.resize(points);
    for (size_t i = 0; i < points; ++i) {
        const double xi = left + dx * double(i);
        double acc = 0.0;
        for (double s : sorted) {
            const double z = (xi - s) / k.bandwidth;
            acc += std::exp(-0.5 * z * z);
        }
        k.x[i] = xi;
        k.y[i] = acc * norm;
    }
    double area = 0.0;
    for (size_t i = 0; i + 1 < points; ++i) area += 0.5 * (k.y[i] + k.y[i + 1]) * dx;
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
