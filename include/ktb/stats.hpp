// Repeated-search statistics: the K-run methodology of the paper's violin
// plots, as the reference's `ktune stats` command runs it
// (tools/ktune.cpp:120-258, include/ktune/stats.hpp, report.hpp:80-112).
//
// Stochastic strategies (random, annealing, PSO) are repeated with seeds
// base_seed + run; each run's best time is one sample.  On several GPUs the
// runs are REPLICAS -- whole independent searches, one device each, handed
// out from a shared run counter: annealing and PSO chains do
// not shard, but K of them do.  Summary and density are computed over the
// samples in run order, so the reports do not depend on the device count.
#pragma once

#include <cstdint>
#include <optional>
#include <ostream>
#include <string>
#include <vector>

#include "ktb/backend.hpp"
#include "ktb/tuner.hpp"

namespace ktb {

struct Summary {
    size_t count = 0;
    double mean = 0.0;
    double stddev = 0.0;  // sample (n-1) deviation; 0 for one value
    double min = 0.0;
    double max = 0.0;
};

// Throws Error on an empty sample (stats.hpp:25-27).
Summary summarize(const std::vector<double>& values);

// Gaussian KDE on an even grid over [min, max], Silverman bandwidth
// 0.9*min(sd, iqr/1.34)*n^-1/5 (either spread alone when the other is 0;
// fixed 0.25 over [min-1, max+1] when both are), renormalized to unit
// trapezoid integral (stats.hpp:64-137).
struct Kde {
    std::vector<double> x, y;
    double bandwidth = 0.0;
};
Kde kde(const std::vector<double>& samples, size_t points = 256);

struct ExperimentStats {
    std::vector<double> values;
    Summary summary;
    Kde density;
};
ExperimentStats make_experiment_stats(std::vector<double> values, size_t points = 256);

struct RunSummary {
    size_t run = 0;
    uint64_t seed = 0;
    double best_time_ms = 0.0;
    std::string best_config;
};

struct StatsOutcome {
    std::vector<RunSummary> runs;
    ExperimentStats best_of_run;
    // Distribution over the whole effective space (one full sweep, sharded
    // over every backend); absent when the space exceeds kSpaceSweepLimit or
    // nothing in it succeeded.
    std::optional<ExperimentStats> space;
    bool space_skipped_for_size = false;
};

// ktune.cpp:118 -- the largest space that still gets the full-space violin.
constexpr unsigned long long kSpaceSweepLimit = 100000;

// `runs` searches with seeds base_seed..base_seed+runs-1, run r on whichever
// backend frees first (one worker per backend).  A run with no successful
// configuration is an error (ktune.cpp:145-151).
StatsOutcome run_stats(const TuningJob& job, const std::vector<Backend*>& backends,
                       const SearchSpace& effective, size_t runs, uint64_t base_seed,
                       bool space_sweep = true);

// Two-column "statistic,value" block, then "density_x,density_y" and the
// grid (report.hpp:98-112); runs CSV "run,seed,best_time_ms,best_config"
// (report.hpp:87-96).  RFC 4180, CRLF.
void write_stats_csv(std::ostream& out, const ExperimentStats& stats);
void write_runs_csv(std::ostream& out, const std::vector<RunSummary>& runs);

// stats.csv -> stats_runs.csv (ktune.cpp:63-69).
std::string derive_report_path(const std::string& path, const std::string& suffix);

}  // namespace ktb
