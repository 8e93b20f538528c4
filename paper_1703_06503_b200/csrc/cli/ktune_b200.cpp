// ktune-b200 -- the reference's `ktune` command line (proj/tools/ktune.cpp)
// over libktc, with the job's backend running on B200s.
//
//   ktune-b200 tune <job.json> [--out results.csv] [--seed N] [--gpus N | --devices 0,2]
//   ktune-b200 stats <job.json> --runs K [--base-seed N] [--out stats.csv]
//                    [--parallel P] [--gpus N | --devices ...]
//   ktune-b200 enumerate <job.json> [--list]
//
// Same subcommands, options, report files, stdout lines and exit codes as
// the reference (0 ok, 1 error, 2 empty space; ktune.cpp:284-298).  Added:
// --gpus N / --devices L choose the GPUs of a "cuda" backend (SURVEY 8(f)
// #1).  `tune` shards full and random searches over them (enumeration units,
// merged as one sequential run would be); `stats` runs its K searches as
// replicas, one whole search per GPU at a time.  For "replay" backends the
// same options (and --parallel) set the number of host workers.
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "ktc.h"

namespace {

struct Failure {
    int code;
    std::string message;
};

void check(int st, const void* handle = nullptr) {
    if (st == KTC_OK) return;
    const char* msg = ktc_last_error(handle);
    throw Failure{st == KTC_ERR_EMPTY_SPACE ? 2 : 1, msg ? msg : "unknown error"};
}

// Shortest round-trip decimal, as the reports print doubles.
std::string fmt(double v) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, r.ptr);
}

std::string join_sizes(const size_t* s, int n) {
    std::string o;
    for (int i = 0; i < n; ++i) o += (i ? "x" : "") + std::to_string(s[i]);
    return o;
}

struct Args {
    std::string cmd, job, out;
    bool has_seed = false, list = false, has_out = false;
    uint64_t seed = 0, base_seed = 1;
    size_t runs = 0, parallel = 1;
    std::vector<int> devices;
};

[[noreturn]] void usage(const std::string& why) {
    throw Failure{1, why + "\nusage: ktune-b200 {tune|stats|enumerate} <job.json> [options]"};
}

uint64_t number(const std::string& opt, const char* v) {
    uint64_t x = 0;
    const char* end = v + std::strlen(v);
    auto r = std::from_chars(v, end, x);
    if (r.ec != std::errc() || r.ptr != end) usage(opt + ": not a non-negative integer: " + v);
    return x;
}

Args parse(int argc, char** argv) {
    if (argc < 2) usage("a subcommand is required");
    Args a;
    a.cmd = argv[1];
    if (a.cmd != "tune" && a.cmd != "stats" && a.cmd != "enumerate")
        usage("unknown subcommand: " + a.cmd);
    for (int i = 2; i < argc; ++i) {
        const std::string o = argv[i];
        auto value = [&]() -> const char* {
            if (i + 1 >= argc) usage(o + " needs a value");
            return argv[++i];
        };
        if (o == "--out" && a.cmd != "enumerate") {
            a.out = value();
            a.has_out = true;
        } else if (o == "--seed" && a.cmd == "tune") {
            a.seed = number(o, value());
            a.has_seed = true;
        } else if (o == "--runs" && a.cmd == "stats") {
            a.runs = number(o, value());
        } else if (o == "--base-seed" && a.cmd == "stats") {
            a.base_seed = number(o, value());
        } else if (o == "--parallel" && a.cmd == "stats") {
            a.parallel = number(o, value());
            if (a.parallel == 0) usage("--parallel must be positive");
        } else if (o == "--gpus" && a.cmd != "enumerate") {
            const uint64_t n = number(o, value());
            if (n == 0 || n > 64) usage("--gpus must be in 1..64");
            a.devices.clear();
            for (uint64_t d = 0; d < n; ++d) a.devices.push_back(int(d));
        } else if (o == "--devices" && a.cmd != "enumerate") {
            a.devices.clear();
            std::stringstream ss(value());
            for (std::string tok; std::getline(ss, tok, ',');)
                a.devices.push_back(int(number(o, tok.c_str())));
            if (a.devices.empty()) usage("--devices needs at least one ordinal");
        } else if (o == "--list" && a.cmd == "enumerate") {
            a.list = true;
        } else if (!o.empty() && o[0] == '-') {
            usage("unknown option for " + a.cmd + ": " + o);
        } else if (a.job.empty()) {
            a.job = o;
        } else {
            usage("unexpected argument: " + o);
        }
    }
    if (a.job.empty()) usage("the job file is required");
    if (a.cmd == "stats" && a.runs == 0) usage("--runs is required and must be positive");
    return a;
}

struct Tuner {
    ktc_tuner* h = nullptr;
    explicit Tuner(const std::string& path) {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Failure{1, "cannot open \"" + path + "\""};
        std::ostringstream text;
        text << in.rdbuf();
        check(ktc_tuner_create(&h));
        const std::string base = std::filesystem::path(path).parent_path().string();
        check(ktc_tuner_load_job(h, text.str().c_str(), base.c_str()), h);
    }
    ~Tuner() { ktc_tuner_destroy(h); }
    ktc_job_info info() const {
        ktc_job_info i;
        check(ktc_tuner_job_info(h, &i), h);
        return i;
    }
    void set_devices(const std::vector<int>& d) {
        if (!d.empty()) check(ktc_tuner_set_devices(h, d.data(), int(d.size())), h);
    }
};

int cmd_tune(const Args& a) {
    Tuner t(a.job);
    if (a.has_seed) check(ktc_tuner_set_seed(t.h, a.seed), t.h);
    t.set_devices(a.devices);
    const std::string out = a.has_out ? a.out : std::string(t.info().output);
    ktc_job_info pre = t.info();
    std::fprintf(stderr, "ktune: info: tuning kernel \"%s\" on %s via %s (%d worker%s)\n",
                 pre.kernel, pre.device, pre.backend, pre.ndevices, pre.ndevices == 1 ? "" : "s");
    check(ktc_tuner_tune(t.h), t.h);
    check(ktc_tuner_write_csv(t.h, out.c_str()), t.h);
    ktc_summary s;
    check(ktc_tuner_summary(t.h, &s), t.h);
    const ktc_job_info inf = t.info();
    std::cout << "kernel: " << inf.kernel << " on " << inf.device << " via " << inf.backend << "\n";
    std::cout << "space: " << s.space_size << " valid configurations\n";
    std::cout << "budget: " << s.budget << " unique evaluations (" << s.unique_evaluations
              << " used, " << s.failed_evaluations << " failed)\n";
    if (s.best_index >= 0) {
        ktc_row r;
        char cfg[1024], msg[512];
        check(ktc_tuner_row(t.h, size_t(s.best_index), &r, cfg, sizeof(cfg), msg, sizeof(msg)),
              t.h);
        std::cout << "best: " << cfg << "\n";
        std::cout << "best time_ms: " << fmt(r.time_ms) << " (step " << r.step << ", global "
                  << join_sizes(r.global, r.ndim) << ", local " << join_sizes(r.local, r.ndim)
                  << ")\n";
    } else {
        std::cout << "best: none (no configuration succeeded)\n";
    }
    std::cout << "throughput: " << fmt(s.configs_per_s) << " configurations/s on "
              << inf.ndevices << (inf.is_cuda ? " GPU" : " worker")
              << (inf.ndevices == 1 ? "" : "s") << "\n";
    std::cout << "wrote " << out << "\n";
    return 0;
}

int cmd_stats(const Args& a) {
    Tuner t(a.job);
    std::vector<int> devs = a.devices;
    const ktc_job_info pre = t.info();
    if (!pre.is_cuda && devs.empty() && a.parallel > 1)
        for (size_t i = 0; i < a.parallel; ++i) devs.push_back(int(i));
    if (pre.is_cuda && a.parallel > 1 && a.devices.empty())
        std::fprintf(stderr, "ktune: warn: --parallel has no effect on the cuda backend; "
                             "use --gpus N (one replica per GPU)\n");
    t.set_devices(devs);
    const std::string out = a.has_out ? a.out : "stats.csv";
    ktc_stats_summary s;
    check(ktc_tuner_stats(t.h, a.runs, a.base_seed, out.c_str(), &s), t.h);
    const std::filesystem::path p(out);
    auto derived = [&](const char* suffix) {
        std::filesystem::path name = p.stem();
        name += suffix;
        name += p.extension();
        return (p.parent_path() / name).string();
    };
    std::cout << "runs: " << a.runs << " (seeds " << a.base_seed << ".."
              << a.base_seed + a.runs - 1 << ")\n";
    std::cout << "best-of-run: mean=" << fmt(s.mean) << " std=" << fmt(s.stddev)
              << " min=" << fmt(s.min) << " max=" << fmt(s.max) << "\n";
    std::cout << "wrote " << out << "\n";
    std::cout << "wrote " << derived("_runs") << "\n";
    unsigned long long raw = 0, constrained = 0, valid = 0;
    check(ktc_tuner_space_counts(t.h, &raw, &constrained, &valid), t.h);
    if (s.space_written)
        std::cout << "wrote " << derived("_space") << "\n";
    else if (valid > 100000)
        std::cout << "space distribution: skipped (" << valid
                  << " configurations exceed 100000)\n";
    else
        std::cout << "space distribution: skipped (no successful evaluations)\n";
    return 0;
}

int cmd_enumerate(const Args& a) {
    Tuner t(a.job);
    unsigned long long raw = 0, constrained = 0, valid = 0;
    check(ktc_tuner_space_counts(t.h, &raw, &constrained, &valid), t.h);
    std::cout << "raw: " << raw << "\n";
    std::cout << "constrained: " << constrained << "\n";
    std::cout << "device-rejected: " << constrained - valid << "\n";
    std::cout << "valid: " << valid << "\n";
    if (a.list) {
        char cfg[1024];
        for (unsigned long long i = 0; i < valid; ++i) {
            check(ktc_tuner_space_config(t.h, i, cfg, sizeof(cfg)), t.h);
            std::cout << cfg << "\n";
        }
    }
    return valid == 0 ? 2 : 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Args a = parse(argc, argv);
        if (a.cmd == "tune") return cmd_tune(a);
        if (a.cmd == "stats") return cmd_stats(a);
        return cmd_enumerate(a);
    } catch (const Failure& f) {
        std::fprintf(stderr, "ktune: error: %s\n", f.message.c_str());
        return f.code;
    }
}
