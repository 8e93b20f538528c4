// ref_tune_cuda.cpp -- the reference's OWN tuner driving the B200 backend.
//
// TEST INFRASTRUCTURE ONLY (drop-in proof).  Built by oracle/Makefile from
// the unmodified reference headers + include/ktune_cuda_backend.hpp, linked
// against libktc.so.  It is what `ktune tune job.json` does (ktune.cpp:85-115:
// load_job -> run_tuning -> write_results_csv), except that the job's backend
// is replaced by ktune::CudaBackend -- the one line a maintainer adds to
// parse_backend (jobfile.hpp:428-508) for `"kind": "cuda"`.
//
//   ref_tune_cuda <job.json> <results.csv> [host]
#include <fstream>
#include <iostream>
#include <sstream>

#include "ktune/jobfile.hpp"
#include "ktune/report.hpp"
#include "ktune/tuner.hpp"
#include "ktune_cuda_backend.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::cerr << "usage: ref_tune_cuda <job.json> <results.csv> [host]\n";
        return 2;
    }
    try {
        ktune::LoadedJob loaded = ktune::load_job(argv[1]);
        const bool host = argc > 3 && std::string(argv[3]) == "host";
        ktune::CudaBackend gpu(0, host ? ktune::CudaBackend::DigestMode::host_outputs
                                       : ktune::CudaBackend::DigestMode::device_verdict);
        ktune::TuningOutcome outcome = ktune::run_tuning(loaded.job, gpu);
        ktune::save_report(argv[2], [&](std::ostream& out) {
            ktune::write_results_csv(out, outcome);
        });
        std::cout << "rows " << outcome.rows.size() << " failed " << outcome.failed_evaluations
                  << " best " << (outcome.best_config ? outcome.best_config->canonical() : "-")
                  << " " << (outcome.best_time_ms ? *outcome.best_time_ms : 0.0) << " ms\n";
        return 0;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
