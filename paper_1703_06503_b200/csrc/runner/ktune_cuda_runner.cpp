// ktune-cuda-runner -- the reference's external-runner protocol on a B200.
//
// The reference's ExternalBackend (proj/include/ktune/external.hpp:185-437)
// spawns one process per evaluation, writes one JSON request on stdin
// (external.hpp:25-55) and reads one JSON reply from stdout
// (external.hpp:57-156).  This binary answers that protocol by evaluating
// the request on the GPU through libktc (ktc_backend_evaluate): NVRTC
// compile for sm_100a (cached on disk in $KTC_CACHE_DIR, default
// ~/.cache/ktc), best-of-N CUDA-event timing, device verification against
// the bit-exact device reference.  With want_outputs the reply carries
// `outputs_digest`: the reference output's digest when the device verdict is
// "pass", a non-matching marker otherwise -- the reference tuner's digest
// comparison (tuner.hpp:271-279) then records the device verdict.
//
//   "backend": {"kind": "external", "argv": [".../ktune-cuda-runner"], "timeout_ms": 120000}
//
// Compatibility path, not the throughput path (one process and one CUDA
// context per evaluation).
#include <cstdlib>
#include <iostream>
#include <iterator>
#include <json.hpp>
#include <string>
#include <vector>

#include "ktc.h"

using Json = nlohmann::json;

namespace {

void reply_error(const std::string& status, const std::string& message) {
    std::cout << Json{{"status", status}, {"message", message}}.dump() << std::endl;
}

int role_of(const std::string& r) {
    if (r == "input") return KTC_ARG_INPUT;
    if (r == "output") return KTC_ARG_OUTPUT;
    if (r == "scalar") return KTC_ARG_SCALAR;
    throw std::runtime_error("unknown argument role \"" + r + "\"");
}

}  // namespace

int main() {
    std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
    Json req;
    try {
        req = Json::parse(text);
    } catch (const std::exception& e) {
        reply_error("runtime_error", std::string("unparsable request: ") + e.what());
        return 0;
    }
    try {
        const std::string kernel = req.at("kernel").get<std::string>();
        const std::string source_ref = req.value("source_ref", std::string());
        std::vector<std::string> names;
        std::vector<long long> values;
        for (const auto& it : req.at("config").items()) {
            names.push_back(it.key());
            values.push_back(it.value().get<long long>());
        }
        std::vector<const char*> name_ptrs;
        for (const auto& n : names) name_ptrs.push_back(n.c_str());
        std::vector<std::string> fills;
        std::vector<ktc_arg> args;
        fills.reserve(req.at("args").size());
        for (const Json& a : req.at("args")) {
            ktc_arg c{};
            c.role = role_of(a.at("role").get<std::string>());
            c.type = a.at("type").get<std::string>() == "i32" ? KTC_I32 : KTC_F32;
            if (c.role == KTC_ARG_SCALAR) c.value = a.at("value").get<double>();
            else c.length = a.at("length").get<size_t>();
            fills.push_back(a.value("fill", std::string("none")));
            args.push_back(c);
        }
        for (size_t i = 0; i < args.size(); ++i) args[i].fill = fills[i].c_str();
        const std::vector<size_t> global = req.at("global").get<std::vector<size_t>>();
        const std::vector<size_t> local = req.at("local").get<std::vector<size_t>>();

        ktc_request r{};
        r.kernel_name = kernel.c_str();
        r.source_ref = source_ref.c_str();
        r.n_params = int(values.size());
        r.param_names = name_ptrs.data();
        r.param_values = values.data();
        r.ndim = int(std::min<size_t>(3, global.size()));
        for (int d = 0; d < r.ndim; ++d) {
            r.global[d] = global[size_t(d)];
            r.local[d] = size_t(d) < local.size() ? local[size_t(d)] : 1;
        }
        r.n_args = int(args.size());
        r.args = args.data();
        r.device_name = "B200";
        r.repetitions = req.value("repetitions", 1);
        r.want_outputs = req.value("want_outputs", false) ? 1 : 0;

        ktc_backend_options opts;
        ktc_backend_default_options(&opts);
        std::string cache;
        if (const char* c = std::getenv("KTC_CACHE_DIR")) cache = c;
        else if (const char* h = std::getenv("HOME")) cache = std::string(h) + "/.cache/ktc";
        opts.cache_dir = cache.empty() ? nullptr : cache.c_str();
        opts.compile_threads = 1;
        int device = 0;
        if (const char* d = std::getenv("KTC_DEVICE")) device = std::atoi(d);
        ktc_backend* be = nullptr;
        if (ktc_backend_open(device, &opts, &be) != KTC_OK) {
            reply_error("runtime_error", std::string("cuda: ") + ktc_last_error(nullptr));
            return 0;
        }
        ktc_result res;
        const int st = ktc_backend_evaluate(be, &r, &res);
        if (st != KTC_OK) {
            reply_error("runtime_error", std::string("cuda: ") + ktc_last_error(nullptr));
            ktc_backend_close(be);
            return 0;
        }
        Json out;
        out["status"] = ktc_status_name(res.status);
        if (res.message[0]) out["message"] = std::string(res.message);
        if (res.status == KTC_STATUS_SUCCESS) {
            out["time_ms"] = res.time_ms;
            if (r.want_outputs && res.verification != KTC_VERIFY_SKIPPED) {
                Json digests = Json::array();
                for (int k = 0; k < res.n_outputs; ++k) {
                    char hex[17] = {0};
                    if (res.verification == KTC_VERIFY_PASS &&
                        ktc_backend_read_reference(be, &r, k, nullptr, 0, hex) == KTC_OK)
                        digests.push_back(std::string(hex));
                    else
                        digests.push_back("device-verify-failed");
                }
                out["outputs_digest"] = digests;
            }
        }
        ktc_backend_close(be);
        std::cout << out.dump() << std::endl;
        return 0;
    } catch (const std::exception& e) {
        reply_error("runtime_error", std::string("malformed request: ") + e.what());
        return 0;
    }
}
