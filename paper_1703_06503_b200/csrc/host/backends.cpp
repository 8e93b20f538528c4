// backends.cpp -- ktb::ReplayBackend and ktb::CudaBackend.
#include <cerrno>
#include <charconv>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string_view>

#include "ktb/backend.hpp"
#include "ktb/tuner.hpp"

namespace ktb {

const char* to_string(Status s) {
    switch (s) {
        case Status::success: return "ok";
        case Status::compile_error: return "compile_error";
        case Status::runtime_error: return "runtime_error";
        case Status::missing: return "missing";
    }
    return "?";
}

Status status_from(const std::string& n) {
    if (n == "ok") return Status::success;
    if (n == "compile_error") return Status::compile_error;
    if (n == "runtime_error") return Status::runtime_error;
    if (n == "missing") return Status::missing;
    throw Error("unknown status \"" + n + "\"");
}

// ---------------------------------------------------------------------------
// ReplayBackend (backend.hpp:485-592): `config,time_ms` tables keyed by
// canonical configuration strings; absent keys evaluate as `missing`.
// ---------------------------------------------------------------------------

ReplayBackend ReplayBackend::load(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error("cannot open replay file \"" + path + "\"");
    return parse(in);
}

namespace {

// One time field: the whole field must be a number (strtod syntax, as the
// reference's std::stod), finite-range, then strictly positive.
double replay_time(const std::string& field, size_t line) {
    errno = 0;
    char* end = nullptr;
    const double t = field.empty() ? 0.0 : std::strtod(field.c_str(), &end);
    if (field.empty() || end != field.c_str() + field.size() || errno == ERANGE)
        throw MalformedReplayFile(line, "unparsable time \"" + field + "\"");
    if (!(t > 0.0)) throw NonPositiveTime(t);
    return t;
}

}  // namespace

ReplayBackend ReplayBackend::parse(std::istream& in) {
    // Whole file in memory, then one pass over its lines (LF or CRLF).
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::map<std::string, double> table;
    size_t pos = 0, line = 0;
    bool have_header = false;
    while (pos < text.size()) {
        size_t eol = text.find('\n', pos);
        if (eol == std::string::npos) eol = text.size();
        std::string_view row(text.data() + pos, eol - pos);
        pos = eol + 1;
        ++line;
        if (!row.empty() && row.back() == '\r') row.remove_suffix(1);
        if (!have_header) {
            if (row != "config,time_ms")
                throw MalformedReplayFile(line, "expected header \"config,time_ms\"");
            have_header = true;
            continue;
        }
        if (row.empty()) continue;
        const size_t comma = row.find(',');
        if (comma == std::string_view::npos || comma == 0)
            throw MalformedReplayFile(line, "expected \"config,time_ms\"");
        const double t = replay_time(std::string(row.substr(comma + 1)), line);
        if (!table.try_emplace(std::string(row.substr(0, comma)), t).second)
            throw MalformedReplayFile(line, "duplicate configuration key");
    }
    if (!have_header) throw MalformedReplayFile(1, "empty file (missing header)");
    return ReplayBackend(std::move(table));
}

void ReplayBackend::save(const std::string& path, const std::map<std::string, double>& table) {
    std::string out = "config,time_ms\n";
    for (const auto& [key, t] : table) out.append(key).append(1, ',').append(format_double(t)).append(1, '\n');
    std::ofstream f(path, std::ios::binary);
    if (!f || !f.write(out.data(), std::streamsize(out.size())))
        throw Error("cannot write replay file \"" + path + "\"");
}

EvaluationResult ReplayBackend::evaluate(const EvaluationRequest& r) {
    EvaluationResult res;
    const std::string key = r.config.canonical();
    auto it = table_.find(key);
    if (it == table_.end()) {
        res.status = Status::missing;
        res.message = "no recorded time for " + key;
        return res;
    }
    res.status = Status::success;
    res.time_ms = it->second;
    return res;
}

// ---------------------------------------------------------------------------
// CudaBackend: ktb::Backend over the ktc C ABI.
// ---------------------------------------------------------------------------

namespace {

struct RequestView {
    std::vector<std::string> names;
    std::vector<const char*> name_ptrs;
    std::vector<long long> values;
    std::vector<ktc_arg> args;
    ktc_request req{};

    explicit RequestView(const EvaluationRequest& r) {
        const auto& ns = r.config.names();
        names.assign(ns.begin(), ns.end());
        for (const auto& n : names) name_ptrs.push_back(n.c_str());
        values.assign(r.config.values().begin(), r.config.values().end());
        for (const ArgumentSpec& a : r.arguments) {
            ktc_arg c{};
            c.role = a.role == ArgRole::input ? KTC_ARG_INPUT
                     : a.role == ArgRole::output ? KTC_ARG_OUTPUT
                                                 : KTC_ARG_SCALAR;
            c.type = a.type == ElementType::i32 ? KTC_I32 : KTC_F32;
            c.length = a.length;
            c.value = a.value;
            c.fill = a.fill.c_str();
            args.push_back(c);
        }
        req.kernel_name = r.kernel_name.c_str();
        req.source_ref = r.source_ref.c_str();
        req.n_params = int(values.size());
        req.param_names = name_ptrs.data();
        req.param_values = values.data();
        req.ndim = int(std::min<size_t>(3, r.global.size()));
        for (int d = 0; d < req.ndim; ++d) {
            req.global[d] = r.global[size_t(d)];
            req.local[d] = d < int(r.local.size()) ? r.local[size_t(d)] : 1;
        }
        req.n_args = int(args.size());
        req.args = args.data();
        req.device_name = r.device_name.c_str();
        req.repetitions = r.repetitions;
        req.want_outputs = r.want_outputs ? 1 : 0;
    }
};

}  // namespace

CudaBackend::CudaBackend(int ordinal, const ktc_backend_options* opts) : ordinal_(ordinal) {
    int st = ktc_backend_open(ordinal, opts, &be_);
    if (st != KTC_OK)
        throw BackendUnavailable(std::string("cuda:") + std::to_string(ordinal) + " (" +
                                 ktc_last_error(nullptr) + ")");
}

CudaBackend::~CudaBackend() { ktc_backend_close(be_); }

std::string CudaBackend::name() const { return ktc_backend_name(be_); }

EvaluationResult CudaBackend::evaluate(const EvaluationRequest& r) {
    RequestView v(r);
    EvaluationResult res;
    int st = ktc_backend_evaluate(be_, &v.req, &last_);
    if (st != KTC_OK) {
        // Harness breakage (device lost, OOM at upload, malformed request):
        // an error of the run, not of this configuration.
        if (st == KTC_ERR_INVALID || st == KTC_ERR_UNSUPPORTED)
            throw Error(std::string("cuda backend: ") + ktc_last_error(nullptr));
        throw Error(std::string("cuda backend failure: ") + ktc_last_error(nullptr));
    }
    totals_.compile_ms += last_.compile_ms;
    totals_.load_ms += last_.load_ms;
    totals_.run_ms += last_.run_ms;
    totals_.verify_ms += last_.verify_ms;
    totals_.evaluations += 1;
    totals_.cache_hits += size_t(last_.compile_cache_hit);
    totals_.launches += size_t(last_.kernel_launches);
    res.status = Status(last_.status);
    res.time_ms = last_.time_ms;
    res.message = last_.message;
    for (int k = 0; k < last_.n_outputs && k < KTC_MAX_OUTPUTS; ++k)
        if (last_.output_digests[k][0]) res.output_digests.emplace_back(last_.output_digests[k]);
    if (last_.verification != KTC_VERIFY_SKIPPED) {
        VerificationReport rep;
        rep.pass = last_.report.pass != 0;
        rep.max_abs_error = last_.report.max_abs_error;
        rep.max_rel_error = last_.report.max_rel_error;
        rep.buffer_index = last_.report.buffer_index;
        rep.element_index = last_.report.element_index;
        rep.elements_compared = last_.report.elements_compared;
        res.device_verification = rep;
    }
    return res;
}

void CudaBackend::prefetch(const EvaluationRequest& r) {
    RequestView v(r);
    ktc_backend_prefetch(be_, &v.req);
}

size_t CudaBackend::prefetch_depth() const { return ktc_backend_prefetch_depth(be_); }

bool CudaBackend::bind_reference(const EvaluationRequest& r, const std::vector<Buffer>& outputs) {
    RequestView v(r);
    std::vector<const void*> ptrs;
    std::vector<size_t> lens;
    std::vector<int> types;
    for (const Buffer& b : outputs) {
        ptrs.push_back(std::visit([](const auto& x) { return static_cast<const void*>(x.data()); }, b));
        lens.push_back(buffer_length(b));
        types.push_back(buffer_type(b) == ElementType::i32 ? KTC_I32 : KTC_F32);
    }
    int st = ktc_backend_set_reference(be_, &v.req, int(outputs.size()), ptrs.data(), lens.data(),
                                       types.data());
    if (st != KTC_OK) throw Error(std::string("bind_reference: ") + ktc_last_error(nullptr));
    return true;
}

}  // namespace ktb
