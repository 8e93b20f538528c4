// capi_tuner.cpp -- ktc.h layer 3: the CLTune-named tuner over the ktb
// search layer, and the reference's JSON job format (jobfile.hpp) with the
// added backend kind "cuda".
#include <chrono>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <json.hpp>
#include <memory>
#include <optional>
#include <sstream>

#include "ktb/landscapes.hpp"
#include "ktb/stats.hpp"
#include "ktb/tuner.hpp"
#include "ktc.h"

namespace ktc {
void set_error(const std::string& msg);
void trace_phase(const char* what, std::chrono::steady_clock::time_point since);
}

using namespace ktb;

struct ktc_tuner {
    TuningJob job;
    std::string family;  // "conv" | "gemm" | "gemm_tf32" | "" (custom)
    std::string backend_spec = "cuda";
    ktc_backend_options opts{};
    std::vector<int> devices{0};
    std::vector<uint64_t> subset;
    std::string checkpoint;
    std::string output = "results.csv";
    std::optional<SearchSpace> effective;
    std::vector<std::unique_ptr<Backend>> backends;
    std::string backends_key;
    std::optional<TuningOutcome> outcome;
    ktc_summary summary{};
    // CLTune SetReference: a reference kernel run once on the device over
    // the same arguments; its outputs become the verification reference.
    struct RefKernel {
        std::string source_ref, name;
        std::vector<size_t> global, local;
    };
    std::optional<RefKernel> ref_kernel;
    std::optional<std::vector<Buffer>> ref_outputs;  // computed or user-given
};

namespace {

int guard(const std::function<void()>& fn) {
    try {
        fn();
        return KTC_OK;
    } catch (const EmptySpace& e) {
        ktc::set_error(e.what());
        return KTC_ERR_EMPTY_SPACE;
    } catch (const EmptySpaceAfterConstraints& e) {
        ktc::set_error(e.what());
        return KTC_ERR_EMPTY_SPACE;
    } catch (const BackendUnavailable& e) {
        ktc::set_error(e.what());
        return KTC_ERR_UNSUPPORTED;
    } catch (const std::exception& e) {
        ktc::set_error(e.what());
        return KTC_ERR_INVALID;
    }
}

// Reports are written in binary mode and checked after the flush
// (report.hpp:114-127).
template <class Write>
void save_text(const std::string& path, Write&& write) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("cannot open \"" + path + "\" for writing");
    write(out);
    out.flush();
    if (!out) throw Error("failed while writing \"" + path + "\"");
}

void touched(ktc_tuner* t) {
    t->effective.reset();
    t->outcome.reset();
}

const SearchSpace& effective(ktc_tuner* t) {
    if (!t->effective) t->effective = compose_space(t->job.kernel, t->job.device, t->job.space);
    return *t->effective;
}

DeviceModel from_c(const ktc_device_model& d) {
    DeviceModel m;
    m.name = d.name;
    m.max_work_group_total = d.max_work_group_total;
    m.max_work_group_dim = {d.max_work_group_dim[0], d.max_work_group_dim[1],
                            d.max_work_group_dim[2]};
    m.local_mem_bytes = d.local_mem_bytes;
    m.peak_gflops = d.peak_gflops;
    m.peak_gbs = d.peak_gbs;
    return m;
}

void to_c(const DeviceModel& m, ktc_device_model* d) {
    std::memset(d, 0, sizeof(*d));
    std::snprintf(d->name, sizeof(d->name), "%s", m.name.c_str());
    d->max_work_group_total = m.max_work_group_total;
    for (int i = 0; i < 3; ++i) d->max_work_group_dim[i] = m.max_work_group_dim[size_t(i)];
    d->local_mem_bytes = m.local_mem_bytes;
    d->peak_gflops = m.peak_gflops;
    d->peak_gbs = m.peak_gbs;
}

DeviceModel query_cuda_device(int ordinal) {
    ktc_ctx* ctx = nullptr;
    if (ktc_open(ordinal, &ctx) != KTC_OK) throw UnknownDevice("cuda:" + std::to_string(ordinal));
    ktc_limits L;
    ktc_query_limits(ctx, &L);
    ktc_close(ctx);
    DeviceModel m;
    m.name = L.name;
    m.max_work_group_total = size_t(L.max_threads_per_block);
    m.max_work_group_dim = {size_t(L.max_block_dim[0]), size_t(L.max_block_dim[1]),
                            size_t(L.max_block_dim[2])};
    m.local_mem_bytes = L.smem_per_block_optin;
    m.peak_gflops = L.peak_fp32_gflops;
    m.peak_gbs = L.peak_hbm_gbs;
    return m;
}

DeviceModel resolve_device(const std::string& name) {
    if (name.rfind("cuda:", 0) == 0) return query_cuda_device(std::stoi(name.substr(5)));
    return device_preset(name);
}

void set_template(ktc_tuner* t, const std::string& fam, KernelSpec k, SearchSpace s) {
    t->family = fam;
    t->job.kernel = std::move(k);
    t->job.space = std::move(s);
    t->job.reference = nullptr;  // device reference (builtin.cu)
    touched(t);
}

// --------------------------------------------------------------------------
// Job files (reference jobfile.hpp): strict keys, template or custom kernel.
// --------------------------------------------------------------------------
using Json = nlohmann::ordered_json;

[[noreturn]] void jfail(const std::string& w) { throw JobFileError(w); }

void keys(const Json& n, const std::string& what, std::initializer_list<const char*> allowed) {
    if (!n.is_object()) jfail(what + " must be a JSON object");
    for (const auto& it : n.items()) {
        bool known = false;
        for (const char* a : allowed) known = known || it.key() == a;
        if (!known) jfail("unknown key \"" + it.key() + "\" in " + what);
    }
}

const Json* find(const Json& n, const char* k) {
    auto it = n.find(k);
    return it == n.end() ? nullptr : &*it;
}

std::string req_str(const Json& n, const char* k, const std::string& what) {
    const Json* v = find(n, k);
    if (!v || !v->is_string()) jfail(what + "." + k + " must be a string");
    return v->get<std::string>();
}

double opt_num(const Json& n, const char* k, const std::string& what, double dflt) {
    const Json* v = find(n, k);
    if (!v) return dflt;
    if (!v->is_number()) jfail(what + "." + k + " must be a number");
    return v->get<double>();
}

uint64_t opt_uns(const Json& n, const char* k, const std::string& what, uint64_t dflt) {
    const Json* v = find(n, k);
    if (!v) return dflt;
    if (!v->is_number_unsigned()) jfail(what + "." + k + " must be a non-negative integer");
    return v->get<uint64_t>();
}

bool opt_bool(const Json& n, const char* k, const std::string& what, bool dflt) {
    const Json* v = find(n, k);
    if (!v) return dflt;
    if (!v->is_boolean()) jfail(what + "." + k + " must be a boolean");
    return v->get<bool>();
}

std::vector<size_t> sizes(const Json& n, const std::string& what) {
    if (!n.is_array() || n.empty()) jfail(what + " must be a non-empty array of positive integers");
    std::vector<size_t> out;
    for (const Json& e : n) {
        if (!e.is_number_unsigned() || e.get<uint64_t>() == 0)
            jfail(what + " must contain positive integers only");
        out.push_back(e.get<size_t>());
    }
    return out;
}

double fraction(const Json& v) {
    if (v.is_number()) {
        const double f = v.get<double>();
        if (!(f > 0.0)) jfail("strategy.fraction must be positive");
        return f;
    }
    if (v.is_string()) {
        const std::string s = v.get<std::string>();
        auto parse = [&](const std::string& p) -> unsigned long long {
            unsigned long long o = 0;
            auto r = std::from_chars(p.data(), p.data() + p.size(), o);
            if (r.ec != std::errc{} || r.ptr != p.data() + p.size() || o == 0)
                jfail("strategy.fraction \"" + s + "\" is not a ratio of positive integers");
            return o;
        };
        const size_t slash = s.find('/');
        if (slash == std::string::npos) return double(parse(s));
        return double(parse(s.substr(0, slash))) / double(parse(s.substr(slash + 1)));
    }
    jfail("strategy.fraction must be a number or an \"a/b\" string");
}

void load_job(ktc_tuner* t, const std::string& text, const std::string& base_dir) {
    Json root;
    try {
        root = Json::parse(text);
    } catch (const nlohmann::json::parse_error& e) {
        throw JobFileError(std::string("invalid JSON: ") + e.what());
    }
    keys(root, "the job file", {"template", "problem", "kernel", "space", "device", "backend",
                                "strategy", "seed", "repetitions", "verify", "output"});
    const Json* tmpl = find(root, "template");
    const Json* kern = find(root, "kernel");
    if (tmpl && kern) jfail("\"template\" and \"kernel\" are mutually exclusive");
    if (!tmpl && !kern) jfail("the job needs either a \"template\" or a \"kernel\"");
    if (!tmpl && find(root, "problem")) jfail("\"problem\" only makes sense with a template");

    ktc_tuner fresh;
    fresh.opts = t->opts;
    fresh.devices = t->devices;
    if (tmpl) {
        if (!tmpl->is_string()) jfail("template must be a string");
        const std::string name = tmpl->get<std::string>();
        const Json* pn = find(root, "problem");
        if (name == "conv") {
            ConvProblem p;
            if (pn) {
                keys(*pn, "problem", {"x", "y", "filter", "weight", "seed"});
                p.x = size_t(opt_uns(*pn, "x", "problem", p.x));
                p.y = size_t(opt_uns(*pn, "y", "problem", p.y));
                p.filter = int(opt_uns(*pn, "filter", "problem", uint64_t(p.filter)));
                p.weight = float(opt_num(*pn, "weight", "problem", p.weight));
                p.seed = opt_uns(*pn, "seed", "problem", p.seed);
            }
            try {
                p.validate();
            } catch (const Error& e) {
                jfail(e.what());
            }
            set_template(&fresh, "conv", conv_kernel(p), conv_space());
        } else if (name == "gemm" || name == "gemm_tf32") {
            GemmProblem p;
            if (pn) {
                keys(*pn, "problem", {"m", "n", "k", "alpha", "beta", "seed"});
                p.m = size_t(opt_uns(*pn, "m", "problem", p.m));
                p.n = size_t(opt_uns(*pn, "n", "problem", p.n));
                p.k = size_t(opt_uns(*pn, "k", "problem", p.k));
                p.alpha = float(opt_num(*pn, "alpha", "problem", p.alpha));
                p.beta = float(opt_num(*pn, "beta", "problem", p.beta));
                p.seed = opt_uns(*pn, "seed", "problem", p.seed);
            }
            try {
                p.validate();
            } catch (const Error& e) {
                jfail(e.what());
            }
            if (name == "gemm") set_template(&fresh, "gemm", gemm_kernel(p), gemm_space());
            else set_template(&fresh, "gemm_tf32", gemm_tf32_kernel(p), gemm_tf32_space());
        } else {
            jfail("unknown template \"" + name + "\" (available: conv, gemm, gemm_tf32)");
        }
    } else {
        const Json& k = *kern;
        keys(k, "kernel", {"name", "source_ref", "global", "local", "modifiers", "local_mem",
                           "arguments"});
        KernelSpec ks;
        ks.name = req_str(k, "name", "kernel");
        ks.source_ref = find(k, "source_ref") ? req_str(k, "source_ref", "kernel") : ks.name + ".cl";
        const Json* g = find(k, "global");
        const Json* l = find(k, "local");
        if (!g || !l) jfail("kernel needs base \"global\" and \"local\" size arrays");
        ks.base_global = sizes(*g, "kernel.global");
        ks.base_local = sizes(*l, "kernel.local");
        if (ks.base_global.size() != ks.base_local.size())
            jfail("kernel.global and kernel.local must have the same rank");
        if (const Json* mods = find(k, "modifiers")) {
            if (!mods->is_array()) jfail("kernel.modifiers must be an array");
            size_t i = 0;
            for (const Json& m : *mods) {
                const std::string what = "kernel.modifiers[" + std::to_string(i++) + "]";
                keys(m, what, {"target", "op", "factors"});
                ThreadSizeModifier tm;
                const std::string target = req_str(m, "target", what), op = req_str(m, "op", what);
                if (target == "global") tm.target = SizeTarget::global;
                else if (target == "local") tm.target = SizeTarget::local;
                else jfail(what + ".target must be \"global\" or \"local\"");
                if (op == "multiply") tm.op = SizeOp::multiply;
                else if (op == "divide") tm.op = SizeOp::divide;
                else jfail(what + ".op must be \"multiply\" or \"divide\"");
                const Json* f = find(m, "factors");
                if (!f || !f->is_array() || f->empty())
                    jfail(what + ".factors must be a non-empty array of strings");
                for (const Json& x : *f) {
                    if (!x.is_string()) jfail(what + ".factors must contain strings only");
                    tm.factors.push_back(x.get<std::string>());
                }
                ks.modifiers.push_back(tm);
            }
        }
        if (const Json* lm = find(k, "local_mem")) {
            if (!lm->is_string()) jfail("kernel.local_mem must be a string");
            ks.local_mem_expr = lm->get<std::string>();
        }
        if (const Json* args = find(k, "arguments")) {
            if (!args->is_array()) jfail("kernel.arguments must be an array");
            size_t i = 0;
            for (const Json& a : *args) {
                const std::string what = "kernel.arguments[" + std::to_string(i++) + "]";
                keys(a, what, {"role", "type", "value", "length", "fill"});
                ArgumentSpec s;
                try {
                    s.role = arg_role_from(req_str(a, "role", what));
                    s.type = element_type_from(req_str(a, "type", what));
                } catch (const JobFileError&) {
                    throw;
                } catch (const Error& e) {
                    jfail(e.what());
                }
                if (s.role == ArgRole::scalar) {
                    const Json* v = find(a, "value");
                    if (!v || !v->is_number()) jfail(what + " is a scalar and needs a numeric \"value\"");
                    if (find(a, "length") || find(a, "fill"))
                        jfail(what + " is a scalar and cannot take \"length\" or \"fill\"");
                    s.value = v->get<double>();
                } else {
                    const Json* len = find(a, "length");
                    if (!len || !len->is_number_unsigned())
                        jfail(what + " is a buffer and needs a non-negative \"length\"");
                    if (find(a, "value")) jfail(what + " is a buffer and cannot take \"value\"");
                    s.length = len->get<size_t>();
                    if (const Json* f = find(a, "fill")) {
                        if (!f->is_string()) jfail(what + ".fill must be a string");
                        s.fill = f->get<std::string>();
                    }
                }
                ks.arguments.push_back(s);
            }
        }
        // Custom kernel sources resolve against the job directory.
        std::filesystem::path src(ks.source_ref);
        if (src.is_relative() && !base_dir.empty())
            ks.source_ref = (std::filesystem::path(base_dir) / src).string();
        fresh.job.kernel = ks;
        fresh.family.clear();
    }
    if (const Json* sp = find(root, "space")) {
        keys(*sp, "space", {"parameters", "constraints"});
        if (const Json* ps = find(*sp, "parameters")) {
            if (tmpl)
                jfail("space.parameters cannot be combined with a template (templates define "
                      "their own parameters)");
            if (!ps->is_object()) jfail("space.parameters must be a JSON object");
            for (const auto& it : ps->items()) {
                const Json& vals = it.value();
                if (!vals.is_array() || vals.empty())
                    jfail("space.parameters." + it.key() +
                          " must be a non-empty array of non-negative integers");
                std::vector<Value> list;
                for (const Json& v : vals) {
                    if (!v.is_number_unsigned())
                        jfail("space.parameters." + it.key() +
                              " must contain non-negative integers only");
                    list.push_back(v.get<Value>());
                }
                try {
                    fresh.job.space.add_parameter(it.key(), list);
                } catch (const Error& e) {
                    jfail(e.what());
                }
            }
        }
        if (const Json* cs = find(*sp, "constraints")) {
            if (!cs->is_array()) jfail("space.constraints must be an array of expressions");
            for (const Json& c : *cs) {
                if (!c.is_string()) jfail("space.constraints must contain strings only");
                try {
                    fresh.job.space.add_constraint(c.get<std::string>());
                } catch (const Error& e) {
                    jfail(e.what());
                }
            }
        }
    }
    if (fresh.job.space.parameters().empty())
        jfail("the job defines no parameters (add space.parameters)");
    if (const Json* dev = find(root, "device")) {
        if (dev->is_string()) {
            try {
                fresh.job.device = resolve_device(dev->get<std::string>());
            } catch (const Error& e) {
                jfail(e.what());
            }
        } else {
            keys(*dev, "device", {"name", "max_work_group_total", "max_work_group_dim",
                                  "local_mem_bytes", "peak_gflops", "peak_gbs"});
            DeviceModel d;
            d.name = req_str(*dev, "name", "device");
            d.max_work_group_total =
                size_t(opt_uns(*dev, "max_work_group_total", "device", d.max_work_group_total));
            if (const Json* dims = find(*dev, "max_work_group_dim")) {
                auto v = sizes(*dims, "device.max_work_group_dim");
                if (v.size() != 3) jfail("device.max_work_group_dim must hold exactly 3 entries");
                d.max_work_group_dim = {v[0], v[1], v[2]};
            }
            d.local_mem_bytes = size_t(opt_uns(*dev, "local_mem_bytes", "device", d.local_mem_bytes));
            d.peak_gflops = opt_num(*dev, "peak_gflops", "device", d.peak_gflops);
            d.peak_gbs = opt_num(*dev, "peak_gbs", "device", d.peak_gbs);
            fresh.job.device = d;
        }
    } else {
        fresh.job.device = device_preset("K40m");
    }
    if (const Json* st = find(root, "strategy")) {
        keys(*st, "strategy", {"kind", "fraction", "temperature", "alpha", "beta", "gamma", "swarm"});
        StrategySpec s;
        try {
            s.kind = strategy_kind_from(req_str(*st, "kind", "strategy"));
        } catch (const JobFileError&) {
            throw;
        } catch (const Error& e) {
            jfail(e.what());
        }
        if (const Json* f = find(*st, "fraction")) s.fraction = fraction(*f);
        s.temperature = opt_num(*st, "temperature", "strategy", s.temperature);
        s.alpha = opt_num(*st, "alpha", "strategy", s.alpha);
        s.beta = opt_num(*st, "beta", "strategy", s.beta);
        s.gamma = opt_num(*st, "gamma", "strategy", s.gamma);
        s.swarm = size_t(opt_uns(*st, "swarm", "strategy", s.swarm));
        if (s.swarm == 0) jfail("strategy.swarm must be at least 1");
        fresh.job.strategy = s;
    }
    fresh.job.seed = opt_uns(root, "seed", "the job file", fresh.job.seed);
    const uint64_t reps = opt_uns(root, "repetitions", "the job file", uint64_t(fresh.job.repetitions));
    if (reps == 0) jfail("repetitions must be at least 1");
    fresh.job.repetitions = int(reps);
    fresh.job.verify = opt_bool(root, "verify", "the job file", false);
    if (fresh.job.verify && fresh.family.empty())
        jfail("verify: true requires a built-in template (custom kernels have no reference oracle)");
    if (const Json* o = find(root, "output")) {
        if (!o->is_string()) jfail("the job file.output must be a string");
        fresh.output = o->get<std::string>();
    }
    if (const Json* be = find(root, "backend")) {
        keys(*be, "backend", {"kind", "path", "devices", "flush_l2", "warmup", "compile_threads",
                              "cache_dir", "rel_tol", "abs_tol", "model", "base_time_ms", "noise",
                              "noise_seed", "failure_rate", "argv", "timeout_ms", "workers"});
        const std::string kind = req_str(*be, "kind", "backend");
        if (kind == "replay") {
            std::filesystem::path p = req_str(*be, "path", "backend");
            if (p.is_relative() && !base_dir.empty()) p = std::filesystem::path(base_dir) / p;
            fresh.backend_spec = "replay:" + p.string();
        } else if (kind == "cuda") {
            fresh.backend_spec = "cuda";
            if (const Json* ds = find(*be, "devices")) {
                fresh.devices.clear();
                for (const Json& d : *ds) {
                    if (!d.is_number_unsigned()) jfail("backend.devices must list device ordinals");
                    fresh.devices.push_back(d.get<int>());
                }
                if (fresh.devices.empty()) jfail("backend.devices must not be empty");
            }
            fresh.opts.flush_l2 = opt_bool(*be, "flush_l2", "backend", fresh.opts.flush_l2) ? 1 : 0;
            fresh.opts.warmup = int(opt_uns(*be, "warmup", "backend", uint64_t(fresh.opts.warmup)));
            fresh.opts.compile_threads =
                int(opt_uns(*be, "compile_threads", "backend", uint64_t(fresh.opts.compile_threads)));
        } else {
            // synthetic / external are reference harness backends, not part
            // of this framework (out of scope).
            throw BackendUnavailable(kind);
        }
    }
    fresh.job.rel_tol = fresh.family == "gemm_tf32" ? 1e-3 : 1e-4;
    t->job = std::move(fresh.job);
    t->family = fresh.family;
    t->backend_spec = fresh.backend_spec;
    t->opts = fresh.opts;
    t->devices = fresh.devices;
    t->output = fresh.output;
    t->subset.clear();
    touched(t);
}

void ensure_backends(ktc_tuner* t) {
    std::string key = t->backend_spec;
    for (int d : t->devices) key += ":" + std::to_string(d);
    key += "|" + std::to_string(t->opts.flush_l2) + std::to_string(t->opts.warmup) +
           std::to_string(t->opts.compile_threads) + std::to_string(t->job.rel_tol) +
           std::to_string(t->job.abs_tol) + "|" + std::to_string(t->opts.prune_factor) + "|" +
           std::to_string(t->opts.isolate) + t->family;
    if (key == t->backends_key && !t->backends.empty()) return;
    t->backends.clear();
    if (t->backend_spec == "cuda") {
        ktc_backend_options o = t->opts;
        o.rel_tol = t->job.rel_tol;
        o.abs_tol = t->job.abs_tol;
        // A user kernel may fault or hang; its evaluations run in a worker
        // process per device so one bad configuration costs one row, not the
        // process (the built-in families are generated and verified here).
        if (t->family.empty()) o.isolate = 1;
        for (int d : t->devices) t->backends.push_back(std::make_unique<CudaBackend>(d, &o));
    } else if (t->backend_spec.rfind("replay:", 0) == 0) {
        // One replay worker per listed "device": exercises the sharded
        // executor on hosts without GPUs (tests of the merge rule).
        const ReplayBackend proto = ReplayBackend::load(t->backend_spec.substr(7));
        for (size_t i = 0; i < t->devices.size(); ++i)
            t->backends.push_back(std::make_unique<ReplayBackend>(proto.table()));
    } else {
        throw BackendUnavailable(t->backend_spec);
    }
    t->backends_key = key;
}

// Runs the CLTune reference kernel once (first device) over the job's
// arguments and keeps its outputs as the host reference of the job.
void compute_reference_outputs(ktc_tuner* t) {
    auto* cb = t->backends.empty() ? nullptr : dynamic_cast<CudaBackend*>(t->backends[0].get());
    if (!cb) throw Error("SetReference(kernel) needs the cuda backend");
    const auto& rk = *t->ref_kernel;
    EvaluationRequest req;
    req.kernel_name = rk.name;
    req.source_ref = rk.source_ref;
    req.global = rk.global;
    req.local = rk.local;
    req.arguments = t->job.kernel.arguments;
    req.device_name = t->job.device.name;
    req.repetitions = 1;
    req.want_outputs = false;  // nothing to verify the reference against
    EvaluationResult r = cb->evaluate(req);
    if (!r.ok()) throw Error("reference kernel " + rk.name + " failed: " + r.message);
    std::vector<Buffer> outs;
    int k = 0;
    for (const ArgumentSpec& a : t->job.kernel.arguments) {
        if (a.role != ArgRole::output) continue;
        int st;
        if (a.type == ElementType::i32) {
            std::vector<int32_t> h(a.length);
            st = ktc_backend_read_output(cb->handle(), k, h.data(), h.size() * 4);
            outs.emplace_back(std::move(h));
        } else {
            std::vector<float> h(a.length);
            st = ktc_backend_read_output(cb->handle(), k, h.data(), h.size() * 4);
            outs.emplace_back(std::move(h));
        }
        if (st != KTC_OK) throw Error("cannot read reference output " + std::to_string(k));
        ++k;
    }
    t->ref_outputs = outs;
    auto shared = std::make_shared<std::vector<Buffer>>(std::move(outs));
    t->job.reference = [shared] { return *shared; };
}

void tune(ktc_tuner* t) {
    const auto tb = std::chrono::steady_clock::now();
    ensure_backends(t);
    ktc::trace_phase("tune: backends", tb);
    if (t->ref_kernel && !t->ref_outputs) compute_reference_outputs(t);
    const SearchSpace& eff = effective(t);
    ktc::trace_phase("tune: + effective space", tb);
    std::vector<Backend*> bes;
    for (auto& b : t->backends) bes.push_back(b.get());
    for (Backend* b : bes)
        if (auto* c = dynamic_cast<CudaBackend*>(b)) c->reset_totals();
    auto t0 = std::chrono::steady_clock::now();
    std::unique_ptr<ResultLog> log;
    if (!t->checkpoint.empty())
        log = std::make_unique<ResultLog>(t->checkpoint, job_signature(t->job));
    TuningOutcome o = run_tuning_sharded(t->job, bes, eff, t->subset, log.get());
    ktc::trace_phase("tune: + search", tb);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ktc_summary& s = t->summary;
    std::memset(&s, 0, sizeof(s));
    s.rows = o.rows.size();
    s.best_index = o.best_index ? (long long)*o.best_index : -1;
    s.best_time_ms = o.best_time_ms ? *o.best_time_ms : std::nan("");
    s.budget = o.budget;
    s.unique_evaluations = o.unique_evaluations;
    s.failed_evaluations = o.failed_evaluations;
    s.total_steps = o.total_steps;
    s.space_size = o.space_size;
    s.wall_s = wall;
    s.configs_per_s = wall > 0 ? double(o.rows.size()) / wall : 0.0;
    for (Backend* b : bes)
        if (auto* c = dynamic_cast<CudaBackend*>(b)) {
            const auto& tt = c->totals();
            s.compile_s += tt.compile_ms / 1e3;
            s.device_s += (tt.load_ms + tt.run_ms + tt.verify_ms) / 1e3;
            s.compile_cache_hits += tt.cache_hits;
            s.kernel_launches += tt.launches;
        }
    t->outcome = std::move(o);
}

void fill_row(const TuningRow& r, ktc_row* out) {
    std::memset(out, 0, sizeof(*out));
    out->step = r.step;
    out->status = int(r.status);
    out->time_ms = r.time_ms ? *r.time_ms : std::nan("");
    out->verification = r.verification == Verification::pass   ? KTC_VERIFY_PASS
                        : r.verification == Verification::fail ? KTC_VERIFY_FAIL
                                                                : KTC_VERIFY_SKIPPED;
    out->best_so_far = r.best_so_far ? *r.best_so_far : std::nan("");
    out->ndim = int(std::min<size_t>(3, r.sizes.global.size()));
    for (int d = 0; d < out->ndim; ++d) {
        out->global[d] = r.sizes.global[size_t(d)];
        out->local[d] = r.sizes.local[size_t(d)];
    }
    out->space_index = r.space_index;
    out->device = r.device;
    if (r.report) {
        out->report.pass = r.report->pass ? 1 : 0;
        out->report.max_abs_error = r.report->max_abs_error;
        out->report.max_rel_error = r.report->max_rel_error;
        out->report.buffer_index = r.report->buffer_index;
        out->report.element_index = r.report->element_index;
        out->report.elements_compared = r.report->elements_compared;
    }
}

void copy_str(const std::string& s, char* out, size_t cap) {
    if (out && cap) std::snprintf(out, cap, "%s", s.c_str());
}

ArgumentSpec arg_from_c(const ktc_arg* a) {
    ArgumentSpec s;
    s.role = a->role == KTC_ARG_INPUT ? ArgRole::input
             : a->role == KTC_ARG_OUTPUT ? ArgRole::output
                                         : ArgRole::scalar;
    s.type = a->type == KTC_I32 ? ElementType::i32 : ElementType::f32;
    s.length = a->length;
    s.value = a->value;
    s.fill = a->fill ? a->fill : "none";
    return s;
}

}  // namespace

extern "C" {

int ktc_device_preset(const char* name, ktc_device_model* out) {
    return guard([&] { to_c(resolve_device(name ? name : ""), out); });
}

int ktc_tuner_create(ktc_tuner** out) {
    *out = new ktc_tuner;
    ktc_backend_default_options(&(*out)->opts);
    (*out)->job.device = device_preset("B200");
    return KTC_OK;
}

void ktc_tuner_destroy(ktc_tuner* t) {
    const auto t0 = std::chrono::steady_clock::now();
    delete t;
    ktc::trace_phase("tuner destroy", t0);
}

int ktc_tuner_template_conv(ktc_tuner* t, size_t x, size_t y, int filter, float weight,
                            uint64_t seed) {
    return guard([&] {
        ConvProblem p{x, y, filter, weight, seed};
        set_template(t, "conv", conv_kernel(p), conv_space());
    });
}

int ktc_tuner_template_gemm(ktc_tuner* t, size_t m, size_t n, size_t k, float alpha, float beta,
                            uint64_t seed) {
    return guard([&] {
        GemmProblem p{m, n, k, alpha, beta, seed};
        set_template(t, "gemm", gemm_kernel(p), gemm_space());
    });
}

int ktc_tuner_template_gemm_tf32(ktc_tuner* t, size_t m, size_t n, size_t k, float alpha,
                                 float beta, uint64_t seed) {
    return guard([&] {
        GemmProblem p{m, n, k, alpha, beta, seed};
        set_template(t, "gemm_tf32", gemm_tf32_kernel(p), gemm_tf32_space());
        t->job.rel_tol = 1e-3;
    });
}

int ktc_tuner_add_kernel(ktc_tuner* t, const char* source_ref, const char* name, int ndim,
                         const size_t* global, const size_t* local) {
    return guard([&] {
        KernelSpec k;
        k.name = name ? name : "";
        k.source_ref = source_ref ? source_ref : "";
        k.base_global.assign(global, global + ndim);
        k.base_local.assign(local, local + ndim);
        t->job.kernel = k;
        t->job.space = SearchSpace{};
        t->family.clear();
        touched(t);
    });
}

int ktc_tuner_add_parameter(ktc_tuner* t, const char* name, const long long* values, int n) {
    return guard([&] {
        t->job.space.add_parameter(name, std::vector<Value>(values, values + n));
        touched(t);
    });
}

int ktc_tuner_add_constraint(ktc_tuner* t, const char* expr) {
    return guard([&] {
        t->job.space.add_constraint(expr);
        touched(t);
    });
}

int ktc_tuner_add_modifier(ktc_tuner* t, int target, int op, const char* const* factors, int n) {
    return guard([&] {
        ThreadSizeModifier m;
        m.target = target == 0 ? SizeTarget::global : SizeTarget::local;
        m.op = op == 0 ? SizeOp::multiply : SizeOp::divide;
        for (int i = 0; i < n; ++i) m.factors.emplace_back(factors[i]);
        t->job.kernel.modifiers.push_back(m);
        touched(t);
    });
}

int ktc_tuner_set_local_memory(ktc_tuner* t, const char* expr) {
    return guard([&] {
        t->job.kernel.local_mem_expr = expr ? expr : "";
        touched(t);
    });
}

int ktc_tuner_add_argument(ktc_tuner* t, const ktc_arg* arg) {
    return guard([&] {
        t->job.kernel.arguments.push_back(arg_from_c(arg));
        if (t->ref_kernel) t->ref_outputs.reset();  // recomputed for the new argument list
        touched(t);
    });
}

int ktc_tuner_set_reference_kernel(ktc_tuner* t, const char* source_ref, const char* name,
                                   int ndim, const size_t* global, const size_t* local) {
    return guard([&] {
        if (ndim < 1 || ndim > 3) throw Error("reference kernel needs 1 to 3 dimensions");
        ktc_tuner::RefKernel k;
        k.source_ref = source_ref ? source_ref : "";
        k.name = name ? name : "";
        k.global.assign(global, global + ndim);
        k.local.assign(local, local + ndim);
        t->ref_kernel = k;
        t->ref_outputs.reset();
        t->job.reference = nullptr;
        touched(t);
    });
}

int ktc_tuner_set_reference_outputs(ktc_tuner* t, int n, const void* const* buffers,
                                    const size_t* lengths, const int* types) {
    return guard([&] {
        std::vector<Buffer> refs;
        for (int i = 0; i < n; ++i) {
            if (types[i] == KTC_I32) {
                const auto* p = static_cast<const int32_t*>(buffers[i]);
                refs.emplace_back(std::vector<int32_t>(p, p + lengths[i]));
            } else {
                const auto* p = static_cast<const float*>(buffers[i]);
                refs.emplace_back(std::vector<float>(p, p + lengths[i]));
            }
        }
        t->ref_kernel.reset();
        t->ref_outputs = std::move(refs);
        auto shared = std::make_shared<std::vector<Buffer>>(*t->ref_outputs);
        t->job.reference = [shared] { return *shared; };
        touched(t);
    });
}

int ktc_tuner_set_device(ktc_tuner* t, const ktc_device_model* dev) {
    return guard([&] {
        t->job.device = from_c(*dev);
        touched(t);
    });
}

int ktc_tuner_set_strategy(ktc_tuner* t, int kind, double fraction, double temperature,
                           double alpha, double beta, double gamma, size_t swarm) {
    return guard([&] {
        StrategySpec s;
        s.kind = kind == KTC_SEARCH_FULL      ? StrategyKind::full
                 : kind == KTC_SEARCH_RANDOM  ? StrategyKind::random
                 : kind == KTC_SEARCH_ANNEALING ? StrategyKind::annealing
                                                : StrategyKind::pso;
        s.fraction = fraction;
        s.temperature = temperature;
        s.alpha = alpha;
        s.beta = beta;
        s.gamma = gamma;
        s.swarm = swarm;
        t->job.strategy = s;
        t->outcome.reset();
    });
}

int ktc_tuner_set_seed(ktc_tuner* t, uint64_t seed) {
    t->job.seed = seed;
    return KTC_OK;
}

int ktc_tuner_set_repetitions(ktc_tuner* t, int reps) {
    if (reps < 1) {
        ktc::set_error("repetitions must be at least 1");
        return KTC_ERR_INVALID;
    }
    t->job.repetitions = reps;
    return KTC_OK;
}

int ktc_tuner_set_verification(ktc_tuner* t, int verify, double rel_tol, double abs_tol) {
    t->job.verify = verify != 0;
    t->job.rel_tol = rel_tol;
    t->job.abs_tol = abs_tol;
    return KTC_OK;
}

int ktc_tuner_set_backend(ktc_tuner* t, const char* spec, const ktc_backend_options* opts) {
    return guard([&] {
        t->backend_spec = spec ? spec : "cuda";
        if (opts) t->opts = *opts;
        t->opts.cache_dir = nullptr;
        t->backends.clear();
        t->backends_key.clear();
    });
}

int ktc_tuner_set_devices(ktc_tuner* t, const int* ordinals, int n) {
    return guard([&] {
        if (n < 1) throw Error("at least one device");
        t->devices.assign(ordinals, ordinals + n);
    });
}

int ktc_tuner_set_subset(ktc_tuner* t, const uint64_t* indices, size_t n) {
    return guard([&] { t->subset.assign(indices, indices + n); });
}

int ktc_tuner_set_checkpoint(ktc_tuner* t, const char* path) {
    t->checkpoint = path ? path : "";
    return KTC_OK;
}

int ktc_tuner_space_counts(ktc_tuner* t, unsigned long long* raw, unsigned long long* constrained,
                           unsigned long long* valid) {
    return guard([&] {
        const SearchSpace& e = effective(t);
        *raw = e.raw_size();
        *constrained = e.constraint_only_count();
        *valid = e.valid_count();
    });
}

int ktc_tuner_space_config(ktc_tuner* t, uint64_t index, char* out, size_t cap) {
    return guard([&] { copy_str(effective(t).config_at(size_t(index)).canonical(), out, cap); });
}

int ktc_tuner_tune(ktc_tuner* t) { return guard([&] { tune(t); }); }

int ktc_tuner_summary(ktc_tuner* t, ktc_summary* out) {
    if (!t->outcome) {
        ktc::set_error("Tune() has not run");
        return KTC_ERR_INVALID;
    }
    *out = t->summary;
    return KTC_OK;
}

int ktc_tuner_row(ktc_tuner* t, size_t i, ktc_row* out, char* config, size_t cap, char* message,
                  size_t msg_cap) {
    if (!t->outcome || i >= t->outcome->rows.size()) {
        ktc::set_error("row index out of range");
        return KTC_ERR_INVALID;
    }
    const TuningRow& r = t->outcome->rows[i];
    fill_row(r, out);
    copy_str(r.config.canonical(), config, cap);
    copy_str(r.message, message, msg_cap);
    return KTC_OK;
}

int ktc_tuner_best(ktc_tuner* t, char* config, size_t cap, double* time_ms) {
    if (!t->outcome || !t->outcome->best_config) {
        ktc::set_error("no successful configuration");
        return KTC_ERR_INVALID;
    }
    copy_str(t->outcome->best_config->canonical(), config, cap);
    *time_ms = *t->outcome->best_time_ms;
    return KTC_OK;
}

int ktc_tuner_write_csv(ktc_tuner* t, const char* path) {
    return guard([&] {
        if (!t->outcome) throw Error("Tune() has not run");
        std::ofstream out(path, std::ios::binary);
        if (!out) throw Error(std::string("cannot open \"") + path + "\" for writing");
        write_results_csv(out, *t->outcome);
    });
}

int ktc_tuner_write_replay(ktc_tuner* t, const char* path) {
    return guard([&] {
        if (!t->outcome) throw Error("Tune() has not run");
        std::map<std::string, double> table;
        for (const TuningRow& r : t->outcome->rows)
            if (r.status == Status::success && r.time_ms && r.verification != Verification::fail)
                table.emplace(r.config.canonical(), *r.time_ms);
        ReplayBackend::save(path, table);
    });
}

int ktc_tuner_stats(ktc_tuner* t, size_t runs, uint64_t base_seed, const char* out_csv,
                    ktc_stats_summary* out) {
    return guard([&] {
        if (!out_csv) throw Error("ktc_tuner_stats: no output path");
        const auto t0 = std::chrono::steady_clock::now();
        ensure_backends(t);
        if (t->ref_kernel && !t->ref_outputs) compute_reference_outputs(t);
        std::vector<Backend*> bes;
        for (auto& b : t->backends) bes.push_back(b.get());
        StatsOutcome st = run_stats(t->job, bes, effective(t), runs, base_seed);
        const std::string path(out_csv);
        save_text(path, [&](std::ostream& o) { write_stats_csv(o, st.best_of_run); });
        save_text(derive_report_path(path, "_runs"),
                  [&](std::ostream& o) { write_runs_csv(o, st.runs); });
        if (st.space)
            save_text(derive_report_path(path, "_space"),
                      [&](std::ostream& o) { write_stats_csv(o, *st.space); });
        if (out) {
            std::memset(out, 0, sizeof(*out));
            const Summary& s = st.best_of_run.summary;
            out->runs = s.count;
            out->mean = s.mean;
            out->stddev = s.stddev;
            out->min = s.min;
            out->max = s.max;
            out->space_written = st.space ? 1 : 0;
            if (st.space) {
                out->space_count = st.space->summary.count;
                out->space_min = st.space->summary.min;
                out->space_mean = st.space->summary.mean;
            }
            out->wall_s =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

int ktc_stats_write(const double* values, size_t n, const char* path) {
    return guard([&] {
        if (!path) throw Error("ktc_stats_write: no output path");
        ExperimentStats st = make_experiment_stats(std::vector<double>(values, values + n));
        save_text(path, [&](std::ostream& o) { write_stats_csv(o, st); });
    });
}

int ktc_runs_write(const ktc_run_summary* runs, size_t n, const char* path) {
    return guard([&] {
        if (!path) throw Error("ktc_runs_write: no output path");
        std::vector<RunSummary> rs;
        rs.reserve(n);
        for (size_t i = 0; i < n; ++i)
            rs.push_back({runs[i].run, runs[i].seed, runs[i].best_time_ms,
                          runs[i].best_config ? runs[i].best_config : ""});
        save_text(path, [&](std::ostream& o) { write_runs_csv(o, rs); });
    });
}

int ktc_tuner_job_info(ktc_tuner* t, ktc_job_info* out) {
    return guard([&] {
        std::memset(out, 0, sizeof(*out));
        copy_str(t->job.kernel.name, out->kernel, sizeof(out->kernel));
        copy_str(t->job.device.name, out->device, sizeof(out->device));
        copy_str(t->outcome ? t->outcome->backend_name : t->backend_spec, out->backend,
                 sizeof(out->backend));
        copy_str(t->output, out->output, sizeof(out->output));
        out->is_cuda = t->backend_spec == "cuda";
        out->ndevices = int(std::min<size_t>(t->devices.size(), 64));
        for (int i = 0; i < out->ndevices; ++i) out->devices[i] = t->devices[size_t(i)];
    });
}

int ktc_tuner_load_job(ktc_tuner* t, const char* json_text, const char* base_dir) {
    return guard([&] { load_job(t, json_text, base_dir ? base_dir : ""); });
}

}  // extern "C"
