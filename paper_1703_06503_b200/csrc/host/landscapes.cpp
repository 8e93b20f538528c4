// landscapes.cpp -- the conv2d and SGEMM case studies (reference
// landscapes.hpp:24-428): spaces, kernel descriptions, metrics, and the
// paper's best-known rows (Tables II and IV).
#include "ktb/landscapes.hpp"

#include <utility>

namespace ktb {

void ConvProblem::validate() const {
    if (x == 0 || y == 0) throw Error("convolution image dimensions must be positive");
    if (filter < 1 || filter % 2 == 0) throw Error("convolution filter size must be odd and positive");
}

void GemmProblem::validate() const {
    if (m == 0 || n == 0 || k == 0) throw Error("matrix dimensions must be positive");
}

SearchSpace conv_space() {
    SearchSpace s;
    s.add_parameter("XWG", {8, 16, 32, 64});
    s.add_parameter("YWG", {8, 16, 32, 64});
    s.add_parameter("XWPT", {1, 2, 4, 8});
    s.add_parameter("YWPT", {1, 2, 4, 8});
    s.add_parameter("LOCAL", {0, 1, 2});
    s.add_parameter("VW", {1, 2, 4, 8});
    s.add_parameter("PAD", {0, 1});
    s.add_parameter("UNR", {0, 1}, {"no", "yes"});
    s.add_constraint("VW <= XWPT && XWPT % VW == 0");
    s.add_constraint("PAD == 0 || LOCAL >= 1");
    return s;
}

static ArgumentSpec scalar(ElementType t, double v) {
    return ArgumentSpec{ArgRole::scalar, t, 0, v, ""};
}

static ArgumentSpec buffer(ArgRole r, size_t n, std::string fill) {
    return ArgumentSpec{r, ElementType::f32, n, 0.0, std::move(fill)};
}

KernelSpec conv_kernel(const ConvProblem& p) {
    p.validate();
    KernelSpec k;
    k.name = "conv";
    k.source_ref = "conv.cl";
    k.base_global = {p.x, p.y};
    k.base_local = {1, 1};
    k.modifiers = {{SizeTarget::global, SizeOp::divide, {"XWPT", "YWPT"}},
                   {SizeTarget::local, SizeOp::multiply, {"XWG", "YWG"}}};
    const std::string h2 = std::to_string(2 * p.halo());
    k.local_mem_expr =
        "(LOCAL >= 1) * 4 * (XWG * XWPT + " + h2 + " + PAD) * (YWG * YWPT + " + h2 + ")";
    k.arguments = {scalar(ElementType::i32, double(p.x)),
                   scalar(ElementType::i32, double(p.y)),
                   scalar(ElementType::i32, double(p.filter)),
                   scalar(ElementType::f32, double(p.weight)),
                   buffer(ArgRole::input, p.padded_x() * p.padded_y(),
                          "uniform:" + std::to_string(p.seed)),
                   buffer(ArgRole::input, size_t(p.filter) * size_t(p.filter),
                          "uniform:" + std::to_string(p.filter_seed())),
                   buffer(ArgRole::output, p.x * p.y, "none")};
    return k;
}

ConvMetrics conv_metrics(const ConvProblem& p, double time_ms) {
    if (!(time_ms > 0.0)) throw NonPositiveTime(time_ms);
    const double elems = double(p.x) * double(p.y), f = double(p.filter), sec = time_ms / 1e3;
    return ConvMetrics{(1.0 + 2.0 * f * f) * elems / sec / 1e9, 2.0 * elems * 4.0 / sec / 1e9};
}

SearchSpace gemm_space() {
    SearchSpace s;
    s.add_parameter("MWG", {16, 32, 64, 128});
    s.add_parameter("NWG", {16, 32, 64, 128});
    s.add_parameter("KWG", {16, 32, 64, 128});
    s.add_parameter("MDIMC", {8, 16, 32});
    s.add_parameter("NDIMC", {8, 16, 32});
    s.add_parameter("SA", {0, 1}, {"no", "yes"});
    s.add_parameter("SB", {0, 1}, {"no", "yes"});
    s.add_parameter("MDIMA", {8, 16, 32});
    s.add_parameter("NDIMB", {8, 16, 32});
    s.add_parameter("STRM", {0, 1}, {"no", "yes"});
    s.add_parameter("STRN", {0, 1}, {"no", "yes"});
    s.add_parameter("VWM", {1, 2, 4, 8});
    s.add_parameter("VWN", {1, 2, 4, 8});
    s.add_parameter("KWI", {2, 8});
    s.add_constraint("MWG % MDIMC == 0");
    s.add_constraint("NWG % NDIMC == 0");
    s.add_constraint("(MDIMC * NDIMC) % MDIMA == 0");
    s.add_constraint("(MDIMC * NDIMC) % NDIMB == 0");
    s.add_constraint("KWG % ((MDIMC * NDIMC) / MDIMA) == 0");
    s.add_constraint("KWG % ((MDIMC * NDIMC) / NDIMB) == 0");
    s.add_constraint("KWG % KWI == 0");
    s.add_constraint("(MWG / MDIMC) % VWM == 0");
    s.add_constraint("(NWG / NDIMC) % VWN == 0");
    return s;
}

static std::vector<ArgumentSpec> gemm_arguments(const GemmProblem& p) {
    return {scalar(ElementType::i32, double(p.m)),
            scalar(ElementType::i32, double(p.n)),
            scalar(ElementType::i32, double(p.k)),
            scalar(ElementType::f32, double(p.alpha)),
            scalar(ElementType::f32, double(p.beta)),
            buffer(ArgRole::input, p.k * p.m, "uniform:" + std::to_string(p.a_seed())),
            buffer(ArgRole::input, p.k * p.n, "uniform:" + std::to_string(p.b_seed())),
            buffer(ArgRole::output, p.m * p.n, "uniform:" + std::to_string(p.c_seed()))};
}

KernelSpec gemm_kernel(const GemmProblem& p) {
    p.validate();
    KernelSpec k;
    k.name = "gemm";
    k.source_ref = "gemm.cl";
    k.base_global = {p.m, p.n};
    k.base_local = {1, 1};
    k.modifiers = {{SizeTarget::global, SizeOp::multiply, {"MDIMC", "NDIMC"}},
                   {SizeTarget::global, SizeOp::divide, {"MWG", "NWG"}},
                   {SizeTarget::local, SizeOp::multiply, {"MDIMC", "NDIMC"}}};
    k.local_mem_expr = "SA * 4 * KWG * MWG + SB * 4 * KWG * NWG";
    k.arguments = gemm_arguments(p);
    return k;
}

double gemm_gflops(const GemmProblem& p, double time_ms) {
    if (!(time_ms > 0.0)) throw NonPositiveTime(time_ms);
    return 2.0 * double(p.m) * double(p.n) * double(p.k) / (time_ms / 1e3) / 1e9;
}

SearchSpace gemm_tf32_space() {
    SearchSpace s;
    s.add_parameter("BN", {64, 128, 256});
    s.add_parameter("BK", {32, 64});
    s.add_parameter("STAGES", {2, 3, 4, 6});
    s.add_parameter("CG", {1, 2});  // 2: CTA pair (cta_group::2), 256 x BN tiles
    return s;
}

KernelSpec gemm_tf32_kernel(const GemmProblem& p) {
    p.validate();
    KernelSpec k;
    k.name = "gemm_tf32";
    k.source_ref = "gemm_tf32.cu";
    // One 128-thread CTA per 128 x BN output tile: grid (M/128, N/BN); with
    // CG = 2 the CTAs pair up along M (clusters of 2) and each stages half
    // of B, hence the shared-memory expression.
    k.base_global = {p.m, p.n};
    k.base_local = {128, 1};
    k.modifiers = {{SizeTarget::global, SizeOp::divide, {"1", "BN"}}};
    k.local_mem_expr = "STAGES * 4 * BK * (128 + BN / CG) + 2048";
    k.arguments = gemm_arguments(p);
    return k;
}

namespace {

using Named = std::vector<std::pair<const char*, Value>>;

Configuration assemble(const SearchSpace& s, const Named& entries) {
    std::vector<Value> v(s.parameters().size());
    for (const auto& e : entries) v[s.parameter_index(e.first)] = e.second;
    return s.make_configuration(std::move(v));
}

Configuration conv_row(const SearchSpace& s, Value xwg, Value ywg, Value xwpt, Value ywpt,
                       Value local, Value vw, Value pad, Value unr) {
    return assemble(s, {{"XWG", xwg}, {"YWG", ywg}, {"XWPT", xwpt}, {"YWPT", ywpt},
                        {"LOCAL", local}, {"VW", vw}, {"PAD", pad}, {"UNR", unr}});
}

Configuration gemm_row(const SearchSpace& s, const Value (&v)[14]) {
    static const char* names[14] = {"MWG", "NWG", "KWG", "MDIMC", "NDIMC", "SA",  "SB",
                                    "MDIMA", "NDIMB", "STRM", "STRN", "VWM", "VWN", "KWI"};
    Named n;
    for (int i = 0; i < 14; ++i) n.emplace_back(names[i], v[i]);
    return assemble(s, n);
}

}  // namespace

// Paper Table II (reference landscapes.hpp:357-386).
Configuration conv_best_known(const SearchSpace& s, const std::string& device, int filter) {
    auto missing = [&]() {
        return Error("no known-best convolution entry for filter size " + std::to_string(filter) +
                     " on " + device);
    };
    if (device == "K40m") {
        if (filter == 3) return conv_row(s, 32, 8, 1, 8, 0, 1, 0, 1);
        if (filter == 7) return conv_row(s, 32, 16, 2, 4, 2, 2, 1, 1);
        if (filter == 11) return conv_row(s, 32, 8, 2, 8, 2, 2, 1, 1);
        throw missing();
    }
    if (device == "GTX480") {
        if (filter == 3) return conv_row(s, 64, 8, 1, 4, 0, 1, 0, 1);
        if (filter == 7) return conv_row(s, 32, 8, 2, 8, 2, 2, 0, 1);
        if (filter == 11) return conv_row(s, 32, 8, 2, 4, 1, 2, 0, 1);
        throw missing();
    }
    throw UnknownDevice(device);
}

std::vector<std::string> conv_best_known_devices() { return {"K40m", "GTX480"}; }

// Paper Table IV (reference landscapes.hpp:394-428).
Configuration gemm_best_known(const SearchSpace& s, const std::string& device) {
    if (device == "K40m") return gemm_row(s, {128, 128, 16, 16, 16, 1, 1, 32, 16, 1, 0, 2, 1, 8});
    if (device == "GTX480") return gemm_row(s, {64, 64, 32, 8, 16, 1, 1, 32, 32, 1, 0, 2, 2, 8});
    if (device == "HD7970") return gemm_row(s, {128, 128, 32, 16, 16, 1, 1, 32, 32, 0, 1, 4, 4, 2});
    if (device == "Iris5100") return gemm_row(s, {64, 64, 16, 8, 8, 1, 1, 8, 16, 1, 1, 4, 4, 8});
    throw UnknownDevice(device);
}

std::vector<std::string> gemm_best_known_devices() { return {"K40m", "GTX480", "HD7970", "Iris5100"}; }

}  // namespace ktb
