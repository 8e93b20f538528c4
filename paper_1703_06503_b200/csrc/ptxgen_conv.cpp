// ptxgen_conv.cpp -- direct PTX generation for the convolution family.
//
// Emits, for one configuration, exactly the kernel that kernels/conv.cu
// describes (same parameters, same HBM / shared-memory layouts, same TMA halo
// staging, the same fused-multiply-add sequence per output -- so the outputs
// are bit-identical to the NVRTC build, tests/test_gpu_ptxgen.py), but as
// PTX text: the configuration is already fully specialized and unrolled here,
// so the tuning-time compile is ptxas only (nvPTXCompiler, in process).
// NVVM's optimizer, ~70% of an NVRTC compile of this family and growing
// super-linearly with the unrolled body, is skipped.
//
// Structure of the emitted entry (see conv.cu for the semantics):
//   prologue   tile origin, thread offsets
//   LOCAL = 0  sliding windows read with ld.global.nc (vector width VW)
//   LOCAL = 1  cooperative halo copy into shared memory (4 copies per trip),
//              bar.sync, windows from shared memory
//   LOCAL = 2  one thread: mbarrier init + expect_tx + TMA 2D boxes per panel;
//              bounded try_wait (trap on timeout); windows from the panels
//   UNR = 1    every (input row, tap, column) FMA unrolled; with CF2 and even
//              YWPT output rows are paired into fma.rn.f32x2 with tap pairs
//              from c_tpair, edge tap rows scalar -- conv.cu's order exactly
//   UNR = 0    rolled tap loops (runtime tap index into c_taps)
//   epilogue   out = W * acc, vector stores, GUARD predicates for ragged tiles
#include <algorithm>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "compile_service.hpp"

namespace ktc {

namespace {

struct ConvGen {
    int FS = 0, XWG = 0, YWG = 0, XWPT = 0, YWPT = 0, LOCAL = 0, VW = 1, PAD = 0, UNR = 1;
    int GUARD = 0, OUT_VEC = 1, CF2 = 1, MINCTA = 1, TRACE = 0;
    int SP = 0, PWO = 0, BW = 0, BH = 0, NB = 0, NP = 0, PF = 0;
};

long long def_value(const Defines& ds, const char* name, bool required, long long fallback = 0) {
    const std::string key = std::string(name) + "=";
    for (const std::string& d : ds)
        if (d.compare(0, key.size(), key) == 0) return std::stoll(d.substr(key.size()));
    if (required) throw std::runtime_error(std::string("ptxgen: missing define ") + name);
    return fallback;
}

ConvGen parse(const Defines& problem, const Defines& c) {
    ConvGen g;
    g.FS = int(def_value(problem, "FS", true));
    g.XWG = int(def_value(c, "XWG", true));
    g.YWG = int(def_value(c, "YWG", true));
    g.XWPT = int(def_value(c, "XWPT", true));
    g.YWPT = int(def_value(c, "YWPT", true));
    g.LOCAL = int(def_value(c, "LOCAL", true));
    g.VW = int(def_value(c, "VW", true));
    g.PAD = int(def_value(c, "PAD", true));
    g.UNR = int(def_value(c, "UNR", true));
    g.GUARD = int(def_value(c, "GUARD", false, 0));
    g.OUT_VEC = int(def_value(c, "OUT_VEC", false, 1));
    g.CF2 = int(def_value(c, "CF2", false, 1));
    g.MINCTA = int(def_value(c, "MINCTA", false, 1));
    g.TRACE = int(def_value(c, "TRACE", false, 0));
    if (g.LOCAL == 1) g.SP = int(def_value(c, "SP", true));
    if (g.LOCAL == 2) {
        g.PWO = int(def_value(c, "PWO", true));
        g.BW = int(def_value(c, "BW", true));
        g.BH = int(def_value(c, "BH", true));
        g.NB = int(def_value(c, "NB", true));
        g.NP = int(def_value(c, "NP", true));
        g.PF = int(def_value(c, "PF", true));
    }
    return g;
}

int log2i(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

// Register and label allocation plus instruction text.
class Ptx {
  public:
    std::string f() { return "%f" + std::to_string(nf_++); }
    std::string r() { return "%r" + std::to_string(nr_++); }
    std::string d() { return "%rd" + std::to_string(nd_++); }
    std::string p() { return "%p" + std::to_string(np_++); }
    std::string label() { return "$L_" + std::to_string(nl_++); }
    void op(const std::string& s) { b_ << "\t" << s << ";\n"; }
    void lab(const std::string& l) { b_ << l << ":\n"; }
    std::string decls() const {
        std::ostringstream s;
        s << "\t.reg .pred %p<" << (np_ + 1) << ">;\n\t.reg .b32 %r<" << (nr_ + 1)
          << ">;\n\t.reg .f32 %f<" << (nf_ + 1) << ">;\n\t.reg .b64 %rd<" << (nd_ + 1) << ">;\n";
        return s.str();
    }
    std::string body() const { return b_.str(); }

  private:
    std::ostringstream b_;
    int nf_ = 0, nr_ = 0, nd_ = 0, np_ = 0, nl_ = 0;
};

std::string imm(long long v) { return std::to_string(v); }

// Vector load of n floats (1, 2, 4 or 8) from [addr + off] in `space`.
void vload(Ptx& x, const char* space, const std::string& addr, long long off,
           const std::vector<std::string>& dst) {
    const int n = int(dst.size());
    auto at = [&](long long o) { return "[" + addr + "+" + imm(o) + "]"; };
    if (n == 1) {
        x.op(std::string("ld.") + space + ".f32 " + dst[0] + ", " + at(off));
    } else if (n == 2) {
        x.op(std::string("ld.") + space + ".v2.f32 {" + dst[0] + ", " + dst[1] + "}, " + at(off));
    } else {
        for (int q = 0; q < n; q += 4)
            x.op(std::string("ld.") + space + ".v4.f32 {" + dst[q] + ", " + dst[q + 1] + ", " +
                 dst[q + 2] + ", " + dst[q + 3] + "}, " + at(off + 4 * q));
    }
}

std::string emit_entry(const ConvGen& g, const std::string& name) {
    const int H = (g.FS - 1) / 2, TX = g.XWG * g.XWPT, TY = g.YWG * g.YWPT, NG = g.XWPT / g.VW,
              NT = g.XWG * g.YWG;
    auto pow2_div = [](int v) { return v % 4 == 0 ? 4 : (v % 2 == 0 ? 2 : 1); };
    const int SVW = g.LOCAL == 0   ? g.VW
                    : g.LOCAL == 1 ? std::min(g.VW, pow2_div(g.SP))
                                   : std::min(g.VW, 4);
    const int WIN = g.VW + g.FS - 1;
    const int NWV = (WIN + SVW - 1) / SVW;
    const int WINP = NWV * SVW;
    const int ROWS = g.YWPT + g.FS - 1;

    Ptx x;
    const std::string P = name + "_param_";
    // ---- prologue
    const std::string rX = x.r(), rY = x.r(), rP = x.r(), fW = x.f();
    const std::string dImg = x.d(), dOut = x.d();
    x.op("ld.param.u32 " + rX + ", [" + P + "0]");
    x.op("ld.param.u32 " + rY + ", [" + P + "1]");
    x.op("ld.param.f32 " + fW + ", [" + P + "2]");
    x.op("ld.param.u64 " + dImg + ", [" + P + "3]");
    x.op("ld.param.u32 " + rP + ", [" + P + "4]");
    x.op("ld.param.u64 " + dOut + ", [" + P + "5]");
    x.op("cvta.to.global.u64 " + dImg + ", " + dImg);
    x.op("cvta.to.global.u64 " + dOut + ", " + dOut);
    const std::string tx = x.r(), ty = x.r(), cx = x.r(), cy = x.r(), x0 = x.r(), y0 = x.r();
    x.op("mov.u32 " + tx + ", %tid.x");
    x.op("mov.u32 " + ty + ", %tid.y");
    x.op("mov.u32 " + cx + ", %ctaid.x");
    x.op("mov.u32 " + cy + ", %ctaid.y");
    // TRACE (diagnostic build, KTC_CONV_TRACE): thread (0,0) records the
    // CTA's start and end %globaltimer and its SM in trace[4 * linear_cta].
    std::string trace_slot, trace_t0, trace_lead;
    if (g.TRACE) {
        trace_slot = x.d();
        trace_t0 = x.d();
        trace_lead = x.p();
        const std::string lin = x.r(), nx = x.r(), o = x.r(), tb = x.d(), t = x.r();
        x.op("mov.u32 " + nx + ", %nctaid.x");
        x.op("mad.lo.u32 " + lin + ", " + cy + ", " + nx + ", " + cx);
        x.op("ld.param.u64 " + tb + ", [" + P + "7]");
        x.op("cvta.to.global.u64 " + tb + ", " + tb);
        x.op("mul.wide.u32 " + trace_slot + ", " + lin + ", 32");
        x.op("add.u64 " + trace_slot + ", " + trace_slot + ", " + tb);
        x.op("or.b32 " + t + ", " + tx + ", " + ty);
        x.op("setp.eq.u32 " + trace_lead + ", " + t + ", 0");
        x.op("mov.u64 " + trace_t0 + ", %globaltimer");
        (void)o;
    }
    x.op("mul.lo.u32 " + x0 + ", " + cx + ", " + imm(TX));
    x.op("mul.lo.u32 " + y0 + ", " + cy + ", " + imm(TY));
    // Column of group gi (floats, relative to the tile): (gi*XWG + tx) * VW.
    std::vector<std::string> colf(static_cast<size_t>(NG));  // u32 float index
    for (int gi = 0; gi < NG; ++gi) {
        colf[size_t(gi)] = x.r();
        x.op("mad.lo.u32 " + colf[size_t(gi)] + ", " + tx + ", " + imm(g.VW) + ", " +
             imm(gi * g.XWG * g.VW));
    }

    // ---- staging: row base addresses and column byte offsets
    const char* space = g.LOCAL == 0 ? "global.nc" : "shared";
    std::vector<std::string> colb(static_cast<size_t>(NG));  // byte offset of the group's window start
    std::string rowbase;                        // address of window row 0 (u64 global / u32 shared)
    long long row_stride_imm = 0;               // shared: bytes per window row
    std::string row_stride_reg;                 // global: bytes per image row (u64)
    std::string sbase;                          // shared base (u32)
    if (g.LOCAL == 0) {
        const std::string row = x.r(), d1 = x.d(), d2 = x.d();
        x.op("mad.lo.u32 " + row + ", " + ty + ", " + imm(g.YWPT) + ", " + y0);
        x.op("mul.wide.u32 " + d1 + ", " + row + ", " + rP);
        x.op("cvt.u64.u32 " + d2 + ", " + x0);
        x.op("add.u64 " + d1 + ", " + d1 + ", " + d2);
        x.op("shl.b64 " + d1 + ", " + d1 + ", 2");
        rowbase = x.d();
        x.op("add.u64 " + rowbase + ", " + dImg + ", " + d1);
        row_stride_reg = x.d();
        x.op("mul.wide.u32 " + row_stride_reg + ", " + rP + ", 4");
        for (int gi = 0; gi < NG; ++gi) {
            colb[size_t(gi)] = x.d();
            x.op("mul.wide.u32 " + colb[size_t(gi)] + ", " + colf[size_t(gi)] + ", 4");
        }
    } else {
        const std::string d = x.d();
        sbase = x.r();
        x.op("mov.u64 " + d + ", smem");
        x.op("cvt.u32.u64 " + sbase + ", " + d);
    }

    if (g.LOCAL == 1) {
        // Cooperative halo-tile copy, TR rows x TC4 float4s, unrolled.
        const int TR = TY + 2 * H, TC4 = (TX + 2 * H + 3) / 4, TOT = TR * TC4, WIDTH = TX + 2 * H;
        const std::string tid = x.r(), gb = x.d();
        x.op("mad.lo.u32 " + tid + ", " + ty + ", " + imm(g.XWG) + ", " + tx);
        {
            const std::string d1 = x.d(), d2 = x.d();
            x.op("mul.wide.u32 " + d1 + ", " + y0 + ", " + rP);
            x.op("cvt.u64.u32 " + d2 + ", " + x0);
            x.op("add.u64 " + d1 + ", " + d1 + ", " + d2);
            x.op("shl.b64 " + d1 + ", " + d1 + ", 2");
            x.op("add.u64 " + gb + ", " + dImg + ", " + d1);
        }
        // conv.cu's `#pragma unroll 4` loop: up to four guarded copies per
        // trip of a rolled loop (four loads in flight, bounded code size).
        const int iters = (TOT + NT - 1) / NT;
        const int U = std::min(iters, 4);
        const std::string base_e = x.r();
        x.op("mov.u32 " + base_e + ", " + tid);
        const std::string top = x.label(), out = x.label();
        const bool looped = iters > U;
        if (looped) x.lab(top);
        for (int u = 0; u < U; ++u) {
            const std::string skip = x.label();
            const std::string e = x.r();
            x.op("add.u32 " + e + ", " + base_e + ", " + imm((long long)u * NT));
            if (looped || (long long)(u + 1) * NT > TOT) {
                const std::string pe = x.p();
                x.op("setp.ge.u32 " + pe + ", " + e + ", " + imm(TOT));
                x.op("@" + pe + " bra " + skip);
            }
            const std::string rr = x.r(), c4 = x.r(), c = x.r();
            x.op("div.u32 " + rr + ", " + e + ", " + imm(TC4));
            x.op("mul.lo.u32 " + c4 + ", " + rr + ", " + imm(TC4));
            x.op("sub.u32 " + c4 + ", " + e + ", " + c4);
            x.op("shl.b32 " + c + ", " + c4 + ", 2");
            const std::string ga = x.d(), d2 = x.d();
            x.op("mul.wide.u32 " + ga + ", " + rr + ", " + rP);
            x.op("cvt.u64.u32 " + d2 + ", " + c);
            x.op("add.u64 " + ga + ", " + ga + ", " + d2);
            x.op("shl.b64 " + ga + ", " + ga + ", 2");
            x.op("add.u64 " + ga + ", " + gb + ", " + ga);
            std::vector<std::string> v = {x.f(), x.f(), x.f(), x.f()};
            vload(x, "global.nc", ga, 0, v);
            const std::string sa = x.r();
            x.op("mad.lo.u32 " + sa + ", " + rr + ", " + imm(g.SP) + ", " + c);
            x.op("shl.b32 " + sa + ", " + sa + ", 2");
            x.op("add.u32 " + sa + ", " + sa + ", " + sbase);
            const std::string pfull = x.p();
            x.op("setp.le.u32 " + pfull + ", " + c + ", " + imm(WIDTH - 4));
            const std::string partial = x.label(), done = x.label();
            if (g.SP % 4 == 0 || g.SP % 2 == 0) {
                x.op("@!" + pfull + " bra " + partial);
                if (g.SP % 4 == 0) {
                    x.op("st.shared.v4.f32 [" + sa + "], {" + v[0] + ", " + v[1] + ", " + v[2] +
                         ", " + v[3] + "}");
                } else {
                    x.op("st.shared.v2.f32 [" + sa + "], {" + v[0] + ", " + v[1] + "}");
                    x.op("st.shared.v2.f32 [" + sa + "+8], {" + v[2] + ", " + v[3] + "}");
                }
                x.op("bra.uni " + done);
            }
            x.lab(partial);
            for (int q = 0; q < 4; ++q) {
                const std::string pq = x.p();
                x.op("setp.lt.u32 " + pq + ", " + c + ", " + imm(WIDTH - q));
                x.op("@" + pq + " st.shared.f32 [" + sa + "+" + imm(4 * q) + "], " + v[size_t(q)]);
            }
            x.lab(done);
            x.lab(skip);
        }
        if (looped) {
            const std::string pl = x.p();
            x.op("add.u32 " + base_e + ", " + base_e + ", " + imm((long long)U * NT));
            x.op("setp.lt.u32 " + pl + ", " + base_e + ", " + imm(TOT));
            x.op("@" + pl + " bra " + top);
        }
        x.lab(out);
        x.op("bar.sync 0");
        rowbase = x.r();
        x.op("mad.lo.u32 " + rowbase + ", " + ty + ", " + imm((long long)g.YWPT * g.SP * 4) + ", " +
             sbase);
        row_stride_imm = (long long)g.SP * 4;
        for (int gi = 0; gi < NG; ++gi) {
            colb[size_t(gi)] = x.r();
            x.op("shl.b32 " + colb[size_t(gi)] + ", " + colf[size_t(gi)] + ", 2");
        }
    } else if (g.LOCAL == 2) {
        const std::string bar = x.r();
        x.op("add.u32 " + bar + ", " + sbase + ", " + imm((long long)g.NP * g.PF * 4));
        const std::string pz = x.p(), t = x.r(), after = x.label();
        x.op("or.b32 " + t + ", " + tx + ", " + ty);
        x.op("setp.ne.u32 " + pz + ", " + t + ", 0");
        x.op("@" + pz + " bra " + after);
        x.op("mbarrier.init.shared::cta.b64 [" + bar + "], 1");
        x.op("fence.mbarrier_init.release.cluster");
        const std::string bytes = x.r();
        x.op("mov.u32 " + bytes + ", " + imm((long long)g.NP * g.NB * g.BW * g.BH * 4));
        x.op("mbarrier.arrive.expect_tx.shared::cta.b64 _, [" + bar + "], " + bytes);
        const std::string tm = x.d();
        x.op("mov.b64 " + tm + ", " + P + "6");
        x.op("cvta.param.u64 " + tm + ", " + tm);
        for (int pnl = 0; pnl < g.NP; ++pnl)
            for (int b = 0; b < g.NB; ++b) {
                const std::string dst = x.r(), xc = x.r(), yc = x.r();
                x.op("add.u32 " + dst + ", " + sbase + ", " +
                     imm(((long long)pnl * g.PF + (long long)b * g.BH * g.BW) * 4));
                x.op("add.u32 " + xc + ", " + x0 + ", " + imm((long long)pnl * g.PWO));
                x.op("add.u32 " + yc + ", " + y0 + ", " + imm((long long)b * g.BH));
                x.op("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [" +
                     dst + "], [" + tm + ", {" + xc + ", " + yc + "}], [" + bar + "]");
            }
        x.lab(after);
        x.op("bar.sync 0");
        // Bounded wait (a lost transaction traps -> runtime_error, never a hang).
        const std::string spin = x.d(), lw = x.label(), ld = x.label(), pd = x.p(), pc = x.p();
        x.op("mov.u64 " + spin + ", 0");
        x.lab(lw);
        x.op("mbarrier.try_wait.parity.shared::cta.b64 " + pd + ", [" + bar + "], 0");
        x.op("@" + pd + " bra " + ld);
        x.op("add.u64 " + spin + ", " + spin + ", 1");
        x.op("setp.lt.u64 " + pc + ", " + spin + ", " + imm(1ll << 26));
        x.op("@" + pc + " bra " + lw);
        x.op("trap");
        x.lab(ld);
        rowbase = x.r();
        x.op("mad.lo.u32 " + rowbase + ", " + ty + ", " + imm((long long)g.YWPT * g.BW * 4) + ", " +
             sbase);
        row_stride_imm = (long long)g.BW * 4;
        const int lp = log2i(g.PWO);
        for (int gi = 0; gi < NG; ++gi) {
            // COLOFF(col) = (col / PWO) * PF + col % PWO, in bytes.
            const std::string q = x.r(), m = x.r(), o = x.r();
            x.op("shr.u32 " + q + ", " + colf[size_t(gi)] + ", " + imm(lp));
            x.op("and.b32 " + m + ", " + colf[size_t(gi)] + ", " + imm(g.PWO - 1));
            x.op("mad.lo.u32 " + o + ", " + q + ", " + imm(g.PF) + ", " + m);
            x.op("shl.b32 " + o + ", " + o + ", 2");
            colb[size_t(gi)] = o;
        }
    }

    // Address of window row r for group gi (+ byte offset applied by loads).
    auto window_addr = [&](int gi, int rrow) -> std::string {
        if (g.LOCAL == 0) {
            const std::string a = x.d();
            if (rrow == 0) {
                x.op("add.u64 " + a + ", " + rowbase + ", " + colb[size_t(gi)]);
            } else {
                x.op("mad.lo.u64 " + a + ", " + row_stride_reg + ", " + imm(rrow) + ", " + rowbase);
                x.op("add.u64 " + a + ", " + a + ", " + colb[size_t(gi)]);
            }
            return a;
        }
        const std::string a = x.r();
        x.op("add.u32 " + a + ", " + rowbase + ", " + colb[size_t(gi)]);
        if (rrow) x.op("add.u32 " + a + ", " + a + ", " + imm(rrow * row_stride_imm));
        return a;
    };

    // ---- accumulators
    std::vector<std::vector<std::string>> acc(size_t(g.YWPT), std::vector<std::string>(size_t(g.XWPT)));
    for (auto& row : acc)
        for (auto& a : row) {
            a = x.f();
            x.op("mov.f32 " + a + ", 0f00000000");
        }

    if (g.UNR == 1) {
        const bool paired = g.CF2 && g.YWPT % 2 == 0;
        // .b64 register of row pair (2p, 2p+1), column c while packed ("" = unpacked)
        std::vector<std::vector<std::string>> accp(size_t(g.YWPT / 2 + 1),
                                                   std::vector<std::string>(size_t(g.XWPT)));
        for (int gi = 0; gi < NG; ++gi) {
            for (int rr = 0; rr < ROWS; ++rr) {
                const std::string a = window_addr(gi, rr);
                std::vector<std::string> w(static_cast<size_t>(WINP));
                for (auto& v : w) v = x.f();
                for (int v = 0; v < NWV; ++v) {
                    std::vector<std::string> part(w.begin() + v * SVW, w.begin() + (v + 1) * SVW);
                    vload(x, space, a, (long long)v * SVW * 4, part);
                }
                auto scalar_row = [&](int j, int jj) {
                    for (int i = 0; i < g.FS; ++i) {
                        const std::string t = x.f();
                        x.op("ld.const.f32 " + t + ", [c_taps+" + imm((jj * g.FS + i) * 4) + "]");
                        for (int e = 0; e < g.VW; ++e) {
                            const std::string& ac = acc[size_t(j)][size_t(gi * g.VW + e)];
                            x.op("fma.rn.f32 " + ac + ", " + t + ", " + w[size_t(e + i)] + ", " + ac);
                        }
                    }
                };
                if (paired) {
                    // Row pairs live in .b64 registers while they take FFMA2s:
                    // packed once after row j's leading edge tap row (jj = 0),
                    // unpacked once before row j+1's trailing one (jj = FS-1),
                    // and each window value is broadcast to a pair once per
                    // input row -- the same FMA sequence per output as one
                    // pack / fma / unpack per FFMA2, with a third of the PTX.
                    std::vector<std::string> wb(static_cast<size_t>(WINP));
                    auto bcast = [&](int k) -> const std::string& {
                        std::string& r = wb[size_t(k)];
                        if (r.empty()) {
                            r = x.d();
                            x.op("mov.b64 " + r + ", {" + w[size_t(k)] + ", " + w[size_t(k)] + "}");
                        }
                        return r;
                    };
                    for (int j = 0; j < g.YWPT; j += 2) {
                        const int jj = rr - j;
                        if (jj >= 1 && jj < g.FS) {
                            for (int e = 0; e < g.VW; ++e) {
                                std::string& pr = accp[size_t(j / 2)][size_t(gi * g.VW + e)];
                                if (pr.empty()) {
                                    pr = x.d();
                                    x.op("mov.b64 " + pr + ", {" + acc[size_t(j)][size_t(gi * g.VW + e)] +
                                         ", " + acc[size_t(j + 1)][size_t(gi * g.VW + e)] + "}");
                                }
                            }
                            for (int i = 0; i < g.FS; ++i) {
                                const std::string t2 = x.d();
                                x.op("ld.const.b64 " + t2 + ", [c_tpair+" + imm((jj * g.FS + i) * 8) + "]");
                                for (int e = 0; e < g.VW; ++e) {
                                    const std::string& pr = accp[size_t(j / 2)][size_t(gi * g.VW + e)];
                                    x.op("fma.rn.f32x2 " + pr + ", " + t2 + ", " + bcast(e + i) + ", " + pr);
                                }
                            }
                        } else if (jj == 0) {
                            scalar_row(j, 0);
                        } else if (jj == g.FS) {
                            for (int e = 0; e < g.VW; ++e) {
                                std::string& pr = accp[size_t(j / 2)][size_t(gi * g.VW + e)];
                                if (!pr.empty()) {
                                    x.op("mov.b64 {" + acc[size_t(j)][size_t(gi * g.VW + e)] + ", " +
                                         acc[size_t(j + 1)][size_t(gi * g.VW + e)] + "}, " + pr);
                                    pr.clear();
                                }
                            }
                            scalar_row(j + 1, g.FS - 1);
                        }
                    }
                } else {
                    for (int j = 0; j < g.YWPT; ++j) {
                        const int jj = rr - j;
                        if (jj >= 0 && jj < g.FS) scalar_row(j, jj);
                    }
                }
            }
        }
    } else {
        // Rolled filter loops: jj outer, i inner (runtime), one load per FMA.
        const std::string jj = x.r(), ii = x.r(), taps = x.d();
        x.op("mov.u64 " + taps + ", c_taps");
        x.op("mov.u32 " + jj + ", 0");
        const std::string ljj = x.label(), lii = x.label();
        // UNR = 0 means rolled: keep ptxas from unrolling the constant-trip
        // tap loops (conv.cu's #pragma unroll 1).
        x.lab(ljj);
        x.op(".pragma \"nounroll\"");
        x.op("mov.u32 " + ii + ", 0");
        x.lab(lii);
        x.op(".pragma \"nounroll\"");
        const std::string tidx = x.r(), toff = x.d(), tad = x.d(), t = x.f();
        x.op("mad.lo.u32 " + tidx + ", " + jj + ", " + imm(g.FS) + ", " + ii);
        x.op("mul.wide.u32 " + toff + ", " + tidx + ", 4");
        x.op("add.u64 " + tad + ", " + taps + ", " + toff);
        x.op("ld.const.f32 " + t + ", [" + tad + "]");
        for (int j = 0; j < g.YWPT; ++j) {
            // row (j + jj) of the window, column offset + i
            const std::string rowsel = x.r();
            x.op("add.u32 " + rowsel + ", " + jj + ", " + imm(j));
            for (int gi = 0; gi < NG; ++gi) {
                std::string a;
                if (g.LOCAL == 0) {
                    const std::string d1 = x.d(), d2 = x.d();
                    a = x.d();
                    x.op("mul.wide.u32 " + d1 + ", " + rowsel + ", " + rP);
                    x.op("shl.b64 " + d1 + ", " + d1 + ", 2");
                    x.op("add.u64 " + d1 + ", " + d1 + ", " + rowbase);
                    x.op("mul.wide.u32 " + d2 + ", " + ii + ", 4");
                    x.op("add.u64 " + d2 + ", " + d2 + ", " + colb[size_t(gi)]);
                    x.op("add.u64 " + a + ", " + d1 + ", " + d2);
                } else {
                    const std::string o = x.r();
                    a = x.r();
                    x.op("mad.lo.u32 " + o + ", " + rowsel + ", " + imm(row_stride_imm) + ", " + rowbase);
                    x.op("add.u32 " + o + ", " + o + ", " + colb[size_t(gi)]);
                    x.op("mad.lo.u32 " + a + ", " + ii + ", 4, " + o);
                }
                for (int e = 0; e < g.VW; ++e) {
                    const std::string v = x.f();
                    x.op(std::string("ld.") + space + ".f32 " + v + ", [" + a + "+" + imm(4 * e) + "]");
                    const std::string& ac = acc[size_t(j)][size_t(gi * g.VW + e)];
                    x.op("fma.rn.f32 " + ac + ", " + t + ", " + v + ", " + ac);
                }
            }
        }
        const std::string pi = x.p(), pj = x.p();
        x.op("add.u32 " + ii + ", " + ii + ", 1");
        x.op("setp.lt.u32 " + pi + ", " + ii + ", " + imm(g.FS));
        x.op("@" + pi + " bra " + lii);
        x.op("add.u32 " + jj + ", " + jj + ", 1");
        x.op("setp.lt.u32 " + pj + ", " + jj + ", " + imm(g.FS));
        x.op("@" + pj + " bra " + ljj);
    }

    // ---- epilogue: out = W * acc
    for (int j = 0; j < g.YWPT; ++j) {
        const std::string row = x.r(), next = x.label();
        x.op("mad.lo.u32 " + row + ", " + ty + ", " + imm(g.YWPT) + ", " + y0);
        if (j) x.op("add.u32 " + row + ", " + row + ", " + imm(j));
        if (g.GUARD) {
            const std::string pr = x.p();
            x.op("setp.ge.s32 " + pr + ", " + row + ", " + rY);
            x.op("@" + pr + " bra " + next);
        }
        const std::string ob = x.d(), d2 = x.d();
        x.op("mul.wide.u32 " + ob + ", " + row + ", " + rX);
        x.op("cvt.u64.u32 " + d2 + ", " + x0);
        x.op("add.u64 " + ob + ", " + ob + ", " + d2);
        x.op("shl.b64 " + ob + ", " + ob + ", 2");
        x.op("add.u64 " + ob + ", " + ob + ", " + dOut);
        for (int gi = 0; gi < NG; ++gi) {
            std::vector<std::string> s(static_cast<size_t>(g.VW));
            for (int e = 0; e < g.VW; ++e) {
                s[size_t(e)] = x.f();
                x.op("mul.f32 " + s[size_t(e)] + ", " + fW + ", " + acc[size_t(j)][size_t(gi * g.VW + e)]);
            }
            const std::string cb = x.d(), a = x.d();
            x.op("mul.wide.u32 " + cb + ", " + colf[size_t(gi)] + ", 4");
            x.op("add.u64 " + a + ", " + ob + ", " + cb);
            const std::string vec = x.label(), gdone = x.label();
            auto store_vec = [&]() {
                if (g.OUT_VEC) {
                    if (g.VW == 1) {
                        x.op("st.global.f32 [" + a + "], " + s[0]);
                    } else if (g.VW == 2) {
                        x.op("st.global.v2.f32 [" + a + "], {" + s[0] + ", " + s[1] + "}");
                    } else {
                        for (int q = 0; q < g.VW; q += 4)
                            x.op("st.global.v4.f32 [" + a + "+" + imm(4 * q) + "], {" + s[size_t(q)] +
                                 ", " + s[size_t(q + 1)] + ", " + s[size_t(q + 2)] + ", " +
                                 s[size_t(q + 3)] + "}");
                    }
                } else {
                    for (int e = 0; e < g.VW; ++e)
                        x.op("st.global.f32 [" + a + "+" + imm(4 * e) + "], " + s[size_t(e)]);
                }
            };
            if (g.GUARD) {
                // Ragged right edge: x0 + col + VW > X -> per-element guarded stores.
                const std::string xe = x.r(), lim = x.r(), pfull = x.p();
                x.op("add.u32 " + xe + ", " + x0 + ", " + colf[size_t(gi)]);
                x.op("sub.s32 " + lim + ", " + rX + ", " + imm(g.VW));
                x.op("setp.le.s32 " + pfull + ", " + xe + ", " + lim);
                x.op("@" + pfull + " bra " + vec);
                for (int e = 0; e < g.VW; ++e) {
                    const std::string pe = x.p(), xi = x.r();
                    x.op("add.u32 " + xi + ", " + xe + ", " + imm(e));
                    x.op("setp.lt.s32 " + pe + ", " + xi + ", " + rX);
                    x.op("@" + pe + " st.global.f32 [" + a + "+" + imm(4 * e) + "], " + s[size_t(e)]);
                }
                x.op("bra.uni " + gdone);
            }
            x.lab(vec);
            store_vec();
            x.lab(gdone);
        }
        x.lab(next);
    }
    if (g.TRACE) {
        const std::string t1 = x.d(), sm = x.r(), sm64 = x.d();
        x.op("bar.sync 0");
        x.op("mov.u64 " + t1 + ", %globaltimer");
        x.op("mov.u32 " + sm + ", %smid");
        x.op("cvt.u64.u32 " + sm64 + ", " + sm);
        x.op("@" + trace_lead + " st.global.v2.u64 [" + trace_slot + "], {" + trace_t0 + ", " + t1 + "}");
        x.op("@" + trace_lead + " st.global.u64 [" + trace_slot + "+16], " + sm64);
    }
    x.op("ret");

    std::ostringstream e;
    e << ".visible .entry " << name << "(\n"
      << "\t.param .u32 " << P << "0,\n\t.param .u32 " << P << "1,\n\t.param .f32 " << P
      << "2,\n\t.param .u64 .ptr .align 1 " << P << "3,\n\t.param .u32 " << P
      << "4,\n\t.param .u64 .ptr .align 1 " << P << "5,\n\t.param .align 64 .b8 " << P
      << "6[128]" << (g.TRACE ? std::string(",\n\t.param .u64 ") + P + "7" : std::string())
      << "\n)\n.maxntid " << NT << ", 1, 1\n.minnctapersm " << g.MINCTA << "\n{\n"
      << x.decls() << x.body() << "}\n";
    return e.str();
}

}  // namespace

std::string conv_ptx_module(const Defines& problem, const std::vector<const Defines*>& configs,
                            const std::string& entry_base) {
    const int FS = int(def_value(problem, "FS", true));
    std::ostringstream m;
    m << "//\n// Generated by libktc ptxgen_conv (conv.cu semantics)\n//\n"
      << ".version 8.8\n.target sm_100a\n.address_size 64\n\n"
      << ".const .align 4 .b8 c_taps[" << FS * FS * 4 << "];\n"
      << ".const .align 8 .b8 c_tpair[" << FS * FS * 8 << "];\n"
      << ".extern .shared .align 128 .b8 smem[];\n\n";
    for (size_t i = 0; i < configs.size(); ++i)
        m << emit_entry(parse(problem, *configs[i]), entry_base + "_k" + std::to_string(i)) << "\n";
    return m.str();
}

}  // namespace ktc
