// ptxgen_gemm.cpp -- direct PTX generation for the SGEMM family.
//
// Emits, for one configuration, the kernel kernels/gemm.cu describes (CLTune
// semantics of MWG/NWG/KWG, MDIMC/NDIMC, MDIMA/NDIMB, KWI, VWM/VWN, STRM/STRN,
// SA/SB, plus the host switches DBUF / OCC / F2) as PTX, so
// the tuning-time compile is ptxas only.  Same memory traffic, same
// per-output FMA order (k ascending; alpha*acc, or gemm.cu's explicit
// fmaf(alpha, acc, beta*c)) -> outputs bit-identical to the NVRTC build
// (tests/test_gpu_ptxgen.py).
//
//   prologue  DBUF: cp.async of K-tile 0 into buffer 0 | register staging:
//             ld.global.nc of K-tile 0
//   k0 loop   (rolled) DBUF: wait_group 0, bar.sync, cp.async of the next
//             K-tile into the other buffer | stash to shared, bar.sync,
//             next tile's loads issued early when the staging registers are
//             few (STAGE_AHEAD), else after the compute
//   kw loop   (rolled, KWG/KWI trips) of KWI unrolled k-steps: MWI x NWI
//             register outer product from shared (SA/SB) or global memory,
//             packed fma.rn.f32x2 pairs (F2)
//   epilogue  alpha/beta, VWN-wide stores along N
#include <algorithm>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "compile_service.hpp"

namespace ktc {

namespace {

long long dv(const Defines& ds, const char* name, bool required, long long fallback = 0) {
    const std::string key = std::string(name) + "=";
    for (const std::string& d : ds)
        if (d.compare(0, key.size(), key) == 0) return std::stoll(d.substr(key.size()));
    if (required) throw std::runtime_error(std::string("ptxgen: missing define ") + name);
    return fallback;
}

struct GemmGen {
    int MWG, NWG, KWG, MDIMC, NDIMC, SA, SB, MDIMA, NDIMB, STRM, STRN, VWM, VWN, KWI;
    int DBUF, OCC, F2, TAILK, SK;
};

GemmGen parse(const Defines& c) {
    GemmGen g;
    g.MWG = int(dv(c, "MWG", true));
    g.NWG = int(dv(c, "NWG", true));
    g.KWG = int(dv(c, "KWG", true));
    g.MDIMC = int(dv(c, "MDIMC", true));
    g.NDIMC = int(dv(c, "NDIMC", true));
    g.SA = int(dv(c, "SA", true));
    g.SB = int(dv(c, "SB", true));
    g.MDIMA = int(dv(c, "MDIMA", true));
    g.NDIMB = int(dv(c, "NDIMB", true));
    g.STRM = int(dv(c, "STRM", true));
    g.STRN = int(dv(c, "STRN", true));
    g.VWM = int(dv(c, "VWM", true));
    g.VWN = int(dv(c, "VWN", true));
    g.KWI = int(dv(c, "KWI", true));
    g.DBUF = int(dv(c, "DBUF", false, 0));
    g.OCC = int(dv(c, "OCC", false, 0));
    g.F2 = int(dv(c, "F2", false, 1));
    g.TAILK = int(dv(c, "TAILK", false, 0));
    g.SK = g.TAILK ? 0 : int(dv(c, "SK", false, 0));
    return g;
}

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

std::string at(const std::string& a, long long off) { return "[" + a + "+" + imm(off) + "]"; }

// n floats (1, 2, 4, 8) from [addr + off] in `space` into dst.
void vld(Ptx& x, const std::string& space, const std::string& addr, long long off,
         const std::vector<std::string>& dst) {
    const int n = int(dst.size());
    if (n == 1) {
        x.op("ld." + space + ".f32 " + dst[0] + ", " + at(addr, off));
    } else if (n == 2) {
        x.op("ld." + space + ".v2.f32 {" + dst[0] + ", " + dst[1] + "}, " + at(addr, off));
    } else {
        for (int q = 0; q < n; q += 4)
            x.op("ld." + space + ".v4.f32 {" + dst[size_t(q)] + ", " + dst[size_t(q + 1)] + ", " +
                 dst[size_t(q + 2)] + ", " + dst[size_t(q + 3)] + "}, " + at(addr, off + 4 * q));
    }
}

void vst(Ptx& x, const std::string& space, const std::string& addr, long long off,
         const std::vector<std::string>& src) {
    const int n = int(src.size());
    if (n == 1) {
        x.op("st." + space + ".f32 " + at(addr, off) + ", " + src[0]);
    } else if (n == 2) {
        x.op("st." + space + ".v2.f32 " + at(addr, off) + ", {" + src[0] + ", " + src[1] + "}");
    } else {
        for (int q = 0; q < n; q += 4)
            x.op("st." + space + ".v4.f32 " + at(addr, off + 4 * q) + ", {" + src[size_t(q)] + ", " +
                 src[size_t(q + 1)] + ", " + src[size_t(q + 2)] + ", " + src[size_t(q + 3)] + "}");
    }
}

// One operand's shared-memory copy geometry (gemm.cu SA/SB blocks).
struct Copy {
    bool on = false;
    int DIM = 0, KD = 0, KW = 0, V = 0, MV = 0, VW = 0, WG = 0, STR = 0;
    std::string l0, l1;    // thread re-shape coordinates
    std::string copies;    // predicate register name ("" = always)
    long long sm_off = 0;  // byte offset of this operand's tiles in smem
};

std::string emit_entry(const GemmGen& g, const std::string& name) {
    const int MWI = g.MWG / g.MDIMC, NWI = g.NWG / g.NDIMC, NT = g.MDIMC * g.NDIMC;
    const int MVI = MWI / g.VWM, NVI = NWI / g.VWN;
    Copy ca, cb;
    ca.on = g.SA != 0;
    cb.on = g.SB != 0;
    if (ca.on) {
        ca.DIM = g.MDIMA;
        ca.KD = NT / g.MDIMA;
        ca.KW = g.KWG / ca.KD;
        ca.V = g.MWG / g.VWM;
        ca.MV = ca.V >= ca.DIM ? ca.V / ca.DIM : 1;
        ca.VW = g.VWM;
        ca.WG = g.MWG;
        ca.STR = g.STRM;
        ca.sm_off = 0;
    }
    if (cb.on) {
        cb.DIM = g.NDIMB;
        cb.KD = NT / g.NDIMB;
        cb.KW = g.KWG / cb.KD;
        cb.V = g.NWG / g.VWN;
        cb.MV = cb.V >= cb.DIM ? cb.V / cb.DIM : 1;
        cb.VW = g.VWN;
        cb.WG = g.NWG;
        cb.STR = g.STRN;
        cb.sm_off = (long long)g.SA * (1 + g.DBUF) * g.KWG * g.MWG * 4;
    }
    const int STAGE_A = ca.on ? ca.KW * ca.MV * ca.VW : 0;
    const int STAGE_B = cb.on ? cb.KW * cb.MV * cb.VW : 0;
    const int STAGE_REGS = STAGE_A + STAGE_B;
    const bool STAGE_AHEAD = STAGE_REGS <= 32;
    const int EST = MWI * NWI + (MWI + NWI) + 40 + (g.DBUF ? 0 : STAGE_REGS * int(STAGE_AHEAD));
    const int MINB_RAW = 65536 / (NT * EST);
    const int MINB = (g.OCC == 0 || MINB_RAW < 1) ? 1 : std::min(MINB_RAW, 16);

    Ptx x;
    const std::string P = name + "_param_";
    const std::string rM = x.r(), rN = x.r(), rK = x.r(), fAl = x.f(), fBe = x.f();
    const std::string dA = x.d(), dB = x.d(), dC = x.d(), dO = x.d();
    x.op("ld.param.u32 " + rM + ", [" + P + "0]");
    x.op("ld.param.u32 " + rN + ", [" + P + "1]");
    x.op("ld.param.u32 " + rK + ", [" + P + "2]");
    x.op("ld.param.f32 " + fAl + ", [" + P + "3]");
    x.op("ld.param.f32 " + fBe + ", [" + P + "4]");
    x.op("ld.param.u64 " + dA + ", [" + P + "5]");
    x.op("ld.param.u64 " + dB + ", [" + P + "6]");
    x.op("ld.param.u64 " + dC + ", [" + P + "7]");
    x.op("ld.param.u64 " + dO + ", [" + P + "8]");
    for (const std::string* q : {&dA, &dB, &dC, &dO}) x.op("cvta.to.global.u64 " + *q + ", " + *q);
    const std::string tx = x.r(), ty = x.r(), cx = x.r(), cy = x.r(), m0 = x.r(), n0 = x.r();
    x.op("mov.u32 " + tx + ", %tid.x");
    x.op("mov.u32 " + ty + ", %tid.y");
    // K range of this CTA: the whole K, or (TAILK) one split of a tail tile.
    const std::string kbeg = x.r(), kend = x.r();
    // TAILK (host switch, part of the compile key): a 1-D grid of `full`
    // whole tiles followed by the remaining (tail) tiles cut into `splits`
    // K-ranges each, so the last wave fills the GPU; a tail CTA stores its
    // partial tile, and the last of a tile's splits to arrive (counter)
    // reduces the partials in split order and runs the epilogue.
    std::string dW, dCnt, rFull, rSplits, pnorm, tail_t, split;
    std::string sk_u, sk_u1, sk_tile, sk_kt0, sk_kt1, sk_j, sk_nseg, sk_maxseg, sk_top, sk_next,
        sk_exit;
    if (g.TAILK) {
        dW = x.d();
        dCnt = x.d();
        rFull = x.r();
        rSplits = x.r();
        const std::string rGX = x.r(), rKT = x.r();
        x.op("ld.param.u64 " + dW + ", [" + P + "9]");
        x.op("ld.param.u64 " + dCnt + ", [" + P + "10]");
        x.op("ld.param.u32 " + rFull + ", [" + P + "11]");
        x.op("ld.param.u32 " + rSplits + ", [" + P + "12]");
        x.op("ld.param.u32 " + rGX + ", [" + P + "13]");
        x.op("ld.param.u32 " + rKT + ", [" + P + "14]");
        x.op("cvta.to.global.u64 " + dW + ", " + dW);
        x.op("cvta.to.global.u64 " + dCnt + ", " + dCnt);
        const std::string b = x.r(), u = x.r(), tile = x.r(), kt0 = x.r(), kt1 = x.r();
        tail_t = x.r();
        split = x.r();
        pnorm = x.p();
        x.op("mov.u32 " + b + ", %ctaid.x");
        x.op("setp.lt.u32 " + pnorm + ", " + b + ", " + rFull);
        x.op("sub.u32 " + u + ", " + b + ", " + rFull);
        x.op("div.u32 " + tail_t + ", " + u + ", " + rSplits);   // tail tile (valid when !pnorm)
        x.op("rem.u32 " + split + ", " + u + ", " + rSplits);
        x.op("add.u32 " + tile + ", " + tail_t + ", " + rFull);
        x.op("selp.u32 " + tile + ", " + b + ", " + tile + ", " + pnorm);
        x.op("rem.u32 " + cx + ", " + tile + ", " + rGX);
        x.op("div.u32 " + cy + ", " + tile + ", " + rGX);
        // split j covers K-tiles [j*kt/s, (j+1)*kt/s)
        x.op("mul.lo.u32 " + kt0 + ", " + split + ", " + rKT);
        x.op("div.u32 " + kt0 + ", " + kt0 + ", " + rSplits);
        x.op("mad.lo.u32 " + kt1 + ", " + split + ", " + rKT + ", " + rKT);
        x.op("div.u32 " + kt1 + ", " + kt1 + ", " + rSplits);
        x.op("mul.lo.u32 " + kt0 + ", " + kt0 + ", " + imm(g.KWG));
        x.op("mul.lo.u32 " + kt1 + ", " + kt1 + ", " + imm(g.KWG));
        x.op("selp.u32 " + kbeg + ", 0, " + kt0 + ", " + pnorm);
        x.op("selp.u32 " + kend + ", " + rK + ", " + kt1 + ", " + pnorm);
    } else if (g.SK) {
        // SK (host switch, part of the compile key): stream-K.  The
        // tiles x K-tiles units are dealt to the 1-D grid of G CTAs as
        // contiguous ranges [c*U/G, (c+1)*U/G); a CTA walks its range as
        // segments (one per tile it touches).  A segment that is a whole
        // tile runs the epilogue; otherwise it stores its partial tile in
        // slot tile*MAXSEG + j (j = its index among the tile's segments) and
        // the last of the tile's segments to arrive sums the partials in
        // segment order (deterministic) and runs the epilogue.
        dW = x.d();
        dCnt = x.d();
        const std::string rU = x.r(), rGX = x.r(), rKT = x.r(), rG = x.r(), c = x.r(), t = x.d();
        sk_maxseg = x.r();
        x.op("ld.param.u64 " + dW + ", [" + P + "9]");
        x.op("ld.param.u64 " + dCnt + ", [" + P + "10]");
        x.op("ld.param.u32 " + rU + ", [" + P + "11]");
        x.op("ld.param.u32 " + sk_maxseg + ", [" + P + "12]");
        x.op("ld.param.u32 " + rGX + ", [" + P + "13]");
        x.op("ld.param.u32 " + rKT + ", [" + P + "14]");
        x.op("cvta.to.global.u64 " + dW + ", " + dW);
        x.op("cvta.to.global.u64 " + dCnt + ", " + dCnt);
        x.op("mov.u32 " + c + ", %ctaid.x");
        x.op("mov.u32 " + rG + ", %nctaid.x");
        sk_u = x.r();
        sk_u1 = x.r();
        // u0(c) = floor(c * U / G)
        auto u0 = [&](const std::string& cc, const std::string& out) {
            x.op("mul.wide.u32 " + t + ", " + cc + ", " + rU);
            const std::string gd = x.d();
            x.op("cvt.u64.u32 " + gd + ", " + rG);
            x.op("div.u64 " + t + ", " + t + ", " + gd);
            x.op("cvt.u32.u64 " + out + ", " + t);
        };
        // cv(v) = the CTA whose range holds unit v = floor(((v+1)*G - 1) / U)
        auto cv = [&](const std::string& v, const std::string& out) {
            const std::string v1 = x.r(), ud = x.d();
            x.op("add.u32 " + v1 + ", " + v + ", 1");
            x.op("mul.wide.u32 " + t + ", " + v1 + ", " + rG);
            x.op("sub.u64 " + t + ", " + t + ", 1");
            x.op("cvt.u64.u32 " + ud + ", " + rU);
            x.op("div.u64 " + t + ", " + t + ", " + ud);
            x.op("cvt.u32.u64 " + out + ", " + t);
        };
        u0(c, sk_u);
        {
            const std::string c1 = x.r();
            x.op("add.u32 " + c1 + ", " + c + ", 1");
            u0(c1, sk_u1);
        }
        sk_top = x.label();
        sk_next = x.label();
        sk_exit = x.label();
        x.lab(sk_top);
        {
            const std::string pe = x.p();
            x.op("setp.ge.u32 " + pe + ", " + sk_u + ", " + sk_u1);
            x.op("@" + pe + " bra " + sk_exit);
        }
        x.op("bar.sync 0");  // the previous segment is done with the staged tiles
        sk_tile = x.r();
        sk_kt0 = x.r();
        sk_kt1 = x.r();
        sk_j = x.r();
        sk_nseg = x.r();
        pnorm = x.p();
        const std::string rest = x.r(), first = x.r(), last = x.r(), v = x.r();
        x.op("div.u32 " + sk_tile + ", " + sk_u + ", " + rKT);
        x.op("mul.lo.u32 " + v + ", " + sk_tile + ", " + rKT);
        x.op("sub.u32 " + sk_kt0 + ", " + sk_u + ", " + v);
        x.op("sub.u32 " + rest + ", " + sk_u1 + ", " + sk_u);
        x.op("add.u32 " + sk_kt1 + ", " + sk_kt0 + ", " + rest);
        x.op("min.u32 " + sk_kt1 + ", " + sk_kt1 + ", " + rKT);
        cv(v, first);  // v = tile * KT
        {
            const std::string vl = x.r();
            x.op("add.u32 " + vl + ", " + v + ", " + rKT);
            x.op("sub.u32 " + vl + ", " + vl + ", 1");
            cv(vl, last);
        }
        x.op("sub.u32 " + sk_j + ", " + c + ", " + first);
        x.op("sub.u32 " + sk_nseg + ", " + last + ", " + first);
        x.op("add.u32 " + sk_nseg + ", " + sk_nseg + ", 1");
        x.op("setp.eq.u32 " + pnorm + ", " + sk_nseg + ", 1");
        x.op("rem.u32 " + cx + ", " + sk_tile + ", " + rGX);
        x.op("div.u32 " + cy + ", " + sk_tile + ", " + rGX);
        x.op("mul.lo.u32 " + kbeg + ", " + sk_kt0 + ", " + imm(g.KWG));
        x.op("mul.lo.u32 " + kend + ", " + sk_kt1 + ", " + imm(g.KWG));
    } else {
        x.op("mov.u32 " + cx + ", %ctaid.x");
        x.op("mov.u32 " + cy + ", %ctaid.y");
        x.op("mov.u32 " + kbeg + ", 0");
        x.op("mov.u32 " + kend + ", " + rK);
    }
    x.op("mul.lo.u32 " + m0 + ", " + cx + ", " + imm(g.MWG));
    x.op("mul.lo.u32 " + n0 + ", " + cy + ", " + imm(g.NWG));
    const std::string tid = x.r();
    x.op("mad.lo.u32 " + tid + ", " + ty + ", " + imm(g.MDIMC) + ", " + tx);
    std::string sbase;
    if (ca.on || cb.on) {
        const std::string d = x.d();
        sbase = x.r();
        x.op("mov.u64 " + d + ", smem");
        x.op("cvt.u32.u64 " + sbase + ", " + d);
    }

    // Copy coordinates: l0 = tid % DIM, l1 = tid / DIM; copying threads.
    for (Copy* c : {&ca, &cb}) {
        if (!c->on) continue;
        c->l0 = x.r();
        c->l1 = x.r();
        int lg = 0;
        while ((1 << lg) < c->DIM) ++lg;
        x.op("and.b32 " + c->l0 + ", " + tid + ", " + imm(c->DIM - 1));
        x.op("shr.u32 " + c->l1 + ", " + tid + ", " + imm(lg));
        if (!(c->V >= c->DIM)) {
            c->copies = x.p();
            x.op("setp.lt.u32 " + c->copies + ", " + c->l0 + ", " + imm(c->V));
        }
    }
    const std::string rMb = x.d(), rNb = x.d();
    x.op("mul.wide.u32 " + rMb + ", " + rM + ", 4");
    x.op("mul.wide.u32 " + rNb + ", " + rN + ", 4");

    // Copy element (row kk0 + l1*KW + ki, vector mv) of operand c lives at
    // base + (kk0 + l1*KW + ki) * ld * 4 + (o0 + mv*VW) * 4 in global memory
    // and at buf + ((l1*KW + ki) * WG + mv*VW) * 4 in the staged tile.
    // Vector index copied by this thread's i-th copy: STR ? l0 + i*DIM : i + l0*MV.
    auto copy_vec = [&](Copy& c, int i) -> std::string {
        const std::string mv = x.r();
        if (c.STR) x.op("add.u32 " + mv + ", " + c.l0 + ", " + imm((long long)i * c.DIM));
        else x.op("mad.lo.u32 " + mv + ", " + c.l0 + ", " + imm(c.MV) + ", " + imm(i));
        return mv;
    };
    // Global address of copy (ki, mv) of operand c for K-tile kk0.
    auto copy_gaddr = [&](Copy& c, bool isA, const std::string& kk0, int ki,
                          const std::string& mv) -> std::string {
        const std::string row = x.r(), d1 = x.d(), col = x.r(), d2 = x.d(), a = x.d();
        x.op("mad.lo.u32 " + row + ", " + c.l1 + ", " + imm(c.KW) + ", " + kk0);
        if (ki) x.op("add.u32 " + row + ", " + row + ", " + imm(ki));
        x.op("mul.wide.u32 " + d1 + ", " + row + ", " + (isA ? rM : rN));
        x.op("mad.lo.u32 " + col + ", " + mv + ", " + imm(c.VW) + ", " + (isA ? m0 : n0));
        x.op("cvt.u64.u32 " + d2 + ", " + col);
        x.op("add.u64 " + d1 + ", " + d1 + ", " + d2);
        x.op("shl.b64 " + d1 + ", " + d1 + ", 2");
        x.op("add.u64 " + a + ", " + (isA ? dA : dB) + ", " + d1);
        return a;
    };
    auto copy_saddr = [&](Copy& c, const std::string& bufoff, int ki, const std::string& mv)
        -> std::string {
        const std::string s = x.r(), t = x.r();
        x.op("mad.lo.u32 " + s + ", " + c.l1 + ", " + imm((long long)c.KW * c.WG) + ", " +
             imm((long long)ki * c.WG));
        x.op("mad.lo.u32 " + s + ", " + mv + ", " + imm(c.VW) + ", " + s);
        x.op("shl.b32 " + s + ", " + s + ", 2");
        x.op("add.u32 " + t + ", " + s + ", " + bufoff);
        return t;
    };

    // cp.async of K-tile kk0 into the tiles at shared addresses buf_a / buf_b.
    auto issue = [&](const std::string& kk0, const std::string& buf_a, const std::string& buf_b) {
        for (Copy* c : {&ca, &cb}) {
            if (!c->on) continue;
            const bool isA = c == &ca;
            const std::string skip = x.label();
            if (!c->copies.empty()) x.op("@!" + c->copies + " bra " + skip);
            for (int ki = 0; ki < c->KW; ++ki)
                for (int i = 0; i < c->MV; ++i) {
                    const std::string mv = copy_vec(*c, i);
                    const std::string ga = copy_gaddr(*c, isA, kk0, ki, mv);
                    const std::string sa = copy_saddr(*c, isA ? buf_a : buf_b, ki, mv);
                    if (c->VW == 1) {
                        x.op("cp.async.ca.shared.global [" + sa + "], [" + ga + "], 4");
                    } else if (c->VW == 2) {
                        x.op("cp.async.ca.shared.global [" + sa + "], [" + ga + "], 8");
                    } else {
                        for (int q = 0; q < c->VW; q += 4)
                            x.op("cp.async.cg.shared.global [" + sa + "+" + imm(4 * q) + "], [" + ga +
                                 "+" + imm(4 * q) + "], 16");
                    }
                }
            x.lab(skip);
        }
        x.op("cp.async.commit_group");
    };

    // Register staging (no DBUF): fetch into registers, stash into buffer 0.
    std::vector<std::string> ra(static_cast<size_t>(STAGE_A)), rb(static_cast<size_t>(STAGE_B));
    for (auto& v : ra) v = x.f();
    for (auto& v : rb) v = x.f();
    auto fetch = [&](const std::string& kk0) {
        for (Copy* c : {&ca, &cb}) {
            if (!c->on) continue;
            const bool isA = c == &ca;
            auto& regs = isA ? ra : rb;
            const std::string skip = x.label();
            if (!c->copies.empty()) x.op("@!" + c->copies + " bra " + skip);
            for (int ki = 0; ki < c->KW; ++ki)
                for (int i = 0; i < c->MV; ++i) {
                    const std::string mv = copy_vec(*c, i);
                    const std::string ga = copy_gaddr(*c, isA, kk0, ki, mv);
                    std::vector<std::string> dst(regs.begin() + (ki * c->MV + i) * c->VW,
                                                 regs.begin() + (ki * c->MV + i + 1) * c->VW);
                    vld(x, "global.nc", ga, 0, dst);
                }
            x.lab(skip);
        }
    };
    auto stash = [&](const std::string& buf_a, const std::string& buf_b) {
        for (Copy* c : {&ca, &cb}) {
            if (!c->on) continue;
            const bool isA = c == &ca;
            auto& regs = isA ? ra : rb;
            const std::string skip = x.label();
            if (!c->copies.empty()) x.op("@!" + c->copies + " bra " + skip);
            for (int ki = 0; ki < c->KW; ++ki)
                for (int i = 0; i < c->MV; ++i) {
                    const std::string mv = copy_vec(*c, i);
                    const std::string sa = copy_saddr(*c, isA ? buf_a : buf_b, ki, mv);
                    std::vector<std::string> src(regs.begin() + (ki * c->MV + i) * c->VW,
                                                 regs.begin() + (ki * c->MV + i + 1) * c->VW);
                    vst(x, "shared", sa, 0, src);
                }
            x.lab(skip);
        }
    };

    // Accumulators.
    std::vector<std::vector<std::string>> acc(static_cast<size_t>(MWI), std::vector<std::string>(static_cast<size_t>(NWI)));
    for (auto& row : acc)
        for (auto& a : row) {
            a = x.f();
            x.op("mov.f32 " + a + ", 0f00000000");
        }

    // Buffer byte offsets (absolute shared addresses) for buffer 0 / 1.
    std::string a_buf0, a_buf1, b_buf0, b_buf1;
    if (ca.on) {
        a_buf0 = x.r();
        x.op("add.u32 " + a_buf0 + ", " + sbase + ", " + imm(ca.sm_off));
        if (g.DBUF) {
            a_buf1 = x.r();
            x.op("add.u32 " + a_buf1 + ", " + a_buf0 + ", " + imm((long long)g.KWG * g.MWG * 4));
        }
    }
    if (cb.on) {
        b_buf0 = x.r();
        x.op("add.u32 " + b_buf0 + ", " + sbase + ", " + imm(cb.sm_off));
        if (g.DBUF) {
            b_buf1 = x.r();
            x.op("add.u32 " + b_buf1 + ", " + b_buf0 + ", " + imm((long long)g.KWG * g.NWG * 4));
        }
    }
    if (g.DBUF) issue(kbeg, a_buf0, b_buf0);
    else if (ca.on || cb.on) fetch(kbeg);

    // Fragment offsets within a K-row (bytes): a: mv*VWM*4 = abase + aimm(mi),
    // b: nv*VWN*4 = bbase + bimm(ni) (the thread part in a register, the
    // vector index as an immediate).
    const std::string abase = x.r(), bbase = x.r();
    x.op("mul.lo.u32 " + abase + ", " + tx + ", " + imm((long long)(g.STRM ? 1 : MVI) * g.VWM * 4));
    x.op("mul.lo.u32 " + bbase + ", " + ty + ", " + imm((long long)(g.STRN ? 1 : NVI) * g.VWN * 4));
    auto aimm = [&](int mi) { return (long long)(g.STRM ? mi * g.MDIMC : mi) * g.VWM * 4; };
    auto bimm = [&](int ni) { return (long long)(g.STRN ? ni * g.NDIMC : ni) * g.VWN * 4; };

    // ---- k0 loop
    const std::string k0 = x.r(), buf = x.r(), lk0 = x.label(), lend = x.label();
    x.op("mov.u32 " + k0 + ", " + kbeg);
    x.op("mov.u32 " + buf + ", 0");
    {
        const std::string pe = x.p();
        x.op("setp.ge.u32 " + pe + ", " + k0 + ", " + kend);
        x.op("@" + pe + " bra " + lend);
    }
    x.lab(lk0);
    x.op(".pragma \"nounroll\"");
    const std::string knext = x.r(), pmore = x.p();
    x.op("add.u32 " + knext + ", " + k0 + ", " + imm(g.KWG));
    x.op("setp.lt.u32 " + pmore + ", " + knext + ", " + kend);
    std::string acur, bcur;  // current tile base (shared u32)
    if (g.DBUF) {
        x.op("cp.async.wait_group 0");
        x.op("bar.sync 0");
        const std::string pb = x.p(), done = x.label();
        x.op("setp.ne.u32 " + pb + ", " + buf + ", 0");
        std::string na, nb;  // the other buffer: next K-tile goes there
        if (ca.on) {
            na = x.r();
            x.op("selp.u32 " + na + ", " + a_buf0 + ", " + a_buf1 + ", " + pb);
        }
        if (cb.on) {
            nb = x.r();
            x.op("selp.u32 " + nb + ", " + b_buf0 + ", " + b_buf1 + ", " + pb);
        }
        x.op("@!" + pmore + " bra " + done);
        issue(knext, na, nb);
        x.lab(done);
        if (ca.on) {
            acur = x.r();
            x.op("selp.u32 " + acur + ", " + a_buf1 + ", " + a_buf0 + ", " + pb);
        }
        if (cb.on) {
            bcur = x.r();
            x.op("selp.u32 " + bcur + ", " + b_buf1 + ", " + b_buf0 + ", " + pb);
        }
    } else if (ca.on || cb.on) {
        stash(a_buf0, b_buf0);
        x.op("bar.sync 0");
        if (STAGE_AHEAD) {
            const std::string skip = x.label();
            x.op("@!" + pmore + " bra " + skip);
            fetch(knext);
            x.lab(skip);
        }
        acur = a_buf0;
        bcur = b_buf0;
    }

    // ---- kw loop (rolled), KWI unrolled k-steps
    const std::string kw = x.r(), lkw = x.label();
    x.op("mov.u32 " + kw + ", 0");
    x.lab(lkw);
    x.op(".pragma \"nounroll\"");
    // Per kw trip: one base per operand; k-steps and vectors are immediates
    // (shared) or one 64-bit add per k-step (global).
    std::string arow, brow, ag, bg;
    if (ca.on) {
        arow = x.r();
        x.op("mad.lo.u32 " + arow + ", " + kw + ", " + imm((long long)g.MWG * 4) + ", " + acur);
        x.op("add.u32 " + arow + ", " + arow + ", " + abase);
    } else {
        const std::string kk = x.r(), d1 = x.d(), d2 = x.d();
        ag = x.d();
        x.op("add.u32 " + kk + ", " + k0 + ", " + kw);
        x.op("mul.wide.u32 " + d1 + ", " + kk + ", " + rM);
        x.op("cvt.u64.u32 " + d2 + ", " + m0);
        x.op("add.u64 " + d1 + ", " + d1 + ", " + d2);
        x.op("shl.b64 " + d1 + ", " + d1 + ", 2");
        x.op("add.u64 " + ag + ", " + dA + ", " + d1);
        const std::string o = x.d();
        x.op("cvt.u64.u32 " + o + ", " + abase);
        x.op("add.u64 " + ag + ", " + ag + ", " + o);
    }
    if (cb.on) {
        brow = x.r();
        x.op("mad.lo.u32 " + brow + ", " + kw + ", " + imm((long long)g.NWG * 4) + ", " + bcur);
        x.op("add.u32 " + brow + ", " + brow + ", " + bbase);
    } else {
        const std::string kk = x.r(), d1 = x.d(), d2 = x.d();
        bg = x.d();
        x.op("add.u32 " + kk + ", " + k0 + ", " + kw);
        x.op("mul.wide.u32 " + d1 + ", " + kk + ", " + rN);
        x.op("cvt.u64.u32 " + d2 + ", " + n0);
        x.op("add.u64 " + d1 + ", " + d1 + ", " + d2);
        x.op("shl.b64 " + d1 + ", " + d1 + ", 2");
        x.op("add.u64 " + bg + ", " + dB + ", " + d1);
        const std::string o = x.d();
        x.op("cvt.u64.u32 " + o + ", " + bbase);
        x.op("add.u64 " + bg + ", " + bg + ", " + o);
    }
    for (int ki = 0; ki < g.KWI; ++ki) {
        // k = kw + ki
        std::vector<std::string> a(static_cast<size_t>(MWI)), b(static_cast<size_t>(NWI));
        for (auto& v : a) v = x.f();
        for (auto& v : b) v = x.f();
        if (ca.on) {
            for (int mi = 0; mi < MVI; ++mi)
                vld(x, "shared", arow, (long long)ki * g.MWG * 4 + aimm(mi),
                    std::vector<std::string>(a.begin() + mi * g.VWM, a.begin() + (mi + 1) * g.VWM));
        } else {
            if (ki) x.op("add.u64 " + ag + ", " + ag + ", " + rMb);
            for (int mi = 0; mi < MVI; ++mi)
                vld(x, "global.nc", ag, aimm(mi),
                    std::vector<std::string>(a.begin() + mi * g.VWM, a.begin() + (mi + 1) * g.VWM));
        }
        if (cb.on) {
            for (int ni = 0; ni < NVI; ++ni)
                vld(x, "shared", brow, (long long)ki * g.NWG * 4 + bimm(ni),
                    std::vector<std::string>(b.begin() + ni * g.VWN, b.begin() + (ni + 1) * g.VWN));
        } else {
            if (ki) x.op("add.u64 " + bg + ", " + bg + ", " + rNb);
            for (int ni = 0; ni < NVI; ++ni)
                vld(x, "global.nc", bg, bimm(ni),
                    std::vector<std::string>(b.begin() + ni * g.VWN, b.begin() + (ni + 1) * g.VWN));
        }
        // outer product (gemm.cu outer_product_t)
        if (g.F2 && NWI % 2 == 0) {
            for (int i = 0; i < MWI; ++i)
                for (int j = 0; j < NWI; j += 2) {
                    const std::string pa = x.d(), pbv = x.d(), pc = x.d(), pd = x.d();
                    x.op("mov.b64 " + pa + ", {" + a[size_t(i)] + ", " + a[size_t(i)] + "}");
                    x.op("mov.b64 " + pbv + ", {" + b[size_t(j)] + ", " + b[size_t(j + 1)] + "}");
                    x.op("mov.b64 " + pc + ", {" + acc[size_t(i)][size_t(j)] + ", " + acc[size_t(i)][size_t(j + 1)] + "}");
                    x.op("fma.rn.f32x2 " + pd + ", " + pa + ", " + pbv + ", " + pc);
                    x.op("mov.b64 {" + acc[size_t(i)][size_t(j)] + ", " + acc[size_t(i)][size_t(j + 1)] + "}, " + pd);
                }
        } else if (g.F2 && MWI % 2 == 0) {
            for (int i = 0; i < MWI; i += 2)
                for (int j = 0; j < NWI; ++j) {
                    const std::string pa = x.d(), pbv = x.d(), pc = x.d(), pd = x.d();
                    x.op("mov.b64 " + pa + ", {" + a[size_t(i)] + ", " + a[size_t(i + 1)] + "}");
                    x.op("mov.b64 " + pbv + ", {" + b[size_t(j)] + ", " + b[size_t(j)] + "}");
                    x.op("mov.b64 " + pc + ", {" + acc[size_t(i)][size_t(j)] + ", " + acc[size_t(i + 1)][size_t(j)] + "}");
                    x.op("fma.rn.f32x2 " + pd + ", " + pa + ", " + pbv + ", " + pc);
                    x.op("mov.b64 {" + acc[size_t(i)][size_t(j)] + ", " + acc[size_t(i + 1)][size_t(j)] + "}, " + pd);
                }
        } else {
            for (int i = 0; i < MWI; ++i)
                for (int j = 0; j < NWI; ++j)
                    x.op("fma.rn.f32 " + acc[size_t(i)][size_t(j)] + ", " + a[size_t(i)] + ", " +
                         b[size_t(j)] + ", " + acc[size_t(i)][size_t(j)]);
        }
    }
    {
        const std::string pk = x.p();
        x.op("add.u32 " + kw + ", " + kw + ", " + imm(g.KWI));
        x.op("setp.lt.u32 " + pk + ", " + kw + ", " + imm(g.KWG));
        x.op("@" + pk + " bra " + lkw);
    }
    if (!g.DBUF && (ca.on || cb.on)) {
        x.op("bar.sync 0");
        if (!STAGE_AHEAD) {
            const std::string skip = x.label();
            x.op("@!" + pmore + " bra " + skip);
            fetch(knext);
            x.lab(skip);
        }
    }
    x.op("xor.b32 " + buf + ", " + buf + ", 1");
    x.op("mov.u32 " + k0 + ", " + knext);
    x.op("@" + pmore + " bra " + lk0);
    x.lab(lend);

    // ---- TAILK / SK: partial tiles meet here
    if (g.TAILK || g.SK) {
        const std::string lepi = x.label();
        x.op("@" + pnorm + " bra " + lepi);
        const long long tile_bytes = (long long)g.MWG * g.NWG * 4;
        // this CTA's partial: W + (slot * tile_bytes); the tile's partials
        // start at slot tslot; cidx = the tile's arrival counter; nparts
        // partials are summed by the last to arrive.
        const std::string slot = x.r(), wmine = x.d(), wtile = x.d(), tmp = x.d();
        const std::string tslot = x.r(), cidx = g.SK ? sk_tile : tail_t,
                          nparts = g.SK ? sk_nseg : rSplits;
        if (g.SK) {
            x.op("mul.lo.u32 " + tslot + ", " + sk_tile + ", " + sk_maxseg);
            x.op("add.u32 " + slot + ", " + tslot + ", " + sk_j);
        } else {
            x.op("mad.lo.u32 " + slot + ", " + tail_t + ", " + rSplits + ", " + split);
            x.op("mul.lo.u32 " + tslot + ", " + tail_t + ", " + rSplits);
        }
        x.op("mul.wide.u32 " + tmp + ", " + slot + ", " + imm(tile_bytes));
        x.op("add.u64 " + wmine + ", " + dW + ", " + tmp);
        x.op("mul.wide.u32 " + tmp + ", " + tslot + ", " + imm(tile_bytes));
        x.op("add.u64 " + wtile + ", " + dW + ", " + tmp);
        // byte offset of (mi, e, ni) inside a tile: same element map as the epilogue
        auto tile_off = [&](int mi, int e) {
            const std::string mo = x.r();
            x.op("shr.u32 " + mo + ", " + abase + ", 2");
            x.op("add.u32 " + mo + ", " + mo + ", " + imm(aimm(mi) / 4 + e));
            x.op("mul.lo.u32 " + mo + ", " + mo + ", " + imm((long long)g.NWG * 4));
            x.op("add.u32 " + mo + ", " + mo + ", " + bbase);
            const std::string d = x.d();
            x.op("cvt.u64.u32 " + d + ", " + mo);
            return d;
        };
        for (int mi = 0; mi < MVI; ++mi)
            for (int e = 0; e < g.VWM; ++e) {
                const std::string off = tile_off(mi, e), a = x.d();
                x.op("add.u64 " + a + ", " + wmine + ", " + off);
                for (int ni = 0; ni < NVI; ++ni) {
                    std::vector<std::string> s(acc[size_t(mi * g.VWM + e)].begin() + ni * g.VWN,
                                               acc[size_t(mi * g.VWM + e)].begin() + (ni + 1) * g.VWN);
                    vst(x, "global", a, bimm(ni), s);
                }
            }
        x.op("fence.acq_rel.gpu");
        x.op("bar.sync 0");
        const std::string ptid0 = x.p(), arrived = x.r(), cnt_a = x.d(), flag = x.r();
        const long long flag_off = (long long)(g.SA * g.KWG * g.MWG + g.SB * g.KWG * g.NWG) * 4 *
                                   (1 + g.DBUF);
        {
            const std::string d = x.d();
            x.op("mov.u64 " + d + ", smem");
            x.op("cvt.u32.u64 " + flag + ", " + d);
            x.op("add.u32 " + flag + ", " + flag + ", " + imm(flag_off));
        }
        x.op("mul.wide.u32 " + cnt_a + ", " + cidx + ", 4");
        x.op("add.u64 " + cnt_a + ", " + dCnt + ", " + cnt_a);
        x.op("setp.eq.u32 " + ptid0 + ", " + tid + ", 0");
        {
            const std::string skip = x.label();
            x.op("@!" + ptid0 + " bra " + skip);
            x.op("atom.acq_rel.gpu.global.add.u32 " + arrived + ", [" + cnt_a + "], 1");
            x.op("st.shared.u32 [" + flag + "], " + arrived);
            x.lab(skip);
        }
        x.op("bar.sync 0");
        {
            const std::string seen = x.r(), last = x.r(), plast = x.p();
            x.op("ld.shared.u32 " + seen + ", [" + flag + "]");
            x.op("sub.u32 " + last + ", " + nparts + ", 1");
            x.op("setp.ne.u32 " + plast + ", " + seen + ", " + last);
            if (g.SK) x.op("@" + plast + " bra " + sk_next);  // another segment sums this tile
            else x.op("@" + plast + " ret");  // not the last split of this tile
        }
        x.op("fence.acq_rel.gpu");
        {
            const std::string skip = x.label();
            x.op("@!" + ptid0 + " bra " + skip);
            x.op("st.relaxed.gpu.global.u32 [" + cnt_a + "], 0");  // ready for the next launch
            x.lab(skip);
        }
        // acc = 0 + partial[0] + partial[1] + ... in split order
        // (deterministic; one rolled loop keeps the code small)
        for (auto& row : acc)
            for (auto& a : row) x.op("mov.f32 " + a + ", 0f00000000");
        std::vector<std::string> offs;
        for (int mi = 0; mi < MVI; ++mi)
            for (int e = 0; e < g.VWM; ++e) offs.push_back(tile_off(mi, e));
        const std::string j = x.r(), wj = x.d(), lj = x.label(), pj = x.p();
        x.op("mov.u32 " + j + ", 0");
        x.op("mov.u64 " + wj + ", " + wtile);
        x.lab(lj);
        x.op(".pragma \"nounroll\"");
        {
            size_t oi = 0;
            for (int mi = 0; mi < MVI; ++mi)
                for (int e = 0; e < g.VWM; ++e) {
                    const std::string a = x.d();
                    x.op("add.u64 " + a + ", " + wj + ", " + offs[oi++]);
                    for (int ni = 0; ni < NVI; ++ni) {
                        auto& row = acc[size_t(mi * g.VWM + e)];
                        std::vector<std::string> v(static_cast<size_t>(g.VWN));
                        for (auto& r : v) r = x.f();
                        vld(x, "global.cg", a, bimm(ni), v);
                        for (int q = 0; q < g.VWN; ++q)
                            x.op("add.rn.f32 " + row[size_t(ni * g.VWN + q)] + ", " +
                                 row[size_t(ni * g.VWN + q)] + ", " + v[size_t(q)]);
                    }
                }
        }
        x.op("add.u64 " + wj + ", " + wj + ", " + imm(tile_bytes));
        x.op("add.u32 " + j + ", " + j + ", 1");
        x.op("setp.lt.u32 " + pj + ", " + j + ", " + nparts);
        x.op("@" + pj + " bra " + lj);
        x.lab(lepi);
    }

    // ---- epilogue: Cout = alpha * acc (+ beta * Cin), VWN-wide along N
    const std::string pbeta = x.p();
    x.op("setp.neu.f32 " + pbeta + ", " + fBe + ", 0f00000000");
    for (int mi = 0; mi < MVI; ++mi) {
        for (int e = 0; e < g.VWM; ++e) {
            // m = m0 + mv*VWM + e, with mv*VWM*4 = abase + aimm(mi)
            const std::string m = x.r();
            x.op("shr.u32 " + m + ", " + abase + ", 2");
            x.op("add.u32 " + m + ", " + m + ", " + m0);
            x.op("add.u32 " + m + ", " + m + ", " + imm(aimm(mi) / 4 + e));
            const std::string rowoff = x.d(), d2 = x.d();
            x.op("mul.wide.u32 " + rowoff + ", " + m + ", " + rN);
            x.op("cvt.u64.u32 " + d2 + ", " + n0);
            x.op("add.u64 " + rowoff + ", " + rowoff + ", " + d2);
            x.op("shl.b64 " + rowoff + ", " + rowoff + ", 2");
            const std::string bo = x.d(), rowb = x.d();
            x.op("cvt.u64.u32 " + bo + ", " + bbase);
            x.op("add.u64 " + rowb + ", " + rowoff + ", " + bo);
            for (int ni = 0; ni < NVI; ++ni) {
                const std::string idx = x.d(), oa = x.d();
                x.op("add.u64 " + idx + ", " + rowb + ", " + imm(bimm(ni)));
                x.op("add.u64 " + oa + ", " + dO + ", " + idx);
                std::vector<std::string> s(static_cast<size_t>(g.VWN));
                for (auto& v : s) v = x.f();
                const std::string lb = x.label(), ld = x.label();
                x.op("@" + pbeta + " bra " + lb);
                for (int q = 0; q < g.VWN; ++q)
                    x.op("mul.f32 " + s[size_t(q)] + ", " + fAl + ", " +
                         acc[size_t(mi * g.VWM + e)][size_t(ni * g.VWN + q)]);
                x.op("bra.uni " + ld);
                x.lab(lb);
                {
                    const std::string ca2 = x.d();
                    x.op("add.u64 " + ca2 + ", " + dC + ", " + idx);
                    std::vector<std::string> c(static_cast<size_t>(g.VWN));
                    for (auto& v : c) v = x.f();
                    vld(x, "global.nc", ca2, 0, c);
                    for (int q = 0; q < g.VWN; ++q) {
                        const std::string t = x.f();
                        x.op("mul.f32 " + t + ", " + fBe + ", " + c[size_t(q)]);
                        x.op("fma.rn.f32 " + s[size_t(q)] + ", " + fAl + ", " +
                             acc[size_t(mi * g.VWM + e)][size_t(ni * g.VWN + q)] + ", " + t);
                    }
                }
                x.lab(ld);
                vst(x, "global", oa, 0, s);
            }
        }
    }
    if (g.SK) {
        x.lab(sk_next);
        const std::string dk = x.r();
        x.op("sub.u32 " + dk + ", " + sk_kt1 + ", " + sk_kt0);
        x.op("add.u32 " + sk_u + ", " + sk_u + ", " + dk);
        x.op("bra.uni " + sk_top);
        x.lab(sk_exit);
    }
    x.op("ret");

    std::ostringstream e;
    e << ".visible .entry " << name << "(\n"
      << "\t.param .u32 " << P << "0,\n\t.param .u32 " << P << "1,\n\t.param .u32 " << P
      << "2,\n\t.param .f32 " << P << "3,\n\t.param .f32 " << P << "4,\n\t.param .u64 .ptr .align 1 "
      << P << "5,\n\t.param .u64 .ptr .align 1 " << P << "6,\n\t.param .u64 .ptr .align 1 " << P
      << "7,\n\t.param .u64 .ptr .align 1 " << P << "8";
    if (g.TAILK || g.SK)
        e << ",\n\t.param .u64 .ptr .align 1 " << P << "9,\n\t.param .u64 .ptr .align 1 " << P
          << "10,\n\t.param .u32 " << P << "11,\n\t.param .u32 " << P << "12,\n\t.param .u32 " << P
          << "13,\n\t.param .u32 " << P << "14";
    e << "\n)\n.maxntid " << NT << ", 1, 1\n"
      << ".minnctapersm " << MINB << "\n{\n" << x.decls() << x.body() << "}\n";
    return e.str();
}

}  // namespace

std::string gemm_ptx_module(const Defines& problem, const std::vector<const Defines*>& configs,
                            const std::string& entry_base) {
    (void)problem;
    std::ostringstream m;
    m << "//\n// Generated by libktc ptxgen_gemm (gemm.cu semantics)\n//\n"
      << ".version 8.8\n.target sm_100a\n.address_size 64\n\n"
      << ".extern .shared .align 16 .b8 smem[];\n\n";
    for (size_t i = 0; i < configs.size(); ++i)
        m << emit_entry(parse(*configs[i]), entry_base + "_k" + std::to_string(i)) << "\n";
    return m.str();
}

}  // namespace ktc
