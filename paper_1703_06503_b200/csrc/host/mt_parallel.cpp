// mt_parallel.cpp -- multi-threaded materialization of `uniform:<seed>` f32
// recipes, bit-identical to the sequential std::mt19937_64 stream.
//
// The reference materializes every uniform input with one sequential
// mt19937_64 (arguments.hpp:126-180, rng.hpp:12-19): one generator call per
// f32 element.  A conv input at configs[0] is 33.6 M elements, ~250 ms on one
// core -- longer than evaluating dozens of configurations on the B200, so a
// fresh tuning job would be bound by its host input generation.
//
// The generator is linear over GF(2): the state after t steps is T^t(S0).
// With P the minimal polynomial of the output recurrence (degree 19937,
// found once per process by Berlekamp-Massey on 2*19937 output bits), the
// state J steps ahead is p(T)(S) with p = x^J mod P (Horner over the state;
// T is one single-word generator step, so a jump costs ~19937 word steps and
// ~10^4 window XORs, about a millisecond).  The stream is cut into chunks of
// J = 2^20 elements; chunk c starts at p_{c}(T)(S0), composed from the
// precomputed x^(2^k J) mod P over the set bits of c, so every worker jumps
// to its own chunks independently and generates them with the ordinary
// recurrence.  (T has a 31-dimensional kernel -- the low bits of the word
// about to be overwritten, which no output ever reads; the jump is exact on
// everything else, which is all the outputs depend on.)
//
// tests/test_capi.py checks the parallel stream against the sequential one
// element for element, and the golden digests pin the materialized images.
#pragma GCC optimize("O3")
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ktb/rng.hpp"

namespace ktb {
namespace {

constexpr int kN = 312, kM = 156;
constexpr uint64_t kA = 0xB5026F5AA96619E9ull, kUpper = 0xFFFFFFFF80000000ull,
                   kLower = 0x7FFFFFFFull;
constexpr int kDeg = 19937;                 // degree of the minimal polynomial
constexpr int kPolyWords = kDeg / 64 + 1;   // 312 words hold degrees 0..19967
constexpr size_t kChunkLog2 = 20;           // J = 2^20 elements per chunk
constexpr size_t kChunk = size_t(1) << kChunkLog2;

// Generator state as a circular window: logical word j is w[(i + j) % kN].
struct State {
    uint64_t w[kN];
    int i = 0;
};

void seed_state(State& s, uint64_t seed) {  // std::mt19937_64 seeding
    s.w[0] = seed;
    for (int k = 1; k < kN; ++k)
        s.w[k] = 6364136223846793005ull * (s.w[k - 1] ^ (s.w[k - 1] >> 62)) + uint64_t(k);
    s.i = 0;
}

inline uint64_t step(State& s) {  // one untempered word; T applied once
    const int i = s.i, i1 = i + 1 == kN ? 0 : i + 1, im = i + kM >= kN ? i + kM - kN : i + kM;
    const uint64_t y = (s.w[i] & kUpper) | (s.w[i1] & kLower);
    const uint64_t v = s.w[im] ^ (y >> 1) ^ ((y & 1u) ? kA : 0u);
    s.w[i] = v;
    s.i = i1;
    return v;
}

inline uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    return y ^ (y >> 43);
}

// ---------------------------------------------------------------- GF(2)[x]
using Poly = std::vector<uint64_t>;  // bit k = coefficient of x^k

inline bool bit(const Poly& p, size_t k) { return (p[k >> 6] >> (k & 63)) & 1u; }

// Minimal polynomial of the recurrence of output bit 0 (Berlekamp-Massey).
Poly minimal_polynomial() {
    const int n_bits = 2 * kDeg + 64;
    const int W = (n_bits + 63) / 64 + 1;
    std::vector<uint64_t> seq(static_cast<size_t>(n_bits));
    State s;
    seed_state(s, 5489u);
    for (int n = 0; n < n_bits; ++n) seq[size_t(n)] = temper(step(s)) & 1u;
    // C, B: connection polynomials; win: bit i = s_{n-i}
    std::vector<uint64_t> C(size_t(W), 0), B(size_t(W), 0), Tmp, win(size_t(W), 0);
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < n_bits; ++n) {
        // win <<= 1; win |= s_n
        for (int k = W - 1; k > 0; --k) win[size_t(k)] = (win[size_t(k)] << 1) | (win[size_t(k - 1)] >> 63);
        win[0] = (win[0] << 1) | seq[size_t(n)];
        uint64_t d = 0;
        const int words = L / 64 + 1;
        for (int k = 0; k < words; ++k) d ^= C[size_t(k)] & win[size_t(k)];
        if (!(__builtin_popcountll(d) & 1)) {
            ++m;
            continue;
        }
        auto add_shifted = [&](std::vector<uint64_t>& dst, const std::vector<uint64_t>& src, int sh) {
            const int ws = sh / 64, bs = sh % 64;
            for (int k = W - 1; k >= ws; --k) {
                uint64_t v = src[size_t(k - ws)] << bs;
                if (bs && k - ws - 1 >= 0) v |= src[size_t(k - ws - 1)] >> (64 - bs);
                dst[size_t(k)] ^= v;
            }
        };
        if (2 * L <= n) {
            Tmp = C;
            add_shifted(C, B, m);
            L = n + 1 - L;
            B = Tmp;
            m = 1;
        } else {
            add_shifted(C, B, m);
            ++m;
        }
    }
    if (L != kDeg) throw std::runtime_error("mt19937_64 jump: unexpected recurrence degree");
    // P(x) = x^L C(1/x): coefficient of x^(L-i) is c_i
    Poly P(size_t(kPolyWords), 0);
    for (int i = 0; i <= L; ++i)
        if (bit(C, size_t(i))) P[size_t(L - i) >> 6] |= uint64_t(1) << ((L - i) & 63);
    return P;
}

inline uint64_t spread32(uint64_t v) {
    v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
    v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    return (v | (v << 1)) & 0x5555555555555555ull;
}

struct Reducer {
    // P shifted left by b bits (b = 0..63), so every reduction step is an
    // aligned word XOR.
    std::vector<Poly> shifted;
    explicit Reducer(const Poly& P) : shifted(64) {
        for (int b = 0; b < 64; ++b) {
            Poly q(size_t(kPolyWords) + 1, 0);
            for (int k = 0; k < kPolyWords; ++k) {
                q[size_t(k)] |= P[size_t(k)] << b;
                if (b) q[size_t(k) + 1] |= P[size_t(k)] >> (64 - b);
            }
            shifted[size_t(b)] = std::move(q);
        }
    }
    // a (degree < 2*kDeg) mod P, in place; returns kPolyWords words.
    Poly reduce(Poly a) const {
        for (int d = int(a.size()) * 64 - 1; d >= kDeg; --d) {
            if (!bit(a, size_t(d))) continue;
            const int sh = d - kDeg, ws = sh / 64;
            const Poly& q = shifted[size_t(sh % 64)];
            for (size_t k = 0; k < q.size() && size_t(ws) + k < a.size(); ++k) a[size_t(ws) + k] ^= q[k];
        }
        a.resize(size_t(kPolyWords));
        return a;
    }
    Poly square(const Poly& p) const {
        Poly a(size_t(2 * kPolyWords), 0);
        for (int k = 0; k < kPolyWords; ++k) {
            a[size_t(2 * k)] = spread32(p[size_t(k)] & 0xFFFFFFFFull);
            a[size_t(2 * k + 1)] = spread32(p[size_t(k)] >> 32);
        }
        return reduce(std::move(a));
    }
};

// r ^= s in logical (window) order: r's word j is r.w[(r.i + j) % kN].
inline void xor_window(State& r, const State& s) {
    int a = r.i, b = s.i, j = 0;
    while (j < kN) {
        const int run = std::min({kN - j, kN - a, kN - b});
        uint64_t* __restrict dst = r.w + a;
        const uint64_t* __restrict src = s.w + b;
        for (int k = 0; k < run; ++k) dst[k] ^= src[k];
        j += run;
        a += run;
        b += run;
        if (a == kN) a = 0;
        if (b == kN) b = 0;
    }
}

// p(T)(s) by Horner: r = 0; for i = deg..0: r = T(r); if p_i: r ^= s.
State jump(const State& s, const Poly& p) {
    State r;
    std::memset(r.w, 0, sizeof r.w);
    r.i = 0;
    int top = kDeg;
    while (top >= 0 && !bit(p, size_t(top))) --top;
    for (int d = top; d >= 0; --d) {
        step(r);
        if (bit(p, size_t(d))) xor_window(r, s);
    }
    return r;
}

// out[0..n) = float(uniform01) of the next n draws from `st`, in blocks of
// kN words (the standard block twist once the window starts at index 0).
void generate(State st, float* out, size_t n) {
    uint64_t x[kN];
    for (int j = 0; j < kN; ++j) x[j] = st.w[(st.i + j) % kN];
    auto mix = [](uint64_t a, uint64_t b, uint64_t c) {
        const uint64_t y = (a & kUpper) | (b & kLower);
        return c ^ (y >> 1) ^ ((y & 1u) ? kA : 0u);
    };
    size_t done = 0;
    while (done < n) {
        for (int k = 0; k < kN - kM; ++k) x[k] = mix(x[k], x[k + 1], x[k + kM]);
        for (int k = kN - kM; k < kN - 1; ++k) x[k] = mix(x[k], x[k + 1], x[k + kM - kN]);
        x[kN - 1] = mix(x[kN - 1], x[0], x[kM - 1]);
        const size_t take = std::min<size_t>(kN, n - done);
        for (size_t k = 0; k < take; ++k)
            out[done + k] = static_cast<float>(double(temper(x[k]) >> 11) * 0x1.0p-53);
        done += take;
    }
}

struct JumpTable {
    std::mutex mu;
    bool ready = false;
    std::unique_ptr<Reducer> red;
    std::deque<Poly> pow2;  // (deque: references stay valid) pow2[k] = x^(2^k * J) mod P
    const Poly& power(size_t k) {
        std::lock_guard<std::mutex> lk(mu);
        if (!ready) {
            const Poly P = minimal_polynomial();
            red = std::make_unique<Reducer>(P);
            Poly x(size_t(kPolyWords), 0);
            x[0] = 2;  // x
            for (size_t s = 0; s < kChunkLog2; ++s) x = red->square(x);
            pow2.push_back(std::move(x));
            ready = true;
        }
        while (pow2.size() <= k) pow2.push_back(red->square(pow2.back()));
        return pow2[k];
    }
};

JumpTable& jump_table() {
    static JumpTable* t = new JumpTable;  // leaked: safe during static destruction
    return *t;
}

}  // namespace

void fill_uniform_f32(uint64_t seed, float* out, size_t n, int threads) {
    const size_t chunks = (n + kChunk - 1) / kChunk;
    if (threads <= 1 || chunks < 4) {
        Rng rng(seed);
        for (size_t i = 0; i < n; ++i) out[i] = static_cast<float>(uniform01(rng));
        return;
    }
    // Worker w owns the contiguous chunk range [w*q, (w+1)*q): one jump
    // sequence to its first chunk, then the ordinary recurrence.
    const size_t workers = std::min<size_t>(size_t(threads), chunks);
    const size_t q = (chunks + workers - 1) / workers;
    size_t bits = 0;
    while ((size_t(1) << bits) < chunks) ++bits;
    std::vector<const Poly*> pw(bits);
    for (size_t k = 0; k < bits; ++k) pw[k] = &jump_table().power(k);
    State s0;
    seed_state(s0, seed);
    std::vector<std::thread> pool;
    pool.reserve(workers);
    for (size_t w = 0; w < workers; ++w) {
        const size_t c0 = w * q;
        if (c0 >= chunks) break;
        pool.emplace_back([&, c0] {
            State st = s0;
            for (size_t k = 0; k < bits; ++k)
                if ((c0 >> k) & 1u) st = jump(st, *pw[k]);
            const size_t lo = c0 * kChunk, hi = std::min(n, (c0 + q) * kChunk);
            generate(st, out + lo, hi - lo);
        });
    }
    for (auto& t : pool) t.join();
}

}  // namespace ktb
