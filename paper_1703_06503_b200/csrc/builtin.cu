// builtin.cu -- fixed (non-tuned) device kernels of the B200 evaluation
// backend, compiled ahead of time by nvcc for sm_100a and embedded in
// libktc.so as a cubin:
//
//   ktc_conv_reference / ktc_gemm_reference
//       The device-side reference ("SetReference" in CLTune terms).  They
//       perform exactly the reference oracle's per-element operation
//       sequence -- rounded fp32 multiply, then rounded fp32 add, in the
//       oracle's loop order (landscapes.hpp:129-140 and :301-309) -- so their
//       output is BIT-IDENTICAL to conv_apply/gemm_apply on the CPU
//       (tests/test_gpu_parity.py checks the FNV digests against the
//       reference's golden digests).  Compiled with -fmad=false and explicit
//       __fmul_rn/__fadd_rn so no FMA contraction can creep in.
//
//   ktc_verify_partial / ktc_verify_final / ktc_verify_after
//       The device-side output verification that replaces the host loop of
//       verify_outputs (tuner.hpp:39-106).  Same pass rule (in double),
//       same report fields, same first-failure / first-argmax indices, and
//       the reference's NaN quirk (a NaN error resets the running maximum)
//       reproduced exactly via a second pass over the suffix after the last
//       NaN.
//
//   ktc_l2_flush
//       Streams a buffer larger than L2 through the cache between timed
//       repetitions (read-only, so no write-back lands inside the next
//       timed kernel).
#include <stdint.h>

#define KTC_VERIFY_THREADS 256

// ---------------------------------------------------------------------------
// Device reference: convolution.  One thread per output; image is the
// re-pitched padded image (row pitch `ipitch` floats).
// ---------------------------------------------------------------------------
extern "C" __global__ void ktc_conv_reference(int X, int Y, int F, float W,
                                              const float* __restrict__ img, int ipitch,
                                              const float* __restrict__ taps,
                                              float* __restrict__ out) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    const int row = blockIdx.y * blockDim.y + threadIdx.y;
    if (col >= X || row >= Y) return;
    float acc = 0.0f;
    for (int j = 0; j < F; ++j) {
        const float* line = img + (size_t)(row + j) * ipitch + col;
        const float* tap = taps + j * F;
        for (int i = 0; i < F; ++i) acc = __fadd_rn(acc, __fmul_rn(tap[i], line[i]));
    }
    out[(size_t)row * X + col] = __fmul_rn(W, acc);
}

// ---------------------------------------------------------------------------
// Device reference: C = alpha * A^T B + beta * C.  Shared-memory tiled, but
// each thread owns one output and adds the products in ascending k with
// separate rounding -- the oracle's exact sequence.
// ---------------------------------------------------------------------------
#define RT 32
extern "C" __global__ void __launch_bounds__(RT * 8)
ktc_gemm_reference(int M, int N, int K, float alpha, float beta,
                   const float* __restrict__ A, const float* __restrict__ B,
                   const float* __restrict__ C, float* __restrict__ out) {
    __shared__ float As[RT][RT + 1];  // [k][m]
    __shared__ float Bs[RT][RT + 1];  // [k][n]
    const int tx = threadIdx.x;       // n within tile (0..31)
    const int ty = threadIdx.y;       // 0..7, each owns 4 rows
    const int m0 = blockIdx.y * RT, n0 = blockIdx.x * RT;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int k0 = 0; k0 < K; k0 += RT) {
        for (int r = ty; r < RT; r += 8) {
            const int k = k0 + r;
            As[r][tx] = (k < K && m0 + tx < M) ? A[(size_t)k * M + m0 + tx] : 0.0f;
            Bs[r][tx] = (k < K && n0 + tx < N) ? B[(size_t)k * N + n0 + tx] : 0.0f;
        }
        __syncthreads();
        const int kmax = min(RT, K - k0);
        for (int kk = 0; kk < kmax; ++kk) {
            const float b = Bs[kk][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(As[kk][ty * 4 + q], b));
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int m = m0 + ty * 4 + q, n = n0 + tx;
        if (m < M && n < N) {
            const size_t idx = (size_t)m * N + n;
            out[idx] = __fadd_rn(__fmul_rn(alpha, acc[q]), __fmul_rn(beta, C[idx]));
        }
    }
}

// ---------------------------------------------------------------------------
// Verification.  Partial state per thread/block:
//   first_fail   lowest index failing the pass rule (UINT64_MAX if none)
//   max_abs      max |c-r| over non-NaN errors, argmax = lowest index of it
//   nan_abs      highest index whose |c-r| is NaN (-1 if none)
//   max_rel      max rel error over non-NaN rel errors
//   nan_rel      highest index whose rel error is NaN (-1 if none)
// ---------------------------------------------------------------------------
struct VerifyPartial {
    unsigned long long first_fail;
    unsigned long long argmax;
    long long nan_abs;
    long long nan_rel;
    double max_abs;
    double max_rel;
};

__device__ __forceinline__ void vp_init(VerifyPartial& p) {
    p.first_fail = ~0ull;
    p.argmax = ~0ull;
    p.nan_abs = -1;
    p.nan_rel = -1;
    p.max_abs = -1.0;
    p.max_rel = -1.0;
}

__device__ __forceinline__ void vp_merge(VerifyPartial& a, const VerifyPartial& b) {
    a.first_fail = a.first_fail < b.first_fail ? a.first_fail : b.first_fail;
    if (b.max_abs > a.max_abs || (b.max_abs == a.max_abs && b.argmax < a.argmax)) {
        a.max_abs = b.max_abs;
        a.argmax = b.argmax;
    }
    a.nan_abs = a.nan_abs > b.nan_abs ? a.nan_abs : b.nan_abs;
    a.nan_rel = a.nan_rel > b.nan_rel ? a.nan_rel : b.nan_rel;
    a.max_rel = a.max_rel > b.max_rel ? a.max_rel : b.max_rel;
}

__device__ __forceinline__ void vp_shfl_merge(VerifyPartial& p, int offset) {
    VerifyPartial o;
    o.first_fail = __shfl_down_sync(0xffffffffu, p.first_fail, offset);
    o.argmax = __shfl_down_sync(0xffffffffu, p.argmax, offset);
    o.nan_abs = __shfl_down_sync(0xffffffffu, p.nan_abs, offset);
    o.nan_rel = __shfl_down_sync(0xffffffffu, p.nan_rel, offset);
    o.max_abs = __shfl_down_sync(0xffffffffu, p.max_abs, offset);
    o.max_rel = __shfl_down_sync(0xffffffffu, p.max_rel, offset);
    vp_merge(p, o);
}

__device__ __forceinline__ void vp_block_reduce(VerifyPartial& p, VerifyPartial* out) {
    __shared__ VerifyPartial warp_part[KTC_VERIFY_THREADS / 32];
    for (int off = 16; off > 0; off >>= 1) vp_shfl_merge(p, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_part[warp] = p;
    __syncthreads();
    if (warp == 0) {
        if (lane < KTC_VERIFY_THREADS / 32) p = warp_part[lane];
        else vp_init(p);
        for (int off = 16; off > 0; off >>= 1) vp_shfl_merge(p, off);
        if (lane == 0) *out = p;
    }
}

// One f32 element, the reference rule in double (tuner.hpp:86-93).  The
// relative error's division is exact but rare: it is only evaluated when it
// could raise the running maximum (abs >= max_rel * mag, with a 2^-40 margin
// for the rounding of the product), or for the NaN / infinite corner cases.
__device__ __forceinline__ void vp_f32(VerifyPartial& p, unsigned long long i, float cf, float rf,
                                       double rel_tol, double abs_tol) {
    const double c = (double)cf, r = (double)rf;
    const double abs_err = fabs(c - r);
    const double mag = fabs(r);
    if (!(abs_err <= abs_tol + rel_tol * mag) && i < p.first_fail) p.first_fail = i;  // NaN fails
    if (abs_err > p.max_abs) {
        p.max_abs = abs_err;
        p.argmax = i;
    } else if (abs_err != abs_err) {
        p.nan_abs = (long long)i;  // indices grow per thread: last wins
    }
    if (mag > 0.0) {
        if (abs_err >= p.max_rel * mag * (1.0 - 0x1.0p-40) || abs_err != abs_err ||
            mag == __longlong_as_double(0x7ff0000000000000ll)) {
            const double rel = abs_err / mag;
            if (rel > p.max_rel) p.max_rel = rel;
            else if (rel != rel) p.nan_rel = (long long)i;
        }
    } else if (0.0 > p.max_rel) {
        p.max_rel = 0.0;  // mag == 0 (or NaN): the reference's rel_err is 0
    }
}

// fp32 screen in front of vp_f32: an element whose effect on the state is
// provably nil is skipped without any double arithmetic.  With D = |c - r|
// (exact) and the float estimate df = fl(|c - r|) (relative error <= 2^-24):
//   * pass is certain when df <= 0.5 * fl(rel * |r| + abs)  (margin >> float
//     rounding of the tolerance), so first_fail cannot move;
//   * D > max_abs is impossible when df < abs_lo = rd(max_abs * (1 - 2^-20));
//   * D / |r| > max_rel is impossible when df < fl(rel_lo * |r|), rel_lo =
//     rd(max_rel * (1 - 2^-20));
//   * non-finite inputs, |r| == 0 while max_rel < 0, and everything else take
//     the exact double path, which then refreshes the screen thresholds.
// The screened rule is therefore identical to vp_f32 (same state, bit for
// bit); it only moves the common case -- a passing element below both running
// maxima -- onto a handful of FP32 instructions, so the verifier runs at the
// HBM rate of its two input streams instead of the FP64 rate.
// Ties matter: outputs of a passing kernel differ from the reference by a
// few ulps, so many elements share the running maximum exactly.  When c and
// r are within a factor of two of each other (same sign), c - r is exact in
// float (Sterbenz), df == D, and "D <= rd(max_abs)" settles the strict
// comparison without the margin.
struct VerifyScreen {
    float abs_rd;   // rd(max_abs)
    float abs_lo;   // rd(max_abs * (1 - 2^-20))
    float rel_lo;   // rd(max_rel * (1 - 2^-20))
    bool rel_nonneg;  // max_rel >= 0 (a zero relative error cannot raise it)
};

// Pins a value in a register: without it ptxas rematerializes the
// thresholds from the double state (F2F + DSETP) at every use in the hot loop.
__device__ __forceinline__ float pin(float v) {
    asm volatile("mov.b32 %0, %0;" : "+f"(v));
    return v;
}

__device__ __forceinline__ void vs_refresh(VerifyScreen& s, const VerifyPartial& p) {
    s.abs_rd = pin(__double2float_rd(p.max_abs));
    s.abs_lo = pin(__double2float_rd(p.max_abs * (1.0 - 0x1.0p-20)));
    s.rel_lo = pin(__double2float_rd(p.max_rel * (1.0 - 0x1.0p-20)));
    s.rel_nonneg = pin(p.max_rel >= 0.0 ? 1.0f : 0.0f) != 0.0f;
}

// Thresholds shared by the warp.  The report keeps the maximum over ALL
// elements (lowest index on ties), so an element strictly below an error
// some other lane has already seen can never be the final maximum, whatever
// this lane's own running state says; per-lane records alone would flag
// ~ln(n)/n of the elements, and a flag costs the whole (divergent) warp.
struct WarpScreen {
    float abs_rd;  // rd(max over lanes of max_abs): an attained error
    float abs_lo;  // the same with the 2^-20 margin for inexact differences
    float rel_lo;  // rd(max over lanes of max_rel * (1 - 2^-20))
};

__device__ __forceinline__ void ws_refresh(WarpScreen& w, const VerifyScreen& s) {
    float a = s.abs_rd, l = s.abs_lo, r = s.rel_lo;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
        l = fmaxf(l, __shfl_xor_sync(0xffffffffu, l, o));
        r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, o));
    }
    w.abs_rd = a;
    w.abs_lo = l;
    w.rel_lo = r;
}

// Per-batch screen thresholds (lane state merged with the warp's).
struct ScreenThr {
    float abs_le;  // skip an exact difference D <= abs_le
    float rel_lt;  // skip when D < rel_lt * |r|
    bool zero_ok;  // a zero error cannot raise max_rel
};

__device__ __forceinline__ ScreenThr screen_thresholds(const VerifyScreen& s, const WarpScreen& w) {
    ScreenThr t;
    // Own maximum: ties keep the earlier index, so D == max_abs is a no-op.
    // Another lane's maximum only dominates strictly: one float below it.
    t.abs_le = pin(fmaxf(s.abs_rd, nextafterf(w.abs_rd, -INFINITY)));
    t.rel_lt = pin(fmaxf(s.rel_lo, w.rel_lo));
    t.zero_ok = s.rel_nonneg;
    return t;
}

// True when element i might change the state (then vp_f32 decides exactly).
// `close` (|c - r| <= 2^-10 |r|) puts c and r within a factor of two of each
// other with the same sign, so fl(c - r) is exact (Sterbenz) and df == D;
// anything else -- far apart, zero reference with nonzero candidate,
// non-finite -- is flagged.
__device__ __forceinline__ bool vs_needs(const ScreenThr& t, float cf, float rf, float half_rel,
                                         float half_abs) {
    const float df = fabsf(cf - rf);
    const float mf = fabsf(rf);
    const bool ok = df <= fmaf(half_rel, mf, half_abs)   // certain pass (NaN compares false)
                    && df <= mf * 0x1.0p-10f              // close: exact difference
                    && df <= t.abs_le                     // cannot raise max_abs
                    && (df < t.rel_lt * mf || (df == 0.0f && t.zero_ok))  // nor max_rel
                    && mf <= 3.4028234663852886e38f;      // finite
    return !ok;
}

__device__ __forceinline__ void vp_i32(VerifyPartial& p, unsigned long long i, int ci, int ri) {
    const double abs_err = fabs((double)ci - (double)ri);
    if (ci != ri && i < p.first_fail) p.first_fail = i;
    if (abs_err > p.max_abs) {
        p.max_abs = abs_err;
        p.argmax = i;
    }
    if (abs_err > p.max_rel) p.max_rel = abs_err;
}

// Each block owns one contiguous chunk (a multiple of 4 elements); threads
// stride through it in float4 steps, so a thread's indices are increasing
// (needed for the nan_* "last" updates).
extern "C" __global__ void __launch_bounds__(KTC_VERIFY_THREADS)
ktc_verify_partial(const void* __restrict__ cand, const void* __restrict__ ref,
                   unsigned long long n, int is_f32, double rel_tol, double abs_tol,
                   VerifyPartial* __restrict__ partials) {
    VerifyPartial p;
    vp_init(p);
    const unsigned long long chunk = ((n + gridDim.x - 1) / gridDim.x + 3) & ~3ull;
    const unsigned long long begin = chunk * blockIdx.x;
    const unsigned long long end = begin + chunk < n ? begin + chunk : n;
    if (is_f32) {
        const float* c = (const float*)cand;
        const float* r = (const float*)ref;
        const unsigned long long end4 = begin + ((end > begin ? end - begin : 0) & ~3ull);
        // One state per thread: the fp32 screen settles almost every element
        // without touching the running maxima, so there is no dependency
        // chain to break.  U float4 pairs are loaded before any is screened
        // (memory-level parallelism for the two HBM streams); flagged
        // elements then go through the exact rule in index order, in one
        // rolled loop (one copy of the double-precision code).  Skips stay valid while flagged elements update the state:
        // the maxima only grow and first_fail only shrinks.
        VerifyScreen sc;
        vs_refresh(sc, p);
        WarpScreen ws;
        ws_refresh(ws, sc);
        // Tolerances beyond float range would make the fp32 pass screen
        // unsound; then every element is flagged (exact path).
        const bool tol_ok = rel_tol < 1e30 && abs_tol < 1e30;
        const float half_rel = tol_ok ? 0.5f * (float)rel_tol : -INFINITY;
        const float half_abs = tol_ok ? 0.5f * (float)abs_tol : -INFINITY;
        constexpr int U = 4;
        const unsigned long long step = 4ull * KTC_VERIFY_THREADS;
        // Warp-uniform trip count (the warp's first lane drives the loop),
        // so the warp-wide threshold exchange below never diverges.
        const unsigned long long lane4 = 4ull * (threadIdx.x & 31);
        for (unsigned long long w0 = begin + 4ull * (threadIdx.x & ~31u); w0 < end4; w0 += U * step) {
            const unsigned long long i0 = w0 + lane4;
            float4 cv[U], rv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned long long i = i0 + u * step;
                if (i < end4) {
                    cv[u] = __ldcs(reinterpret_cast<const float4*>(c + i));
                    rv[u] = __ldg(reinterpret_cast<const float4*>(r + i));
                } else {
                    cv[u] = rv[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                }
            }
            const ScreenThr thr = screen_thresholds(sc, ws);
            unsigned need = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                need |= unsigned(vs_needs(thr, cv[u].x, rv[u].x, half_rel, half_abs)) << (4 * u);
                need |= unsigned(vs_needs(thr, cv[u].y, rv[u].y, half_rel, half_abs)) << (4 * u + 1);
                need |= unsigned(vs_needs(thr, cv[u].z, rv[u].z, half_rel, half_abs)) << (4 * u + 2);
                need |= unsigned(vs_needs(thr, cv[u].w, rv[u].w, half_rel, half_abs)) << (4 * u + 3);
                if (i0 + u * step >= end4) need &= ~(0xfu << (4 * u));
            }
#pragma unroll 1
            while (need) {
                const int b = __ffs(need) - 1;
                need &= need - 1;
                const unsigned long long i = i0 + (b >> 2) * step + (b & 3);
                // The pair from registers (a select chain, no dynamic
                // indexing): re-reading memory here would put a round trip
                // on every flagged element of every lane.
                float cf = 0.0f, rf = 0.0f;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if ((b >> 2) == u) {
                        const int l = b & 3;
                        cf = l == 0 ? cv[u].x : l == 1 ? cv[u].y : l == 2 ? cv[u].z : cv[u].w;
                        rf = l == 0 ? rv[u].x : l == 1 ? rv[u].y : l == 2 ? rv[u].z : rv[u].w;
                    }
                }
                vp_f32(p, i, cf, rf, rel_tol, abs_tol);
                vs_refresh(sc, p);
            }
            ws_refresh(ws, sc);  // every lane reaches here: the loop bound is warp-uniform
        }
        for (unsigned long long i = end4 + threadIdx.x; i < end; i += KTC_VERIFY_THREADS)
            vp_f32(p, i, __ldg(c + i), __ldg(r + i), rel_tol, abs_tol);
    } else {
        const int* c = (const int*)cand;
        const int* r = (const int*)ref;
        for (unsigned long long i = begin + threadIdx.x; i < end; i += KTC_VERIFY_THREADS)
            vp_i32(p, i, __ldg(c + i), __ldg(r + i));
    }
    vp_block_reduce(p, partials + blockIdx.x);
}

extern "C" __global__ void __launch_bounds__(KTC_VERIFY_THREADS)
ktc_verify_final(const VerifyPartial* __restrict__ partials, int count,
                 VerifyPartial* __restrict__ result) {
    VerifyPartial p;
    vp_init(p);
    for (int i = threadIdx.x; i < count; i += KTC_VERIFY_THREADS) vp_merge(p, partials[i]);
    vp_block_reduce(p, result);
}

// Second pass, only run when a NaN error occurred before the last element:
// the reference's running max restarts after the last NaN (tuner.hpp:53-62),
// so the reported maximum is the max over the suffix (start, n).
extern "C" __global__ void __launch_bounds__(KTC_VERIFY_THREADS)
ktc_verify_after(const void* __restrict__ cand, const void* __restrict__ ref,
                 unsigned long long n, int is_f32, long long abs_start, long long rel_start,
                 VerifyPartial* __restrict__ partials) {
    VerifyPartial p;
    vp_init(p);
    const unsigned long long stride = (unsigned long long)gridDim.x * KTC_VERIFY_THREADS;
    for (unsigned long long i = (unsigned long long)blockIdx.x * KTC_VERIFY_THREADS + threadIdx.x;
         i < n; i += stride) {
        double c, r;
        if (is_f32) {
            c = (double)((const float*)cand)[i];
            r = (double)((const float*)ref)[i];
        } else {
            c = (double)((const int*)cand)[i];
            r = (double)((const int*)ref)[i];
        }
        const double abs_err = fabs(c - r);
        double rel_err = abs_err;
        if (is_f32) {
            const double mag = fabs(r);
            rel_err = mag > 0.0 ? abs_err / mag : 0.0;
        }
        if ((long long)i > abs_start && abs_err > p.max_abs) p.max_abs = abs_err;
        if ((long long)i > rel_start && rel_err > p.max_rel) p.max_rel = rel_err;
    }
    vp_block_reduce(p, partials + blockIdx.x);
}

// ---------------------------------------------------------------------------
// L2 flush: read `n4` float4s; the never-taken store keeps the loads alive.
// ---------------------------------------------------------------------------
extern "C" __global__ void ktc_l2_flush(const float4* __restrict__ buf, unsigned long long n4,
                                        float* __restrict__ sink) {
    float s = 0.0f;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += stride) {
        const float4 v = buf[i];  // normal caching: displaces resident lines
        s += v.x + v.y + v.z + v.w;
    }
    if (s == -1.0f) *sink = s;  // buffer holds zeros: never true
}
