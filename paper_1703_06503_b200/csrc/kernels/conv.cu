// conv.cu -- tunable 2D convolution family, compiled at tuning time by NVRTC
// for sm_100a, one specialization per configuration of conv_space()
// (reference landscapes.hpp:62-75).  Computes, for the re-pitched padded
// image (row pitch IPITCH floats):
//     out[r*X + c] = W * sum_{j<FS} sum_{i<FS} taps[j*FS+i] * img[(r+j)*IPITCH + c+i]
// which is conv_apply (landscapes.hpp:120-143) with fp32 FMA accumulation
// (taps in ascending j, i order, as the oracle).
//
// Parameters (all compile-time, set by the host as -D defines):
//   XWG, YWG    thread block shape (reference local size, landscapes.hpp:90)
//   XWPT, YWPT  outputs per thread in x / y (thread coarsening)
//   VW          vector width: a thread's x-outputs come in XWPT/VW groups of
//               VW contiguous outputs; consecutive threads own consecutive
//               groups, so every load/store is a coalesced VW-wide vector
//   LOCAL       0: read the image straight from global (L1-cached ld.global.nc)
//               1: cooperative global->shared copy of the halo tile
//               2: TMA (cp.async.bulk.tensor.2d) copy of the halo tile into
//                  shared memory, completion tracked by an mbarrier: the
//                  "extra halo loaders" of the paper are the TMA engine, so
//                  no extra threads are launched (local = XWG x YWG stays true)
//   PAD         +1 column (LOCAL=1) / +4 columns (LOCAL=2) in the shared tile
//   UNR         1: filter loops fully unrolled with a register sliding window
//                  (each input row is read once per thread, taps are
//                  constant-bank operands of FFMA);
//               0: filter loops rolled (#pragma unroll 1)
//   FS          filter size (compile-time)
//   CF2         (host) 1: UNR=1 pairs output rows into packed FFMA2 (c_tpair)
//   GUARD       1 when X % (XWG*XWPT) or Y % (YWG*YWPT) is non-zero
// Derived (host-computed): SP (LOCAL=1 pitch), PWO/BW/BH/NB/NP/PF (LOCAL=2
// panel geometry: PWO output columns per panel, box BW x BH floats, NB boxes
// per panel, NP panels, PF floats per panel).

typedef unsigned int u32;

__constant__ float c_taps[FS * FS];
// Tap pairs for row-paired FFMA2: c_tpair[jj*FS + i] = (taps[jj][i], taps[jj-1][i]),
// jj >= 1 (set by the host next to c_taps).
__constant__ float2 c_tpair[FS * FS];

struct __align__(64) TensorMap {
    unsigned long long v[16];
};

// ---------------------------------------------------------------------------
// Vector helpers.  N in {1, 2, 4, 8}.
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void ld_global(float* d, const float* __restrict__ p) {
    if (N == 1) {
        d[0] = __ldg(p);
    } else if (N == 2) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(p));
        d[0] = v.x; d[1] = v.y;
    } else {
#pragma unroll
        for (int q = 0; q < N; q += 4) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(p + q));
            d[q] = v.x; d[q + 1] = v.y; d[q + 2] = v.z; d[q + 3] = v.w;
        }
    }
}

template <int N>
__device__ __forceinline__ void ld_shared(float* d, const float* p) {
    if (N == 1) {
        d[0] = p[0];
    } else if (N == 2) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        d[0] = v.x; d[1] = v.y;
    } else {
#pragma unroll
        for (int q = 0; q < N; q += 4) {
            const float4 v = *reinterpret_cast<const float4*>(p + q);
            d[q] = v.x; d[q + 1] = v.y; d[q + 2] = v.z; d[q + 3] = v.w;
        }
    }
}

template <int N>
__device__ __forceinline__ void st_global(float* p, const float* s) {
    if (N == 1) {
        p[0] = s[0];
    } else if (N == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(s[0], s[1]);
    } else {
#pragma unroll
        for (int q = 0; q < N; q += 4)
            *reinterpret_cast<float4*>(p + q) = make_float4(s[q], s[q + 1], s[q + 2], s[q + 3]);
    }
}

// Largest power of two <= 4 dividing both VW and the shared pitch: the
// widest aligned shared-memory vector a window load can use.
#define POW2_DIV(p) (((p) % 4 == 0) ? 4 : (((p) % 2 == 0) ? 2 : 1))
#define MIN_(a, b) ((a) < (b) ? (a) : (b))

// ---------------------------------------------------------------------------
// TMA / mbarrier primitives (LOCAL == 2).
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 smem_addr(const void* p) {
    return static_cast<u32>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

// Bounded wait: a lost transaction traps (-> launch error -> runtime_error
// for this configuration) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
    u32 done = 0;
    for (long long spin = 0; spin < (1ll << 26); ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
    }
    __trap();
}

__device__ __forceinline__ void tma_load_2d(u32 dst, const TensorMap* map, u32 bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}

//@@KTC_BODY@@ -- everything below is instantiated once per configuration
// (inside its own namespace when several configurations share one NVRTC
// program); KTC_ENTRY names the kernel.
#ifndef CF2  // host-chosen (backend.cpp plan_conv): row-paired FFMA2
#define CF2 1
#define KTC_CF2_DEFAULT
#endif
#define H ((FS - 1) / 2)
#define TX (XWG * XWPT)
#define TY (YWG * YWPT)
#define NG (XWPT / VW)
#define NT (XWG * YWG)
#if LOCAL == 0
#define SVW VW
#elif LOCAL == 1
#define SVW MIN_(VW, POW2_DIV(SP))
#else
#define SVW MIN_(VW, 4)
#endif
#define WIN (VW + FS - 1)
#define NWV ((WIN + SVW - 1) / SVW)  // vector loads per window row
#define WINP (NWV * SVW)

extern "C" __global__ void __launch_bounds__(NT, 1)
KTC_ENTRY(const int X, const int Y, const float W, const float* __restrict__ img, const int ipitch,
       float* __restrict__ out, const __grid_constant__ TensorMap tmap) {
    const int tx = threadIdx.x;
    const int ty = threadIdx.y;
    const int x0 = blockIdx.x * TX;  // tile origin: output (x0, y0) == padded input (x0, y0)
    const int y0 = blockIdx.y * TY;

    float acc[YWPT][XWPT];
#pragma unroll
    for (int j = 0; j < YWPT; ++j)
#pragma unroll
        for (int q = 0; q < XWPT; ++q) acc[j][q] = 0.0f;

#if LOCAL >= 1
    extern __shared__ __align__(128) float smem[];
#endif

#if LOCAL == 0
    // Row r of this thread's input window: padded row y0 + ty*YWPT + r.
    const float* __restrict__ base = img + (size_t)(y0 + ty * YWPT) * ipitch + x0;
#define ROWPTR(r) (base + (size_t)(r) * ipitch)
#define COLOFF(col) (col)
#elif LOCAL == 1
    {
        // Cooperative halo-tile copy: (TY + 2H) rows of (TX + 2H) floats,
        // moved as aligned float4s (ipitch % 4 == 0, x0 % 8 == 0).
        const int TR = TY + 2 * H;
        const int TC4 = (TX + 2 * H + 3) / 4;
        const int tid = ty * XWG + tx;
        const float* __restrict__ g = img + (size_t)y0 * ipitch + x0;
#pragma unroll 4
        for (int e = tid; e < TR * TC4; e += NT) {
            const int r = e / TC4, c = (e - r * TC4) * 4;
            const float4 v = __ldg(reinterpret_cast<const float4*>(g + (size_t)r * ipitch + c));
            float* s = smem + r * SP + c;
            if (c + 4 <= TX + 2 * H && (SP % 4 == 0)) {
                *reinterpret_cast<float4*>(s) = v;
            } else if (c + 4 <= TX + 2 * H && (SP % 2 == 0)) {
                reinterpret_cast<float2*>(s)[0] = make_float2(v.x, v.y);
                reinterpret_cast<float2*>(s)[1] = make_float2(v.z, v.w);
            } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (c + q < TX + 2 * H) s[q] = vv[q];
            }
        }
        __syncthreads();
    }
    const float* base = smem + (ty * YWPT) * SP;
#define ROWPTR(r) (base + (r) * SP)
#define COLOFF(col) (col)
#else  // LOCAL == 2
    {
        // Panel p holds padded columns [x0 + p*PWO, x0 + p*PWO + BW) for
        // NB*BH rows; boxes land back to back (BH % 8 == 0 keeps each box
        // 128-byte aligned).  The mbarrier lives past the panels.
        float* panels = smem;
        unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + NP * PF);
        const u32 bar_a = smem_addr(bar);
        if (tx == 0 && ty == 0) {
            mbar_init(bar_a, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(bar_a, (u32)(NP * NB * BW * BH * 4));
#pragma unroll 1
            for (int p = 0; p < NP; ++p)
#pragma unroll 1
                for (int b = 0; b < NB; ++b)
                    tma_load_2d(smem_addr(panels + p * PF + b * BH * BW), &tmap, bar_a,
                                x0 + p * PWO, y0 + b * BH);
        }
        __syncthreads();  // barrier initialised before anyone waits on it
        mbar_wait(bar_a, 0);
    }
    const float* base = smem + (ty * YWPT) * BW;
#define ROWPTR(r) (base + (r) * BW)
#define COLOFF(col) (((col) / PWO) * PF + ((col) % PWO))
#endif

#if UNR == 1
    // Register sliding window: for every input row r the thread loads its
    // WIN-wide window once and applies it to every output row it feeds.
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        const int col = (g * XWG + tx) * VW;
#pragma unroll
        for (int r = 0; r < YWPT + FS - 1; ++r) {
            float w[WINP];
            const float* rp = ROWPTR(r) + COLOFF(col);
#pragma unroll
            for (int v = 0; v < NWV; ++v) {
#if LOCAL == 0
                ld_global<SVW>(w + v * SVW, rp + v * SVW);
#else
                ld_shared<SVW>(w + v * SVW, rp + v * SVW);
#endif
            }
#if CF2 && YWPT % 2 == 0
            // Output rows j, j+1 read input row r through tap rows jj, jj-1:
            // one packed FFMA2 per (tap pair, column) with the input value
            // broadcast -- half the FMA-pipe instructions, each lane an exact
            // fmaf, the same per-output order (jj, i ascending) as below.
            // Tap rows outside [0, FS) leave single rows: scalar FFMA.
#pragma unroll
            for (int j = 0; j < YWPT; j += 2) {
                const int jj = r - j;
                if (jj >= 1 && jj < FS) {
#pragma unroll
                    for (int i = 0; i < FS; ++i) {
                        const float2 t2 = c_tpair[jj * FS + i];
#pragma unroll
                        for (int e = 0; e < VW; ++e) {
                            const float2 q = __ffma2_rn(t2, make_float2(w[e + i], w[e + i]),
                                                        make_float2(acc[j][g * VW + e], acc[j + 1][g * VW + e]));
                            acc[j][g * VW + e] = q.x;
                            acc[j + 1][g * VW + e] = q.y;
                        }
                    }
                } else if (jj == 0 || jj == FS) {
                    const int jr = jj == 0 ? j : j + 1;  // the row that has a tap row
                    const int jt = jj == 0 ? 0 : FS - 1;
#pragma unroll
                    for (int i = 0; i < FS; ++i) {
                        const float t = c_taps[jt * FS + i];
#pragma unroll
                        for (int e = 0; e < VW; ++e)
                            acc[jr][g * VW + e] = fmaf(t, w[e + i], acc[jr][g * VW + e]);
                    }
                }
            }
#else
#pragma unroll
            for (int j = 0; j < YWPT; ++j) {
                const int jj = r - j;
                if (jj >= 0 && jj < FS) {
#pragma unroll
                    for (int i = 0; i < FS; ++i) {
                        const float t = c_taps[jj * FS + i];
#pragma unroll
                        for (int e = 0; e < VW; ++e)
                            acc[j][g * VW + e] = fmaf(t, w[e + i], acc[j][g * VW + e]);
                    }
                }
            }
#endif
        }
    }
#else
    // Rolled filter loops: one tap per iteration, one input load per FFMA.
#pragma unroll 1
    for (int jj = 0; jj < FS; ++jj) {
#pragma unroll 1
        for (int i = 0; i < FS; ++i) {
            const float t = c_taps[jj * FS + i];
#pragma unroll
            for (int j = 0; j < YWPT; ++j) {
                const float* rp = ROWPTR(j + jj);
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    const int col = (g * XWG + tx) * VW;
#pragma unroll
                    for (int e = 0; e < VW; ++e) {
#if LOCAL == 0
                        const float v = __ldg(rp + col + e + i);
#else
                        const float v = rp[COLOFF(col + e) + i];
#endif
                        acc[j][g * VW + e] = fmaf(t, v, acc[j][g * VW + e]);
                    }
                }
            }
        }
    }
#endif

    // Epilogue: out = W * acc, VW-wide coalesced stores.
#pragma unroll
    for (int j = 0; j < YWPT; ++j) {
        const int row = y0 + ty * YWPT + j;
#if GUARD
        if (row >= Y) continue;
#endif
        float* orow = out + (size_t)row * X + x0;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int col = (g * XWG + tx) * VW;
            float s[VW];
#pragma unroll
            for (int e = 0; e < VW; ++e) s[e] = W * acc[j][g * VW + e];
#if GUARD
            if (x0 + col + VW > X) {
                for (int e = 0; e < VW; ++e)
                    if (x0 + col + e < X) orow[col + e] = s[e];
                continue;
            }
#endif
#if OUT_VEC
            st_global<VW>(orow + col, s);
#else
            st_global<1>(orow + col, s);
            for (int e = 1; e < VW; ++e) orow[col + e] = s[e];
#endif
        }
    }
}
#undef ROWPTR
#undef COLOFF
#undef H
#undef TX
#undef TY
#undef NG
#undef NT
#undef SVW
#undef WIN
#undef NWV
#undef WINP
#ifdef KTC_CF2_DEFAULT
#undef CF2
#undef KTC_CF2_DEFAULT
#endif
