// gemm.cu -- tunable fp32 SGEMM family, compiled at tuning time by NVRTC for
// sm_100a, one specialization per configuration of gemm_space() (reference
// landscapes.hpp:218-249).  Computes gemm_apply (landscapes.hpp:293-312):
//     Cout[m*N + n] = ALPHA * sum_k A[k*M + m] * B[k*N + n] + BETA * Cin[m*N + n]
// with A stored K x M (M contiguous), B K x N (N contiguous), C M x N (N
// contiguous).  fp32 FFMA on the CUDA cores only, so the result is
// comparable to the fp32 oracle within the reference's default tolerance.
//
// Parameters (compile-time -D defines, semantics of the paper's Sec. VI-A):
//   MWG, NWG, KWG   C tile per thread block (M x N) and K step per iteration
//   MDIMC, NDIMC    thread block; each thread owns an MWI x NWI register tile
//                   (MWI = MWG/MDIMC, NWI = NWG/NDIMC)
//   SA, SB          stage the A / B tile of each K step in shared memory
//   MDIMA, NDIMB    thread re-shape used for those shared-memory copies:
//                   MDIMA x KDIMA over the A tile, KDIMB x NDIMB over the B
//                   tile (KDIMA = MDIMC*NDIMC/MDIMA, KDIMB = MDIMC*NDIMC/NDIMB)
//   STRM, STRN      0: a thread's vectors along M (N) are contiguous;
//                   1: they are MDIMC (NDIMC) vectors apart -- consecutive
//                   threads then touch consecutive vectors
//   VWM, VWN        vector width of A (M) and B/C (N) accesses
//   KWI             unroll factor of the inner K loop
// C is N-contiguous, so output stores vectorize along N (VWN).

template <int N>
__device__ __forceinline__ void vload(float* d, const float* p) {
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
__device__ __forceinline__ void vload_g(float* d, const float* __restrict__ p) {
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
__device__ __forceinline__ void vstore(float* p, const float* s) {
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

// Asynchronous global -> shared copy of N floats (cp.async; 16-byte pieces
// bypass L1).  Used for double-buffered tiles: no staging registers.
template <int N>
__device__ __forceinline__ void cp_async(float* s, const float* __restrict__ g) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
    if (N == 1) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(g) : "memory");
    } else if (N == 2) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
    } else {
#pragma unroll
        for (int q = 0; q < N; q += 4)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + 4 * q), "l"(g + q)
                         : "memory");
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// acc[i][j] += a[i] * b[j] over an MI x NJ register tile.  PAIRED: the
// Blackwell packed FP32 FMA (FFMA2, fma.rn.f32x2): two independent
// round-to-nearest FMAs per instruction with one operand broadcast, so each
// lane's result is bit-identical to fmaf while the FMA-pipe issue count
// halves -- the SIMT SGEMM is issue-bound without it.  Pairs run along j
// (NJ even), else along i (MI even), else scalar.
template <int MI, int NJ, bool PAIRED>
__device__ __forceinline__ void outer_product_t(float (&acc)[MI][NJ], const float* a, const float* b) {
    if (PAIRED && NJ % 2 == 0) {
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; j += 2) {
                const float2 r = __ffma2_rn(make_float2(a[i], a[i]), make_float2(b[j], b[j + 1]),
                                            make_float2(acc[i][j], acc[i][j + 1]));
                acc[i][j] = r.x;
                acc[i][j + 1] = r.y;
            }
    } else if (PAIRED && MI % 2 == 0) {
#pragma unroll
        for (int i = 0; i < MI; i += 2)
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const float2 r = __ffma2_rn(make_float2(a[i], a[i + 1]), make_float2(b[j], b[j]),
                                            make_float2(acc[i][j], acc[i + 1][j]));
                acc[i][j] = r.x;
                acc[i + 1][j] = r.y;
            }
    } else {
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
}

//@@KTC_BODY@@ -- instantiated once per configuration; KTC_ENTRY names the kernel.
#ifndef DBUF  // host-chosen (backend.cpp plan_gemm): double-buffered cp.async tiles
#define DBUF 0
#define KTC_DBUF_DEFAULT
#endif
#define MWI (MWG / MDIMC)
#define NWI (NWG / NDIMC)
#define NT (MDIMC * NDIMC)
#define MVI (MWI / VWM)  // A vectors per thread per k
#define NVI (NWI / VWN)  // B vectors per thread per k

#if SA
#define KDIMA (NT / MDIMA)
#define KWA (KWG / KDIMA)
#define VA (MWG / VWM)                          // A vectors per k-row of the tile
#define MVA ((VA >= MDIMA) ? (VA / MDIMA) : 1)  // per copying thread
#define STAGE_A (KWA * MVA * VWM)
#else
#define STAGE_A 0
#endif
#if SB
#define KDIMB (NT / NDIMB)
#define KWB (KWG / KDIMB)
#define VB (NWG / VWN)
#define NVB ((VB >= NDIMB) ? (VB / NDIMB) : 1)
#define STAGE_B (KWB * NVB * VWN)
#else
#define STAGE_B 0
#endif
// Register double buffering of the shared-memory copies when their staging
// registers (per thread) stay small.
#define STAGE_REGS (STAGE_A + STAGE_B)
#define STAGE_AHEAD (STAGE_REGS <= 32)

// Occupancy target handed to ptxas (OCC=1, host-chosen): as many CTAs per SM
// as an estimate of the live registers (accumulators + one A/B fragment +
// addressing, + staging registers without DBUF) allows; OCC=0 leaves ptxas
// the whole 255-register budget.
#ifndef F2  // host-chosen: packed FFMA2 outer products
#define F2 1
#define KTC_F2_DEFAULT
#endif
#define outer_product(acc, a, b) outer_product_t<MWI, NWI, (F2 != 0)>(acc, a, b)
#ifndef OCC
#define OCC 0
#define KTC_OCC_DEFAULT
#endif
#define EST_REGS (MWI * NWI + (MWI + NWI) + 40 + (DBUF ? 0 : STAGE_REGS * STAGE_AHEAD))
#define MINB_RAW (65536 / (NT * EST_REGS))
#define MINB (OCC == 0 || MINB_RAW < 1 ? 1 : (MINB_RAW > 16 ? 16 : MINB_RAW))

extern "C" __global__ void __launch_bounds__(NT, MINB)
KTC_ENTRY(const int M, const int N, const int K, const float alpha, const float beta,
     const float* __restrict__ A, const float* __restrict__ B, const float* __restrict__ Cin,
     float* __restrict__ Cout) {
    const int tx = threadIdx.x;  // along M
    const int ty = threadIdx.y;  // along N
    const int m0 = blockIdx.x * MWG;
    const int n0 = blockIdx.y * NWG;

#if SA || SB
    extern __shared__ __align__(16) float smem[];
    const int tid = ty * MDIMC + tx;
#endif
#if SA
    float* alm = smem;  // [1 + DBUF][KWG][MWG]
#endif
#if SB
    float* blm = smem + SA * (1 + DBUF) * KWG * MWG;  // [1 + DBUF][KWG][NWG]
#endif

    float acc[MWI][NWI];
#pragma unroll
    for (int i = 0; i < MWI; ++i)
#pragma unroll
        for (int j = 0; j < NWI; ++j) acc[i][j] = 0.0f;

    // Shared-memory tiles are copied by the MDIMA x KDIMA (NDIMB x KDIMB)
    // thread re-shape.  DBUF (set by the host when two tiles fit): cp.async
    // straight into the other buffer while this one is consumed -- one
    // barrier per K step, no staging registers.  Otherwise the copy goes
    // through registers; when those are few, the NEXT K-tile's global loads
    // are issued before computing on the current one.
#if SA
    const int la0 = tid % MDIMA, la1 = tid / MDIMA;
    const bool a_copies = (VA >= MDIMA) || (la0 < VA);
#define A_SRC(kk0, kia, mv) (A + (size_t)((kk0) + la1 * KWA + (kia)) * M + m0 + (mv) * VWM)
#define A_DST(kia, mv) (((la1 * KWA + (kia)) * MWG) + (mv) * VWM)
#define A_MV(mia) (STRM ? (la0 + (mia) * MDIMA) : ((mia) + la0 * MVA))
#endif
#if SB
    const int lb0 = tid % NDIMB, lb1 = tid / NDIMB;
    const bool b_copies = (VB >= NDIMB) || (lb0 < VB);
#define B_SRC(kk0, kib, nv) (B + (size_t)((kk0) + lb1 * KWB + (kib)) * N + n0 + (nv) * VWN)
#define B_DST(kib, nv) (((lb1 * KWB + (kib)) * NWG) + (nv) * VWN)
#define B_MV(nib) (STRN ? (lb0 + (nib) * NDIMB) : ((nib) + lb0 * NVB))
#endif
#if DBUF
    auto issue = [&](int kk0, int buf) {
#if SA
        if (a_copies) {
#pragma unroll
            for (int kia = 0; kia < KWA; ++kia)
#pragma unroll
                for (int mia = 0; mia < MVA; ++mia)
                    cp_async<VWM>(alm + buf * KWG * MWG + A_DST(kia, A_MV(mia)), A_SRC(kk0, kia, A_MV(mia)));
        }
#endif
#if SB
        if (b_copies) {
#pragma unroll
            for (int kib = 0; kib < KWB; ++kib)
#pragma unroll
                for (int nib = 0; nib < NVB; ++nib)
                    cp_async<VWN>(blm + buf * KWG * NWG + B_DST(kib, B_MV(nib)), B_SRC(kk0, kib, B_MV(nib)));
        }
#endif
        cp_async_commit();
    };
    issue(0, 0);
#elif SA || SB
#if SA
    float ra[KWA][MVA * VWM];
#endif
#if SB
    float rb[KWB][NVB * VWN];
#endif
    auto fetch = [&](int kk0) {
#if SA
        if (a_copies) {
#pragma unroll
            for (int kia = 0; kia < KWA; ++kia)
#pragma unroll
                for (int mia = 0; mia < MVA; ++mia)
                    vload_g<VWM>(&ra[kia][mia * VWM], A_SRC(kk0, kia, A_MV(mia)));
        }
#endif
#if SB
        if (b_copies) {
#pragma unroll
            for (int kib = 0; kib < KWB; ++kib)
#pragma unroll
                for (int nib = 0; nib < NVB; ++nib)
                    vload_g<VWN>(&rb[kib][nib * VWN], B_SRC(kk0, kib, B_MV(nib)));
        }
#endif
    };
    auto stash = [&]() {
#if SA
        if (a_copies) {
#pragma unroll
            for (int kia = 0; kia < KWA; ++kia)
#pragma unroll
                for (int mia = 0; mia < MVA; ++mia)
                    vstore<VWM>(alm + A_DST(kia, A_MV(mia)), &ra[kia][mia * VWM]);
        }
#endif
#if SB
        if (b_copies) {
#pragma unroll
            for (int kib = 0; kib < KWB; ++kib)
#pragma unroll
                for (int nib = 0; nib < NVB; ++nib)
                    vstore<VWN>(blm + B_DST(kib, B_MV(nib)), &rb[kib][nib * VWN]);
        }
#endif
    };
    fetch(0);
#endif

    // One k-step's register fragments: MWI values of A and NWI of B, as
    // MVI (NVI) vectors of VWM (VWN), from the staged tile or from global.
#if SA
    const float* at = alm;
#endif
#if SB
    const float* bt = blm;
#endif
    int k0 = 0;
    auto load_frag = [&](float* a, float* b, int k) {
#pragma unroll
        for (int mi = 0; mi < MVI; ++mi) {
            const int mv = STRM ? (tx + mi * MDIMC) : (mi + tx * MVI);
#if SA
            vload<VWM>(a + mi * VWM, at + k * MWG + mv * VWM);
#else
            vload_g<VWM>(a + mi * VWM, A + (size_t)(k0 + k) * M + m0 + mv * VWM);
#endif
        }
#pragma unroll
        for (int ni = 0; ni < NVI; ++ni) {
            const int nv = STRN ? (ty + ni * NDIMC) : (ni + ty * NVI);
#if SB
            vload<VWN>(b + ni * VWN, bt + k * NWG + nv * VWN);
#else
            vload_g<VWN>(b + ni * VWN, B + (size_t)(k0 + k) * N + n0 + nv * VWN);
#endif
        }
    };

    int buf = 0;
#pragma unroll 1
    for (k0 = 0; k0 < K; k0 += KWG) {
#if DBUF
        cp_async_wait_all();
        __syncthreads();  // tile k0 landed; everyone is done with the other buffer
        if (k0 + KWG < K) issue(k0 + KWG, buf ^ 1);
#elif SA || SB
        stash();
        __syncthreads();
#if STAGE_AHEAD
        if (k0 + KWG < K) fetch(k0 + KWG);
#endif
#endif
#if SA
        at = alm + DBUF * buf * KWG * MWG;
#endif
#if SB
        bt = blm + DBUF * buf * KWG * NWG;
#endif

#pragma unroll 1
        for (int kw = 0; kw < KWG; kw += KWI) {
#pragma unroll
            for (int ki = 0; ki < KWI; ++ki) {
                float a[MWI], b[NWI];
                load_frag(a, b, kw + ki);
                outer_product(acc, a, b);
            }
        }
#if !DBUF && (SA || SB)
        __syncthreads();
#if !STAGE_AHEAD
        if (k0 + KWG < K) fetch(k0 + KWG);
#endif
#endif
        buf ^= 1;
    }

    // Epilogue: Cout = alpha * acc + beta * Cin, VWN-wide stores along N.
#pragma unroll
    for (int mi = 0; mi < MVI; ++mi) {
        const int mv = STRM ? (tx + mi * MDIMC) : (mi + tx * MVI);
#pragma unroll
        for (int e = 0; e < VWM; ++e) {
            const int m = m0 + mv * VWM + e;
#pragma unroll
            for (int ni = 0; ni < NVI; ++ni) {
                const int nv = STRN ? (ty + ni * NDIMC) : (ni + ty * NVI);
                const size_t idx = (size_t)m * N + n0 + nv * VWN;
                float s[VWN];
                if (beta != 0.0f) {
                    float c[VWN];
                    vload_g<VWN>(c, Cin + idx);
#pragma unroll
                    // Explicit fmaf: the contraction is fixed (NVVM would
                    // otherwise pick either product per configuration).
                    for (int q = 0; q < VWN; ++q) s[q] = fmaf(alpha, acc[mi * VWM + e][ni * VWN + q], beta * c[q]);
                } else {
#pragma unroll
                    for (int q = 0; q < VWN; ++q) s[q] = alpha * acc[mi * VWM + e][ni * VWN + q];
                }
                vstore<VWN>(Cout + idx, s);
            }
        }
    }
}
#undef MWI
#undef NWI
#undef NT
#undef MVI
#undef NVI
#undef KDIMA
#undef KWA
#undef VA
#undef MVA
#undef KDIMB
#undef KWB
#undef VB
#undef NVB
#undef STAGE_REGS
#undef STAGE_A
#undef STAGE_B
#undef STAGE_AHEAD
#undef A_SRC
#undef A_DST
#undef A_MV
#undef B_SRC
#undef B_DST
#undef B_MV
#undef EST_REGS
#undef MINB_RAW
#undef MINB
#ifdef KTC_OCC_DEFAULT
#undef OCC
#undef KTC_OCC_DEFAULT
#endif
#undef outer_product
#ifdef KTC_F2_DEFAULT
#undef F2
#undef KTC_F2_DEFAULT
#endif
#ifdef KTC_DBUF_DEFAULT
#undef DBUF
#undef KTC_DBUF_DEFAULT
#endif
