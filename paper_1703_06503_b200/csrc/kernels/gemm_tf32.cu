// gemm_tf32.cu -- SGEMM on the 5th-generation tensor cores (tcgen05, TF32
// inputs, fp32 accumulation in TMEM), the B200 variant of the SGEMM family
// (kernel name "gemm_tf32", reported separately from the fp32 CUDA-core
// family, verified with its own tolerance rel 1e-3).  Same problem and
// argument list as gemm.cu:
//     Cout[m*N + n] = ALPHA * sum_k A[k*M + m] * B[k*N + n] + BETA * Cin[m*N + n]
//
// A (K x M, M contiguous) and B (K x N, N contiguous) are both MN-major
// operands, which UMMA accepts for TF32, so no transpose pass is needed:
//
//   TMA   A tile 128(M) x BK(K) as 4 boxes of 32 x BK, B tile BN x BK as
//         BN/32 boxes, SWIZZLE_128B: each box is BK rows of 128 B, i.e. the
//         canonical MN-major SW128 atom (8 K-rows x 128 B) stacked along K;
//   ring  STAGES stages of A+B, full/empty mbarriers per stage;
//   MMA   one elected lane of warp 1 issues tcgen05.mma.cta_group::1.kind::tf32
//         (M=128, N=BN, K=8) for each 8-row K group, accumulating into a
//         128-lane x BN-column fp32 TMEM tile; tcgen05.commit releases the
//         stage and finally signals the epilogue;
//   epi   all 4 warps: tcgen05.ld 32x32b (warp w owns TMEM lanes 32w..32w+31
//         = rows), alpha/beta, 128-byte row segments stored to global.
//
// Parameters: BN (64, 128, 256), BK (32, 64), STAGES (2, 3, 4, 6), CG (1, 2:
// CTA pair, tcgen05.mma.cta_group::2 with M = 256 -- half the operand bytes
// per SM of a 128 x BN tile, the L2 -> SM traffic that bounds the 1-CTA
// kernel at 2048^3).  The tensor core reads the fp32 operand bits as TF32
// (truncating the low 13 mantissa bits), hence the variant's own tolerance.
// Block: 128 threads; grid (M/128, N/BN), clusters of CG CTAs along x.


typedef unsigned int u32;
typedef unsigned long long u64;

struct __align__(64) TensorMap {
    unsigned long long v[16];
};

__device__ __forceinline__ u32 smem_u32(const void* p) {
    return static_cast<u32>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
    for (long long spin = 0; spin < (1ll << 28); ++spin) {
        u32 done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
    }
    __trap();  // a lost transaction becomes a launch error, never a hang
}

__device__ __forceinline__ void tma_load_2d(u32 dst, const TensorMap* map, u32 bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<u64>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}

// CTA-pair (cta_group::2) forms: the TMA of either CTA completes its bytes on
// the leader's barrier (a shared::cluster address from mapa), and the
// leader's MMA commit arrives on the same-offset barrier of both CTAs.
__device__ __forceinline__ void tma_load_2d_pair(u32 dst, const TensorMap* map, u32 bar_cluster,
                                                 int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<u64>(map)), "r"(bar_cluster), "r"(x), "r"(y)
        : "memory");
}

__device__ __forceinline__ u32 mapa_rank(u32 addr, u32 rank) {
    u32 out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
    return out;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__device__ __forceinline__ u32 cluster_rank() {
    u32 r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void umma_tf32_pair(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc,
                                               u32 accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit_pair(u32 bar) {
    const unsigned short mask = 3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar),
        "h"(mask)
        : "memory");
}

// TMA store of a staged smem box (bulk-group completion).
__device__ __forceinline__ void tma_store_2d(const TensorMap* map, u32 src, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
            reinterpret_cast<u64>(map)),
        "r"(src), "r"(x), "r"(y)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Stream-K helpers.
__device__ __forceinline__ void tmem_ld32(u32 taddr, u32 (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Arrive on an mbarrier of any CTA of the cluster (shared::cluster address).
__device__ __forceinline__ void mbar_arrive_cluster(u32 bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_local(u32 bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void named_sync(u32 id, u32 n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// UMMA shared-memory descriptor for MN-major 32-bit operands (sm_100): the
// only layout UMMA accepts for MN-major TF32 is SWIZZLE_128B_BASE32B
// (128-byte MN rows, 32-byte swizzle atoms over 4-row K groups), which is
// what TMA's SWIZZLE_128B_ATOM_32B mode writes.  Fields: start>>4 [0,14),
// LBO>>4 [16,30) = stride between 32-element MN atoms, SBO>>4 [32,46) =
// stride between 4-row K groups, version 1 at [46,48), layout type 1 at
// [61,64).
__device__ __forceinline__ u64 umma_desc(u32 addr, u32 lbo, u32 sbo) {
    u64 d = 0;
    d |= (u64)((addr >> 4) & 0x3FFF);
    d |= (u64)((lbo >> 4) & 0x3FFF) << 16;
    d |= (u64)((sbo >> 4) & 0x3FFF) << 32;
    d |= (u64)1 << 46;
    d |= (u64)1 << 61;
    return d;
}

// Instruction descriptor: D f32, A/B tf32, both MN-major, M = m (128, or
// 256 for a CTA pair), N = bn.
__device__ __forceinline__ u32 make_idesc(u32 m, u32 bn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((bn >> 3) << 17) |
           ((m >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc,
                                          u32 accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit(u32 bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}

//@@KTC_BODY@@ -- instantiated once per configuration; KTC_ENTRY names the kernel.
// CG = 1: one CTA per 128 x BN tile.  CG = 2: a CTA pair (cluster of 2 along
// x, same TPC) per 256 x BN tile: CTA r loads A rows m0 + 128r.. and B
// columns n0 + r*BN/2.., the leader (r = 0) issues M=256 MMAs that read both
// CTAs' shared memory, and each CTA's TMEM receives its own 128 rows x BN.
#define BM 128
#define NT 128
#define BNL (BN / CG)
#define A_BOX_BYTES (BK * 128)
#define A_STAGE_BYTES (4 * A_BOX_BYTES)
#define B_STAGE_BYTES ((BNL / 32) * A_BOX_BYTES)
#define STAGE_BYTES (A_STAGE_BYTES + B_STAGE_BYTES)
#define TMEM_COLS (BN < 32 ? 32 : BN)

#if !SK
extern "C" __global__ void __launch_bounds__(NT, 1)
#if CG == 2
__cluster_dims__(2, 1, 1)
#endif
KTC_ENTRY(const int M, const int N, const int K, const float alpha, const float beta,
          const float* __restrict__ A, const float* __restrict__ B,
          const float* __restrict__ Cin, float* __restrict__ Cout,
          const __grid_constant__ TensorMap tmap_a, const __grid_constant__ TensorMap tmap_b,
          const __grid_constant__ TensorMap tmap_c) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B atoms (same offset in both CTAs
    // of a pair: the leader's MMA descriptors address the peer's operands).
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<u64>(smem_raw) + 1023) & ~u64(1023));
    u64* bars = reinterpret_cast<u64*>(smem + STAGES * STAGE_BYTES);  // full[S], empty[S], acc
    u32* tmem_slot = reinterpret_cast<u32*>(bars + 2 * STAGES + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u32 rank = CG == 2 ? cluster_rank() : 0u;
    // Grouped rasterisation: clusters are launched x-fastest; tile (mp, np)
    // of the pid-th cluster walks GROUP_M tile-rows per column so that the
    // clusters resident at one time share A rows and B columns in L2 (at
    // 8192^3 the plain order re-read A from DRAM about once per wave).
    const int GROUP_M = 8;
    const int nmp = gridDim.x / CG;  // tile-rows (CTA pairs for CG = 2)
    const int pid = blockIdx.y * nmp + blockIdx.x / CG;
    const int span = GROUP_M * gridDim.y;
    const int first = (pid / span) * GROUP_M;
    const int rows = min(nmp - first, GROUP_M);
    const int mp = first + (pid % span) % rows, np = (pid % span) / rows;
    const int m0 = (mp * CG + (int)rank) * BM, n0 = np * BN;
    const int kblocks = K / BK;
    const u32 full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES),
              accb = smem_u32(bars + 2 * STAGES);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(accb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<u64>(&tmap_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<u64>(&tmap_b)) : "memory");
    }
    if (warp == 1) {  // TMEM allocation: one warp (the same warp in both CTAs of a pair)
#if CG == 2
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"((u32)TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
#else
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"((u32)TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
#endif
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
#if CG == 2
    cluster_sync_all();  // both CTAs' barriers exist before any cross-CTA arrive
#else
    __syncthreads();
#endif
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = *tmem_slot;

    // Warp 0 produces, warp 1 issues the MMAs: one elected lane does the
    // work, the rest of the warp stays converged with it (__syncwarp per
    // K-block) instead of spinning on the accumulator barrier, which would
    // split the warp and steal issue slots from the elected lane.
    if (warp == 0) {
        // ---- TMA producer (both CTAs of a pair; bytes land on the leader's full barrier) ----
        for (int kb = 0; kb < kblocks; ++kb) {
            if (lane == 0) {
                const int s = kb % STAGES;
                const u32 phase = (u32)((kb / STAGES) & 1);
                mbar_wait(empty0 + 8 * s, phase ^ 1u);
                const u32 full = full0 + 8 * s;
                if (rank == 0) mbar_expect_tx(full, CG * STAGE_BYTES);
                const u32 sa = smem_u32(smem + s * STAGE_BYTES);
                const u32 sb = sa + A_STAGE_BYTES;
#if CG == 2
                const u32 fullc = mapa_rank(full, 0);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    tma_load_2d_pair(sa + j * A_BOX_BYTES, &tmap_a, fullc, m0 + 32 * j, kb * BK);
#pragma unroll
                for (int j = 0; j < BNL / 32; ++j)
                    tma_load_2d_pair(sb + j * A_BOX_BYTES, &tmap_b, fullc,
                                     n0 + (int)rank * BNL + 32 * j, kb * BK);
#else
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    tma_load_2d(sa + j * A_BOX_BYTES, &tmap_a, full, m0 + 32 * j, kb * BK);
#pragma unroll
                for (int j = 0; j < BN / 32; ++j)
                    tma_load_2d(sb + j * A_BOX_BYTES, &tmap_b, full, n0 + 32 * j, kb * BK);
#endif
            }
            __syncwarp();
        }
    } else if (warp == 1 && rank == 0) {
        // ---- MMA issuer (one elected thread of the leader CTA) ----
        for (int kb = 0; kb < kblocks; ++kb) {
            if (lane == 0) {
                const int s = kb % STAGES;
                mbar_wait(full0 + 8 * s, (u32)((kb / STAGES) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const u32 sa = smem_u32(smem + s * STAGE_BYTES);
                const u32 sb = sa + A_STAGE_BYTES;
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    // K = 8 per MMA = two 4-row groups of 512 B.
                    const u64 ad = umma_desc(sa + kk * 1024, A_BOX_BYTES, 512);
                    const u64 bd = umma_desc(sb + kk * 1024, A_BOX_BYTES, 512);
#if CG == 2
                    umma_tf32_pair(tmem, ad, bd, make_idesc(256, BN), (kb | kk) != 0 ? 1u : 0u);
#else
                    umma_tf32(tmem, ad, bd, make_idesc(128, BN), (kb | kk) != 0 ? 1u : 0u);
#endif
                }
#if CG == 2
                umma_commit_pair(empty0 + 8 * s);  // both CTAs' stage s reusable
#else
                umma_commit(empty0 + 8 * s);  // stage reusable once these MMAs retire
#endif
            }
            __syncwarp();
        }
#if CG == 2
        if (lane == 0) umma_commit_pair(accb);  // both accumulator halves complete
#else
        if (lane == 0) umma_commit(accb);  // accumulator complete
#endif
        __syncwarp();
    }

    // ---- epilogue: all warps (each CTA of a pair owns 128 rows x BN in its TMEM) ----
    mbar_wait(accb, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = warp * 32 + lane;  // TMEM lane == tile row
    if (beta == 0.0f) {
        // Stores through TMA: each 128-row x 32-column chunk is staged in the
        // now idle operand ring (two 16 KB buffers, 128-byte swizzle so the
        // row-per-thread writes are bank-conflict free) and written by one
        // bulk tensor store of full lines, overlapping the next chunk's
        // TMEM load.
        const u32 stg = smem_u32(smem);
        int buf = 0;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32, buf ^= 1) {
            u32 v[32];
            tmem_ld32(tmem + ((u32)(warp * 32) << 16) + (u32)c0, v);
            if (threadIdx.x == 0 && c0 >= 64)
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer free
            __syncthreads();
            const u32 sb = stg + (u32)buf * 16384u + (u32)row * 128u;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const u32 dst = sb + (u32)((q ^ (row & 7)) << 4);
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst),
                             "f"(alpha * __uint_as_float(v[4 * q])),
                             "f"(alpha * __uint_as_float(v[4 * q + 1])),
                             "f"(alpha * __uint_as_float(v[4 * q + 2])),
                             "f"(alpha * __uint_as_float(v[4 * q + 3]))
                             : "memory");
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) tma_store_2d(&tmap_c, stg + (u32)buf * 16384u, n0 + c0, m0);
        }
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else {
    float* crow = Cout + (size_t)(m0 + row) * N + n0;
    const float* cin = Cin + (size_t)(m0 + row) * N + n0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
        u32 v[32];
        tmem_ld32(tmem + ((u32)(warp * 32) << 16) + (u32)c0, v);
#pragma unroll
        for (int q = 0; q < 32; q += 4) {
            float4 o;
            o.x = alpha * __uint_as_float(v[q]);
            o.y = alpha * __uint_as_float(v[q + 1]);
            o.z = alpha * __uint_as_float(v[q + 2]);
            o.w = alpha * __uint_as_float(v[q + 3]);
            const float4 c = __ldg(reinterpret_cast<const float4*>(cin + c0 + q));
            o.x += beta * c.x;
            o.y += beta * c.y;
            o.z += beta * c.z;
            o.w += beta * c.w;
            *reinterpret_cast<float4*>(crow + c0 + q) = o;
        }
    }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
#if CG == 2
    cluster_sync_relaxed();  // neither CTA frees TMEM / exits while its pair is still reading
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"((u32)TMEM_COLS)
                     : "memory");
    }
#else
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"((u32)TMEM_COLS)
                     : "memory");
    }
#endif
}
#else
// ---- SK (host switch): stream-K over persistent CTAs / CTA pairs.  The
// pair-tiles x K-blocks units are dealt as contiguous ranges [c*U/G,
// (c+1)*U/G) to the G resident clusters; a cluster walks its range as
// segments (one per tile it touches).  Warp 0 produces (TMA), warp 1 of the
// leader issues the MMAs, warps 2-5 are the epilogue (TMEM lane quarter =
// warp % 4).  A whole-tile segment stores the output; a partial one stores
// its 128 x BN partial in workspace slot ((tile*CG + rank)*MAXSEG + j), and
// the last segment of the tile to arrive (counter) sums the partials in
// segment order (its own re-read from TMEM: deterministic) and stores the
// output.  TMEM is handed back to the MMA warp through tmem_empty.
#define NTH 192
extern "C" __global__ void __launch_bounds__(NTH, 1)
#if CG == 2
__cluster_dims__(2, 1, 1)
#endif
KTC_ENTRY(const int M, const int N, const int K, const float alpha, const float beta,
          const float* __restrict__ A, const float* __restrict__ B,
          const float* __restrict__ Cin, float* __restrict__ Cout,
          const __grid_constant__ TensorMap tmap_a, const __grid_constant__ TensorMap tmap_b,
          const __grid_constant__ TensorMap tmap_c, float* __restrict__ W, unsigned* __restrict__ cnt, const unsigned U,
          const unsigned maxseg, const unsigned ntm, const unsigned KB) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<u64>(smem_raw) + 1023) & ~u64(1023));
    // full[S], empty[S], acc[2], tmem_empty[2], partial-staging barrier: the
    // accumulator is double-buffered in TMEM (2 x BN columns), so the MMAs of
    // segment s+1 run while the epilogue drains segment s.
    u64* bars = reinterpret_cast<u64*>(smem + STAGES * STAGE_BYTES);
    u32* tmem_slot = reinterpret_cast<u32*>(bars + 2 * STAGES + 5);
    volatile u32* flag = tmem_slot + 1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u32 rank = CG == 2 ? cluster_rank() : 0u;
    const unsigned c = blockIdx.x / CG, G = gridDim.x / CG;
#if SKTRACE
    // diagnostic timeline (KTC_TF32_SK_TRACE): 16 u64 per CTA after the partial slots
    unsigned long long* dbg = reinterpret_cast<unsigned long long*>(
                                  W + (size_t)(U / KB) * CG * maxseg * (BM * BN)) +
                              (size_t)blockIdx.x * 16;
    if (threadIdx.x == 0) dbg[0] = gtimer();
#define SKT(i) dbg[i] = gtimer()
#else
#define SKT(i)
#endif
    const unsigned u0 = (unsigned)((unsigned long long)c * U / G);
    const unsigned u1 = (unsigned)((unsigned long long)(c + 1) * U / G);
    const u32 full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES),
              accb = smem_u32(bars + 2 * STAGES), tempty = smem_u32(bars + 2 * STAGES + 2),
              pbar = smem_u32(bars + 2 * STAGES + 4);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(accb, 1);
        mbar_init(accb + 8, 1);
        mbar_init(tempty, CG);  // one arrival per CTA's epilogue group
        mbar_init(tempty + 8, CG);
        mbar_init(pbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<u64>(&tmap_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<u64>(&tmap_b)) : "memory");
    }
    if (warp == 1) {
#if CG == 2
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"((u32)(2 * TMEM_COLS))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
#else
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"((u32)(2 * TMEM_COLS))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
#endif
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
#if CG == 2
    cluster_sync_all();
#else
    __syncthreads();
#endif
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = *tmem_slot;

    if (warp == 0) {
        // ---- TMA producer: the cluster's units in order (runs ahead across segments)
        unsigned it = 0;
        for (unsigned u = u0; u < u1; ++u, ++it) {
            if (lane == 0) {
                const unsigned t = u / KB, kb = u - t * KB;
                const unsigned mp = t % ntm, np = t / ntm;
                const int m0 = (int)((mp * CG + rank) * BM), n0 = (int)(np * BN);
                const int s = (int)(it % STAGES);
                const u32 phase = (it / STAGES) & 1u;
                mbar_wait(empty0 + 8 * s, phase ^ 1u);
                const u32 full = full0 + 8 * s;
                if (rank == 0) mbar_expect_tx(full, CG * STAGE_BYTES);
                const u32 sa = smem_u32(smem + s * STAGE_BYTES);
                const u32 sb = sa + A_STAGE_BYTES;
#if CG == 2
                const u32 fullc = mapa_rank(full, 0);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    tma_load_2d_pair(sa + j * A_BOX_BYTES, &tmap_a, fullc, m0 + 32 * j, (int)kb * BK);
#pragma unroll
                for (int j = 0; j < BNL / 32; ++j)
                    tma_load_2d_pair(sb + j * A_BOX_BYTES, &tmap_b, fullc,
                                     n0 + (int)rank * BNL + 32 * j, (int)kb * BK);
#else
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    tma_load_2d(sa + j * A_BOX_BYTES, &tmap_a, full, m0 + 32 * j, (int)kb * BK);
#pragma unroll
                for (int j = 0; j < BN / 32; ++j)
                    tma_load_2d(sb + j * A_BOX_BYTES, &tmap_b, full, n0 + 32 * j, (int)kb * BK);
#endif
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ---- MMA issuer (leader CTA, one elected lane), one accumulator per segment
        if (rank == 0) {
            unsigned it = 0, seg = 0;
            for (unsigned u = u0; u < u1; ++seg) {
                const unsigned t = u / KB, kb0 = u - t * KB;
                const unsigned kb1 = min(KB, kb0 + (u1 - u));
                const u32 buf = seg & 1u;
                if (lane == 0) {
                    // TMEM buffer `buf` was last used by segment seg-2
                    if (seg >= 2) mbar_wait(tempty + 8 * buf, ((seg >> 1) - 1) & 1u);
                    if (seg < 3) SKT(2 + seg * 4);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    for (unsigned kb = kb0; kb < kb1; ++kb, ++it) {
                        const int s = (int)(it % STAGES);
                        mbar_wait(full0 + 8 * s, (it / STAGES) & 1u);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const u32 sa = smem_u32(smem + s * STAGE_BYTES);
                        const u32 sb = sa + A_STAGE_BYTES;
#pragma unroll
                        for (int kk = 0; kk < BK / 8; ++kk) {
                            const u64 ad = umma_desc(sa + kk * 1024, A_BOX_BYTES, 512);
                            const u64 bd = umma_desc(sb + kk * 1024, A_BOX_BYTES, 512);
                            const u32 acc = (kb != kb0 || kk != 0) ? 1u : 0u;
#if CG == 2
                            umma_tf32_pair(tmem + buf * BN, ad, bd, make_idesc(256, BN), acc);
#else
                            umma_tf32(tmem + buf * BN, ad, bd, make_idesc(128, BN), acc);
#endif
                        }
#if CG == 2
                        umma_commit_pair(empty0 + 8 * s);
#else
                        umma_commit(empty0 + 8 * s);
#endif
                    }
#if CG == 2
                    umma_commit_pair(accb + 8 * buf);
#else
                    umma_commit(accb + 8 * buf);
#endif
                    if (seg < 3) SKT(3 + seg * 4);
                } else {
                    it += kb1 - kb0;
                }
                __syncwarp();
                u += kb1 - kb0;
            }
        }
    } else {
        // ---- epilogue warps 2..5: TMEM lane quarter = warp % 4 (hardware rule)
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const bool lead = (warp == 2 && lane == 0);
        const u32 tempty_leader = CG == 2 ? mapa_rank(tempty, 0) : tempty;
        int sbuf = 0;  // TMA-store staging buffer (output through the idle ring)
        unsigned seg = 0, pphase = 0;
        for (unsigned u = u0; u < u1; ++seg) {
            const unsigned t = u / KB, kb0 = u - t * KB;
            const unsigned kb1 = min(KB, kb0 + (u1 - u));
            const unsigned mp = t % ntm, np = t / ntm;
            const int m0 = (int)((mp * CG + rank) * BM), n0 = (int)(np * BN);
            // segments of tile t: the clusters holding its first and last unit
            const unsigned first = (unsigned)(((unsigned long long)(t * KB + 1) * G - 1) / U);
            const unsigned last = (unsigned)(((unsigned long long)((t + 1) * KB) * G - 1) / U);
            const unsigned nseg = last - first + 1, j = c - first;
            const u32 buf = seg & 1u;
            mbar_wait(accb + 8 * buf, (seg >> 1) & 1u);
            if (lead && seg < 3) SKT(4 + seg * 4);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const u32 trow = tmem + ((u32)(q * 32) << 16) + buf * BN;
            float* crow = Cout + (size_t)(m0 + row) * N + n0;
            const float* cin = Cin + (size_t)(m0 + row) * N + n0;
            bool final_tile = nseg == 1;
            float* wbase = W + (size_t)(t * CG + rank) * maxseg * (size_t)(BM * BN);
            if (!final_tile) {
                // Partials column-major within the tile (element (row, col) at
                // col * BM + row): the 32 lanes of a warp hold 32 consecutive
                // rows, so every store / load below is one 128-byte line.
                float* wmine = wbase + (size_t)j * (BM * BN) + row;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    u32 v[32];
                    tmem_ld32(trow + (u32)c0, v);
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        __stcg(wmine + (size_t)(c0 + e) * BM, __uint_as_float(v[e]));
                }
                // publish: the group's stores are ordered before the lead's
                // release fence by the barrier (cumulativity), then count
                named_sync(1, 128);
                if (lead) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    *flag = atomicAdd(&cnt[t * CG + rank], 1u);
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
                named_sync(1, 128);
                final_tile = *flag == nseg - 1;
                if (final_tile && lead) cnt[t * CG + rank] = 0u;  // ready for the next launch
            }
            // The other segments' partials, half a tile at a time, staged by
            // bulk copies into the operand ring -- free once this is the
            // cluster's last segment (all its loads consumed) -- so the sum
            // reads shared memory instead of latency-bound global loads.
            constexpr unsigned HALF = BM * (BN / 2) * 4;
            const bool last_seg = u + (kb1 - kb0) >= u1;  // the operand ring is idle
            const bool staged = final_tile && nseg > 1 && last_seg &&
                                (nseg - 1) * HALF <= (unsigned)(STAGES * STAGE_BYTES);
            // Output through TMA stores from the idle ring (as in the one-tile
            // kernel) when beta == 0 and two 16 KB staging buffers fit after
            // the staged partials.
            const u32 stg_base = smem_u32(smem) + (staged ? (nseg - 1) * HALF : 0u);
            const bool tma_out = final_tile && last_seg && beta == 0.0f &&
                                 (staged ? (nseg - 1) * HALF : 0u) + 32768u <=
                                     (unsigned)(STAGES * STAGE_BYTES);
            // one 128 x 32 output chunk: registers -> swizzled staging -> bulk store
            auto out_chunk = [&](int c0, const float (&acc)[32]) {
                if (tma_out) {
                    if (lead) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    named_sync(1, 128);
                    const u32 sb = stg_base + (u32)sbuf * 16384u + (u32)row * 128u;
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq) {
                        const u32 dst = sb + (u32)((qq ^ (row & 7)) << 4);
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst),
                                     "f"(alpha * acc[4 * qq]), "f"(alpha * acc[4 * qq + 1]),
                                     "f"(alpha * acc[4 * qq + 2]), "f"(alpha * acc[4 * qq + 3])
                                     : "memory");
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    named_sync(1, 128);
                    if (lead) tma_store_2d(&tmap_c, stg_base + (u32)sbuf * 16384u, n0 + c0, m0);
                    sbuf ^= 1;
                } else {
#pragma unroll
                    for (int e = 0; e < 32; e += 4) {
                        float4 o;
                        o.x = alpha * acc[e];
                        o.y = alpha * acc[e + 1];
                        o.z = alpha * acc[e + 2];
                        o.w = alpha * acc[e + 3];
                        if (beta != 0.0f) {
                            const float4 cc = __ldg(reinterpret_cast<const float4*>(cin + c0 + e));
                            o.x += beta * cc.x;
                            o.y += beta * cc.y;
                            o.z += beta * cc.z;
                            o.w += beta * cc.w;
                        }
                        *reinterpret_cast<float4*>(crow + c0 + e) = o;
                    }
                }
            };
            if (staged) {
                const u32 ring = smem_u32(smem);
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    if (lead) {
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        mbar_expect_tx(pbar, (nseg - 1) * HALF);
                        unsigned k = 0;
                        for (unsigned i = 0; i < nseg; ++i) {
                            if (i == j) continue;
                            const float* src = wbase + (size_t)i * (BM * BN) + (size_t)h * (BM * (BN / 2));
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                                " [%0], [%1], %2, [%3];" ::"r"(ring + k * HALF),
                                "l"(reinterpret_cast<u64>(src)), "r"(HALF), "r"(pbar)
                                : "memory");
                            ++k;
                        }
                    }
                    mbar_wait(pbar, pphase);
                    pphase ^= 1u;
                    const float* sp = reinterpret_cast<const float*>(smem);
#pragma unroll 1
                    for (int c0 = h * (BN / 2); c0 < (h + 1) * (BN / 2); c0 += 32) {
                        u32 v[32];
                        tmem_ld32(trow + (u32)c0, v);
                        float acc[32];
#pragma unroll
                        for (int e = 0; e < 32; ++e) acc[e] = 0.0f;
                        unsigned k = 0;
                        for (unsigned i = 0; i < nseg; ++i) {
                            if (i == j) {
#pragma unroll
                                for (int e = 0; e < 32; ++e) acc[e] += __uint_as_float(v[e]);
                            } else {
                                const float* q = sp + (size_t)k * (HALF / 4) +
                                                 (size_t)(c0 - h * (BN / 2)) * BM + row;
#pragma unroll
                                for (int e = 0; e < 32; ++e) acc[e] += q[(size_t)e * BM];
                                ++k;
                            }
                        }
                        out_chunk(c0, acc);
                    }
                    named_sync(1, 128);  // the ring is read before the next half lands
                }
            } else if (final_tile) {
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    u32 v[32];
                    tmem_ld32(trow + (u32)c0, v);
                    float acc[32];
                    if (nseg == 1) {
#pragma unroll
                        for (int e = 0; e < 32; ++e) acc[e] = __uint_as_float(v[e]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e) acc[e] = 0.0f;
                        for (unsigned i = 0; i < nseg; ++i) {
                            if (i == j) {
#pragma unroll
                                for (int e = 0; e < 32; ++e) acc[e] += __uint_as_float(v[e]);
                            } else {
                                const float* wp = wbase + (size_t)i * (BM * BN) + row;
#pragma unroll
                                for (int e = 0; e < 32; ++e)
                                    acc[e] += __ldcg(wp + (size_t)(c0 + e) * BM);
                            }
                        }
                    }
                    out_chunk(c0, acc);
                }
            }
            if (tma_out && lead) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            // hand TMEM back to the MMA warp (one arrival per CTA)
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            named_sync(1, 128);
            if (lead) mbar_arrive_cluster(tempty_leader + 8 * buf);
            if (lead && seg < 3) SKT(5 + seg * 4);
            u += kb1 - kb0;
        }
    }
    if (warp == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
#if CG == 2
    cluster_sync_relaxed();
#else
    __syncthreads();
#endif
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1) {
#if CG == 2
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"((u32)(2 * TMEM_COLS))
                     : "memory");
#else
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"((u32)(2 * TMEM_COLS))
                     : "memory");
#endif
    }
#if SKTRACE
    if (threadIdx.x == 0) {
        dbg[14] = gtimer();
        u32 sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        dbg[15] = sm;
    }
#endif
}
#undef SKT
#undef NTH
#endif
#undef BM
#undef NT
#undef BNL
#undef A_BOX_BYTES
#undef A_STAGE_BYTES
#undef B_STAGE_BYTES
#undef STAGE_BYTES
#undef TMEM_COLS
