// atax_cluster.cuh -- single-pass ATAX / BATAX:  y = [beta] A'(A x), A read from HBM ONCE.
//
// The reference contracts t = A x to a per-row scalar by running the two j
// loops of a row back to back, the second touch of the row coming from the
// CPU cache ({_i{_j 1}{_j 2}}, fuse.py:660-688).
// A 32768-double row is 256 KiB -- more than one SM's shared memory -- so here
// a thread-block CLUSTER of C CTAs holds a panel of RG rows between them:
//
//   CTA k of the cluster owns columns [k*W, (k+1)*W) of every row of the panel
//   and keeps them in shared memory, filled by TMA bulk copies
//   (cp.async.bulk, one per row segment, completion on an mbarrier) through an
//   S-stage ring, so S-1 panels are always in flight while one is consumed;
//   phase 1  every CTA reduces its slice of the row dots (registers -> warp
//            shuffle -> shared memory) and PUSHES its partial sums into the
//            shared memory of every CTA of the cluster with st.async, which
//            counts the bytes on the RECEIVER's mbarrier for that panel;
//   phase 2  L panels later (software pipeline: the exchange latency is hidden
//            behind L iterations of work, no lock-step cluster barrier) every
//            CTA waits on its own mbarrier, adds the C partials in rank order
//            (t_i, identical bits in all CTAs), then y[j] += A[i,j] * t_i from
//            the SAME shared-memory tile, column sums living in registers for
//            the whole kernel.
// A ninth warp is the TMA producer: it refills a stage as soon as the eight
// consumer warps have released it (an "empty" mbarrier per stage).
//
// HBM traffic is therefore 8*M*N bytes + the y partials (one N-vector per
// cluster), the algorithmic minimum of SURVEY.md section 8d.  Clusters take
// contiguous row ranges (the reference's block formula); a finaliser adds the
// per-cluster y partials in ascending order.
#pragma once
#include "common.cuh"

namespace bto {

struct AtaxArgs {
    const double *A;
    const double *x;
    double *ypart;       // [nclusters][N]
    long M, N;
    int W;               // columns per CTA (even)
    int stages;          // ring depth S
    int rows;            // rows per panel (<= the kernel's RG bound)
    int lookahead;       // L: phase 1 runs L panels ahead of phase 2 (1..3, <= stages-2)
    int nclusters;
};

constexpr int kAtaxMaxCluster = 16;
constexpr int kAtaxMaxRows = 8;
constexpr int kAtaxMaxStages = 8;
constexpr int kAtaxSlots = 8;                      // exchange slots; needs > 2*L + 1
constexpr int kAtaxThreads = kThreads + 32;        // 8 consumer warps + 1 producer warp

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// TMA 1-D bulk copy global -> shared, completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes,
                                          uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Asynchronous remote store: write `v` into the same-named shared variable of
// CTA `rank` and count 8 bytes on that CTA's mbarrier when the data has landed.
// The mbarrier's tx-count carries the ordering, so neither side needs a
// cluster-scope fence (a release/acquire pair at cluster scope costs far more
// than the store itself).
__device__ __forceinline__ void st_async_cluster(double *local, uint64_t *local_bar,
                                                 uint32_t rank, double v)
{
    uint32_t raddr, rbar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(local_bar)), "r"(rank));
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
                 ::"r"(raddr), "d"(v), "r"(rbar)
                 : "memory");
}

__device__ __forceinline__ void consumer_sync()      // the 256 consumer threads only
{
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t cluster_index()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_arrive()
{
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}

__device__ __forceinline__ void cluster_wait()
{
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// store a double into the same shared-memory variable of CTA `rank` of the cluster
__device__ __forceinline__ void st_cluster(double *local, uint32_t rank, double v)
{
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(v) : "memory");
}

// C    cluster size (1 = plain CTA, a whole row fits one CTA's slice)
// KMAX double2 column pairs per thread: the CTA slice is at most 512*KMAX columns
// RG   bound on rows per panel = min(8, 16 / KMAX)  (a stage is <= 64 KiB)
template <int C, int KMAX>
__global__ void __launch_bounds__(kAtaxThreads, 1)
atax_cluster_kernel(const AtaxArgs a)
{
    constexpr int RG = (16 / KMAX) < kAtaxMaxRows ? (16 / KMAX) : kAtaxMaxRows;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *tiles = reinterpret_cast<double *>(smem_raw);        // [S][rows][W]
    __shared__ __align__(8) uint64_t full[kAtaxMaxStages];       // TMA landed (tx bytes)
    __shared__ __align__(8) uint64_t empty[kAtaxMaxStages];      // 8 consumer warps released
    __shared__ __align__(8) uint64_t pbar[kAtaxSlots];           // C partials of a panel arrived
    __shared__ double warp_part[2][RG][kWarps];                  // phase-1 warp sums
    __shared__ double part[kAtaxSlots][RG][C];                   // pushed by every CTA of the cluster

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = C > 1 ? cluster_rank() : 0u;
    const long cluster = C > 1 ? (long)cluster_index() : (long)blockIdx.x;
    const long N = a.N;
    const int W = a.W, S = a.stages, L = a.lookahead;
    const int rg = a.rows;                                       // rows per panel, <= RG
    const long c0 = (long)rank * W;
    const int wlen = (int)((N - c0) < W ? (N - c0 > 0 ? N - c0 : 0) : W);   // my columns
    const long row_lo = (a.M * cluster) / a.nclusters;
    const long row_hi = (a.M * (cluster + 1)) / a.nclusters;
    const int ngroups = (int)((row_hi - row_lo + rg - 1) / rg);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        for (int s = 0; s < kAtaxSlots; ++s) mbar_init(&pbar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (C > 1) {          // every CTA's barriers exist before any remote arrive
        cluster_arrive();
        cluster_wait();
    }

    if (warp == kWarps) {
        // ---------------- TMA producer warp ----------------
        if (lane == 0 && wlen > 0) {
            const uint32_t seg = (uint32_t)wlen * 8u;
            for (int g = 0; g < ngroups; ++g) {
                const int s = g % S;
                if (g >= S) mbar_wait(&empty[s], (uint32_t)((g / S - 1) & 1));
                const long r0 = row_lo + (long)g * rg;
                const int nr = (int)((row_hi - r0) < rg ? (row_hi - r0) : rg);
                mbar_expect_tx(&full[s], seg * (uint32_t)nr);
                double *dst = tiles + (size_t)s * rg * W;
                for (int r = 0; r < nr; ++r) {
                    bulk_load(dst + (size_t)r * W, a.A + (r0 + r) * N + c0, seg, &full[s]);
                }
            }
        }
    } else {
        // ---------------- consumer warps ----------------
        // column weights x and the running column sums live in registers
        double2 xr[KMAX], ysum[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int j = 2 * tid + 2 * kThreads * k;
            xr[k] = (j < wlen) ? *reinterpret_cast<const double2 *>(a.x + c0 + j)
                               : make_double2(0.0, 0.0);
            ysum[k] = make_double2(0.0, 0.0);
        }

        // phase 1 of panel g: this CTA's slice of the row dots, pushed to the cluster
        auto phase1 = [&](int g) {
            const int s = g % S, par = g & 1, slot = g % kAtaxSlots;
            if (wlen > 0) mbar_wait(&full[s], (uint32_t)((g / S) & 1));
            const double *tile = tiles + (size_t)s * rg * W;
            const long r0 = row_lo + (long)g * rg;
            const int nr = (int)((row_hi - r0) < rg ? (row_hi - r0) : rg);
            double d[RG];
#pragma unroll
            for (int r = 0; r < RG; ++r) {
                double acc = 0.0;
                if (r < nr) {
#pragma unroll
                    for (int k = 0; k < KMAX; ++k) {
                        const int j = 2 * tid + 2 * kThreads * k;
                        if (j < wlen) {
                            const double2 e =
                                *reinterpret_cast<const double2 *>(tile + (size_t)r * W + j);
                            acc = fma(e.x, xr[k].x, acc);
                            acc = fma(e.y, xr[k].y, acc);
                        }
                    }
                }
                d[r] = acc;
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {     // RG independent shuffle chains
#pragma unroll
                for (int r = 0; r < RG; ++r) d[r] += __shfl_xor_sync(kFullMask, d[r], off);
            }
            if (lane == 0) {
#pragma unroll
                for (int r = 0; r < RG; ++r) warp_part[par][r][warp] = d[r];
            }
            consumer_sync();
            if (tid < C) {
                // thread p serves peer p: the same 8-warp sum in every thread (same bits)
                if (C > 1 && tid == 0) mbar_expect_tx(&pbar[slot], (uint32_t)(C * nr * 8));
                for (int r = 0; r < nr; ++r) {
                    double sum = warp_part[par][r][0];
#pragma unroll
                    for (int w = 1; w < kWarps; ++w) sum += warp_part[par][r][w];
                    if (C > 1) st_async_cluster(&part[slot][r][rank], &pbar[slot], (uint32_t)tid, sum);
                    else part[slot][r][0] = sum;
                }
                if (C == 1) mbar_arrive(&pbar[slot]);
            }
        };

        for (int g = 0; g < L && g < ngroups; ++g) phase1(g);

        for (int g = 0; g < ngroups; ++g) {
            if (g + L < ngroups) phase1(g + L);
            const int s = g % S, slot = g % kAtaxSlots;
            mbar_wait(&pbar[slot], (uint32_t)((g / kAtaxSlots) & 1));
            // t_i: the C partials in rank order -- every CTA computes the same bits
            double t[RG];
#pragma unroll
            for (int r = 0; r < RG; ++r) {
                double sum = part[slot][r][0];
#pragma unroll
                for (int peer = 1; peer < C; ++peer) sum += part[slot][r][peer];
                t[r] = sum;
            }
            // phase 2 on the tile that is still in shared memory
            const double *tile = tiles + (size_t)s * rg * W;
            const long r0 = row_lo + (long)g * rg;
            const int nr = (int)((row_hi - r0) < rg ? (row_hi - r0) : rg);
#pragma unroll
            for (int r = 0; r < RG; ++r) {
                if (r < nr) {
#pragma unroll
                    for (int k = 0; k < KMAX; ++k) {
                        const int j = 2 * tid + 2 * kThreads * k;
                        if (j < wlen) {
                            const double2 e =
                                *reinterpret_cast<const double2 *>(tile + (size_t)r * W + j);
                            ysum[k].x = fma(e.x, t[r], ysum[k].x);
                            ysum[k].y = fma(e.y, t[r], ysum[k].y);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);     // this warp is done with stage s
        }

        double *dst = a.ypart + cluster * N + c0;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int j = 2 * tid + 2 * kThreads * k;
            if (j < wlen) *reinterpret_cast<double2 *>(dst + j) = ysum[k];
        }
    }
    __syncwarp();
    if (C > 1) {          // nobody leaves while a peer may still store into its shared memory
        cluster_arrive();
        cluster_wait();
    }
}

}  // namespace bto
