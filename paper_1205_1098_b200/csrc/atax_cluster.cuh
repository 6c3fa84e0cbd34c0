// atax_cluster.cuh -- single-pass ATAX / BATAX:  y = [beta] A'(A x), A read from HBM ONCE.
//
// The reference contracts t = A x to a per-row scalar by running the two j
// loops of a row back to back, the second touch of the row coming from the
// CPU cache ({_i{_j 1}{_j 2}}, fuse.py:660-688).
// A 32768-double row is 256 KiB -- more than one SM's shared memory -- so here
// a thread-block CLUSTER of C CTAs holds a panel of TR rows between them:
//
//   CTA k of the cluster owns columns [k*W, (k+1)*W) of every row of the panel
//   and keeps them in shared memory, filled by TMA bulk copies
//   (cp.async.bulk, one per row segment, completion on an mbarrier) through an
//   S-stage ring, so up to S-1 panels are in flight while one is consumed;
//   phase 1  every CTA reduces its slice of the row dots (registers -> warp
//            shuffle -> shared memory) and PUSHES its partial sums into the
//            shared memory of every CTA of the cluster with st.async, which
//            counts the bytes on the RECEIVER's mbarrier for that panel;
//            the tile is read from shared memory ONCE, into registers, and the
//            stage is refilled right away;
//   phase 2  one panel later (software pipeline: the exchange latency hides
//            behind the next panel's phase 1, no lock-step cluster barrier)
//            every CTA waits on its own mbarrier, adds the C partials in rank
//            order (t_i, identical bits in all CTAs), then y[j] += A[i,j] * t_i
//            from the tile it still holds in REGISTERS; column sums live in
//            registers for the whole kernel.
// One thread (of warp 1) issues the TMA copies: phase 1 ends with a CTA barrier after every
// warp has its part of the tile in registers, so right after that barrier the
// stage is free and is refilled with the panel S steps ahead (no "empty"
// mbarrier, and no extra warp -- a ninth warp would cap the kernel at 168
// registers per thread, too few for two register tiles).
// One shared-memory read per element instead of two matters because under the
// 1 kW power cap the SM
// clock drops to ~1.75 GHz and the per-panel latency chain is what bounds the
// kernel (profiles/r01/drift_probe.log).
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
    int nclusters;
};

constexpr int kAtaxMaxCluster = 16;      // sizes built: 1 .. 10 and 16 (9: 15 clusters = 135 SMs on a B200
                                         // where 8 gives 15 x 8 = 120; 3, 5, 6, 7: full-width slices for
                                         // mid-size matrices, 10 for rows of 36865 .. 40960 columns; profiles/r02/cluster_probe.log)
constexpr int kAtaxMaxRows = 8;
constexpr int kAtaxMaxStages = 8;
constexpr int kAtaxSlots = 8;                      // exchange slots; phase 1 runs one panel ahead, needs > 3
constexpr int kAtaxThreads = kThreads;             // 8 warps; one thread of warp 1 also issues the TMA copies
constexpr int kIssuer = 32;                        // ... this one (warp 0 pushes the exchange partials)



__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}


// TMA 1-D bulk copy global -> shared, completion counted in bytes on `bar`
// BTO_TMA_POLICY: 0 = no L2 hint, 1 = evict_first, 2 = evict_last, 3 = evict_normal (explicit)
#ifndef BTO_TMA_POLICY
#define BTO_TMA_POLICY 0
#endif
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes,
                                          uint64_t *bar)
{
#if BTO_TMA_POLICY == 0
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
#else
    uint64_t policy;
#if BTO_TMA_POLICY == 1
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
#elif BTO_TMA_POLICY == 2
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy));
#else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
#endif
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
#endif
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

// the same with the remote addresses already mapped (mapa once per kernel, not once per store)
__device__ __forceinline__ void st_async_remote(uint32_t raddr, uint32_t rbar, double v)
{
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
                 ::"r"(raddr), "d"(v), "r"(rbar)
                 : "memory");
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

// fixed pairwise tree over n values: the largest power of two first, the rest added to it
// (n = 9: ((v0+v1)+(v2+v3)) + ((v4+v5)+(v6+v7)), then + v8); ~log2(n) dependent adds
template <int n>
__device__ __forceinline__ double tree_sum(const double *v)
{
    if constexpr (n == 1) {
        return v[0];
    } else if constexpr ((n & (n - 1)) == 0) {
        return tree_sum<n / 2>(v) + tree_sum<n / 2>(v + n / 2);
    } else {
        constexpr int head = n >= 8 ? 8 : (n >= 4 ? 4 : 2);
        return tree_sum<head>(v) + tree_sum<n - head>(v + head);
    }
}

// C    cluster size (1 = plain CTA, a whole row fits one CTA's slice)
// KMAX double2 column pairs per thread: the CTA slice is at most 512*KMAX columns
// TR   rows per panel; a panel is TR*KMAX double2 (<= 16) per thread in registers
// MINB CTAs per SM.  1: two register tiles, phase 2 runs one panel behind phase 1 (the exchange
//      latency hides behind the next panel).  2: ONE tile and no software pipeline -- phase 2
//      follows phase 1 of the same panel and the exchange latency is exposed, but the other CTA
//      on the SM (a different cluster) works meanwhile: two independent latency chains per SM
//      instead of one, at half the registers each.  The per-panel chain (smem reads, reduction,
//      barrier, DSMEM round trip) is what bounds this kernel whenever the SM clock drops under the
//      power cap (7.05 TB/s at 1965 MHz, 6.05 at ~1650, profiles/r02/atax_sustained.md).
// What bounds the kernel (profiles/r02/atax_sustained.md, SM ~1650 MHz under the power cap): the TMA
// stream + CTA barrier alone run at 7.25 TB/s, all the arithmetic without the cluster exchange at
// 7.0, the whole kernel at 6.05-6.15 -- the per-panel chain (shared-memory read, dot, butterfly,
// barrier, st.async round trip, rank-ordered sum) is ~1150 cycles + ~500 per row whatever the panel
// height, so it follows the SM clock.  Four one-row register tiles (three panels of slack) were
// measured at 3.9 TB/s: twice the panels, the same chain per panel.
// Round 2 also measured, and dropped (profiles/r02/atax_sustained.md): loads without predicates for
// the iterations every thread has (-5 %: the predicated schedule interleaves loads and FMAs better),
// warps without tail columns skipping the last iteration behind warp-uniform branches (-10 %), and
// a split CTA barrier where only warp 0 waits (-15 %: the other warps then poll the exchange
// mbarrier while warp 0 is still pushing).  What did help (+4 % alone, +6.7 % in the power-capped
// suite: 6.74 -> 7.19 TB/s): issuing the refill copies from warp 1 -- the stall samples sit on
// the waits for the PEERS' partials (14 % vs 2 % on the waits for the copies), and warp 0's pushes
// used to queue behind thread 0's refill code.  One lane per (row, peer) instead of one per peer
// with a loop over the rows: no further change.
template <int C, int KMAX, int TR, int MINB = 1>
__global__ void __launch_bounds__(kAtaxThreads, MINB)
atax_cluster_kernel(const AtaxArgs a)
{
    static_assert(TR * KMAX <= 16 && TR <= kAtaxMaxRows, "register tile too large");
    static_assert(kWarps == 8, "the warp-sum tree below is written for 8 warps");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *tiles = reinterpret_cast<double *>(smem_raw);        // [S][TR][W]
    __shared__ __align__(8) uint64_t full[kAtaxMaxStages];       // TMA landed (tx bytes)
    __shared__ __align__(8) uint64_t pbar[kAtaxSlots];           // C partials of a panel arrived
    constexpr int CP = (C + 1) & ~1;     // a row's partials padded to whole 16-byte words (LDS.128; +0.9 %)
    __shared__ __align__(16) double warp_part[2][TR][kWarps];    // phase-1 warp sums
    __shared__ __align__(16) double part[kAtaxSlots][TR][CP];    // pushed by every CTA of the cluster

    wait_for_producer_grid();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = C > 1 ? cluster_rank() : 0u;
    const long cluster = C > 1 ? (long)cluster_index() : (long)blockIdx.x;
    const long N = a.N;
    const int W = a.W, S = a.stages;
    const long c0 = (long)rank * W;
    const int wlen = (int)((N - c0) < W ? (N - c0 > 0 ? N - c0 : 0) : W);   // my columns
    const long row_lo = (a.M * cluster) / a.nclusters;
    const long row_hi = (a.M * (cluster + 1)) / a.nclusters;
    const int ngroups = (int)((row_hi - row_lo + TR - 1) / TR);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
        }
        for (int s = 0; s < kAtaxSlots; ++s) mbar_init(&pbar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (C > 1) {          // every CTA's barriers exist before any remote store
        cluster_arrive();
        cluster_wait();
    }

    // the issuer thread: fill stage g % S with panel g
    auto issue = [&](int g) {
        if (wlen <= 0) return;
        const int s = g % S;
        const uint32_t seg = (uint32_t)wlen * 8u;
        const long r0 = row_lo + (long)g * TR;
        const int nr = (int)((row_hi - r0) < TR ? (row_hi - r0) : TR);
        mbar_expect_tx(&full[s], seg * (uint32_t)nr);
        double *dst = tiles + (size_t)s * TR * W;
        for (int r = 0; r < nr; ++r) {
            bulk_load(dst + (size_t)r * W, a.A + (r0 + r) * N + c0, seg, &full[s]);
        }
    };
    if (tid == kIssuer) {
        for (int g = 0; g < S && g < ngroups; ++g) issue(g);
    }
    // where thread p < C pushes: this CTA's column of CTA p's `part`, and CTA p's exchange barriers
    uint32_t peer_part = 0, peer_bar = 0;
    if (C > 1 && tid < C) {
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(peer_part) : "r"(smem_u32(&part[0][0][rank])), "r"((uint32_t)tid));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(peer_bar) : "r"(smem_u32(&pbar[0])), "r"((uint32_t)tid));
    }

    {
        // column weights x and the running column sums live in registers
        double2 xr[KMAX], ysum[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int j = 2 * tid + 2 * kThreads * k;
            xr[k] = (j < wlen) ? *reinterpret_cast<const double2 *>(a.x + c0 + j)
                               : make_double2(0.0, 0.0);
            ysum[k] = make_double2(0.0, 0.0);
        }

        // phase 1 of panel g: shared memory -> registers (once), this CTA's slice
        // of the row dots, pushed to the cluster
        auto phase1 = [&](int g, double2 (&tile)[TR][KMAX]) {
            const int s = g % S, par = g & 1, slot = g % kAtaxSlots;
            if (wlen > 0) mbar_wait(&full[s], (uint32_t)((g / S) & 1));
            const double *src = tiles + (size_t)s * TR * W;
            const long r0 = row_lo + (long)g * TR;
            const int nr = (int)((row_hi - r0) < TR ? (row_hi - r0) : TR);
#pragma unroll
            for (int r = 0; r < TR; ++r) {
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    const int j = 2 * tid + 2 * kThreads * k;
                    tile[r][k] = (r < nr && j < wlen)
                                     ? *reinterpret_cast<const double2 *>(src + (size_t)r * W + j)
                                     : make_double2(0.0, 0.0);
                }
            }
            double d[TR];
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                // independent accumulators: with two warps per scheduler a single
                // 2*KMAX-long FMA chain would expose the fp64 latency
                double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
#pragma unroll
                for (int k = 0; k < KMAX; k += 2) {
                    acc0 = fma(tile[r][k].x, xr[k].x, acc0);
                    acc1 = fma(tile[r][k].y, xr[k].y, acc1);
                    if (k + 1 < KMAX) {
                        acc2 = fma(tile[r][k + 1].x, xr[k + 1].x, acc2);
                        acc3 = fma(tile[r][k + 1].y, xr[k + 1].y, acc3);
                    }
                }
                d[r] = (acc0 + acc1) + (acc2 + acc3);
            }
            // halving butterfly: a lane hands the rows it does not keep to its partner, so TR rows
            // cost TR - 1 + (5 - log2 TR) shuffled doubles instead of 5 TR (2 rows: 5, not 10);
            // afterwards lane l holds the warp's sum of row l / (32 / TR) in d[0]
            warp_transpose_sum<TR>(d, lane);
            if ((lane % (32 / TR)) == 0) warp_part[par][lane / (32 / TR)][warp] = d[0];
            __syncthreads();
            // every warp holds its part of the tile in registers (the FMAs above
            // consumed the loads): the stage is free, refill it S panels ahead.  The copies are
            // issued from warp 1 so that warp 0's pushes -- which every CTA of the cluster is
            // waiting for -- do not queue behind the address arithmetic of the refill.
            if (tid == kIssuer && g + S < ngroups) issue(g + S);
            if (tid < C) {
                // thread p serves peer p: the same 8-warp sum in every thread (same bits).
                // ALL TR rows are pushed, also those past the end of the row range (their tiles are
                // zeros, so their sums are exact zeros): phase 2 multiplies every row's t with its
                // tile, and 0 x t is only 0 if t is a number -- an entry of `part` that nobody wrote
                // in this launch is whatever the previous kernel left in shared memory, NaN bit
                // patterns included (round-2 fuzz: one BATAX result in 37 000 with 960 NaN columns,
                // the slice of one CTA; scripts/batax_rare_probe.py).
                if (C > 1 && tid == 0) mbar_expect_tx(&pbar[slot], (uint32_t)(C * TR * 8));
#pragma unroll
                for (int r = 0; r < TR; ++r) {
                    const double *wp = warp_part[par][r];      // fixed pairwise tree
                    const double sum = ((wp[0] + wp[1]) + (wp[2] + wp[3])) +
                                       ((wp[4] + wp[5]) + (wp[6] + wp[7]));
                    if (C > 1) {
                        st_async_remote(peer_part + (uint32_t)((slot * TR + r) * CP * 8),
                                        peer_bar + (uint32_t)(slot * 8), sum);
                    } else {
                        part[slot][r][0] = sum;
                    }
                }
                if (C == 1) mbar_arrive(&pbar[slot]);
            }
        };

        // phase 2 of panel g from the register tile
        auto phase2 = [&](int g, const double2 (&tile)[TR][KMAX]) {
            const int slot = g % kAtaxSlots;
            mbar_wait(&pbar[slot], (uint32_t)((g / kAtaxSlots) & 1));
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                // t_i: the C partials in rank order -- every CTA computes the same bits
                // (rows past the end of the range hold zeros in the tile)
                double t = tree_sum<C>(part[slot][r]);
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    ysum[k].x = fma(tile[r][k].x, t, ysum[k].x);
                    ysum[k].y = fma(tile[r][k].y, t, ysum[k].y);
                }
            }
        };

        if constexpr (MINB == 1) {
            // two register tiles, loop unrolled by two so neither is ever copied
            double2 tile_a[TR][KMAX], tile_b[TR][KMAX];
            if (ngroups > 0) phase1(0, tile_a);
            for (int g = 0; g < ngroups; g += 2) {
                if (g + 1 < ngroups) phase1(g + 1, tile_b);
                phase2(g, tile_a);
                if (g + 1 >= ngroups) break;
                if (g + 2 < ngroups) phase1(g + 2, tile_a);
                phase2(g + 1, tile_b);
            }
        } else {
            double2 tile[TR][KMAX];
            for (int g = 0; g < ngroups; ++g) {
                phase1(g, tile);
                phase2(g, tile);
            }
        }

        double *dst = a.ypart + cluster * N + c0;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int j = 2 * tid + 2 * kThreads * k;
            if (j < wlen) st_partial2(dst + j, ysum[k]);
        }
    }
    __syncwarp();
    if (C > 1) {          // nobody leaves while a peer may still store into its shared memory
        cluster_arrive();
        cluster_wait();
    }
}

}  // namespace bto
