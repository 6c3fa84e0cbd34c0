// common.cuh -- device helpers shared by the fused BLAS-1/BLAS-2 kernels (sm_100a).
//
// Everything here is HBM-bound fp64 streaming work: 128-bit coalesced loads
// that bypass L1 (each matrix element is used once), warp-shuffle reductions
// with a FIXED combination order (the reference guarantees bit-stable results
// at a fixed thread count, cemit.py:8-10; we guarantee it at a fixed launch
// geometry), and rounded-separately arithmetic where the reference's C rounds
// separately (cemit.py:112-136 prints one binary op per statement and gcc on
// baseline x86-64 does not contract them into FMAs).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bto {

constexpr int kThreads = 256;            // every kernel here uses 256-thread CTAs
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFullMask = 0xffffffffu;

// ---- streaming global loads / stores ---------------------------------------
// Read-once operands come through the non-coherent path.  BYPASS_L1 adds
// L1::no_allocate, which keeps them from evicting the small vectors (weights, x)
// that are re-used from L1 -- but measured on B200 it makes a streaming kernel
// bistable: AXPYDOT runs at 7.0 TB/s until any other large kernel has run, then at
// 6.3 TB/s for good (profiles/r01/axpydot_state_probe.log); with plain .nc loads it
// stays at 7.0, BiCGK and GEMVER gain 1-2 %, only the two-matrix GESUMMV pass is
// faster (3 %) with the bypass.  So the bypass is a per-kernel choice.
template <bool BYPASS_L1 = false>
__device__ __forceinline__ double2 ld_stream2(const double *p)   // 16 B aligned
{
    double2 v;
    if constexpr (BYPASS_L1) {
        asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    } else {
        asm("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    }
    return v;
}

template <bool BYPASS_L1 = false>
__device__ __forceinline__ double ld_stream1(const double *p)
{
    double v;
    if constexpr (BYPASS_L1) {
        asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    } else {
        asm("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    }
    return v;
}

// stores for write-once outputs (z, B); BTO_STORE_POLICY picks the cache
// operator: 0 = .cs (evict-first), 1 = default write-back, 2 = .wt, 3 = .cg
#ifndef BTO_STORE_POLICY
#define BTO_STORE_POLICY 0
#endif
__device__ __forceinline__ void st_stream2(double *p, double2 v)   // 16 B aligned
{
#if BTO_STORE_POLICY == 0
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};"
#elif BTO_STORE_POLICY == 1
    asm volatile("st.global.v2.f64 [%0], {%1, %2};"
#elif BTO_STORE_POLICY == 2
    asm volatile("st.global.wt.v2.f64 [%0], {%1, %2};"
#else
    asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};"
#endif
                 :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// Stores of partial results (workspace rows the join kernel reads next) and of the small
// result vectors.  BTO_PARTIAL_POLICY: 0 = default write-back, 1 = .wt (write-through: the
// line stays in L2 for the join but is clean), 2 = .cs
#ifndef BTO_PARTIAL_POLICY
#define BTO_PARTIAL_POLICY 0
#endif
__device__ __forceinline__ void st_partial1(double *p, double v)
{
#if BTO_PARTIAL_POLICY == 1
    asm volatile("st.global.wt.f64 [%0], %1;" :: "l"(p), "d"(v) : "memory");
#elif BTO_PARTIAL_POLICY == 2
    asm volatile("st.global.cs.f64 [%0], %1;" :: "l"(p), "d"(v) : "memory");
#else
    *p = v;
#endif
}
__device__ __forceinline__ void st_partial2(double *p, double2 v)   // 16 B aligned
{
#if BTO_PARTIAL_POLICY == 1
    asm volatile("st.global.wt.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
#elif BTO_PARTIAL_POLICY == 2
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
#else
    *reinterpret_cast<double2 *>(p) = v;
#endif
}

__device__ __forceinline__ void st_stream1(double *p, double v)
{
    asm volatile("st.global.cs.f64 [%0], %1;" :: "l"(p), "d"(v) : "memory");
}

// loads that must observe data written earlier in the same grid by other CTAs
__device__ __forceinline__ double ld_cg(const double *p)
{
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// Programmatic dependent launch: every kernel of the library is launched while
// its predecessor in the stream is still running and waits here, before it
// touches memory, until that grid has completed and flushed; the launch latency
// hides under the predecessor's tail.  A no-op for a normally launched kernel.
// (An explicit griddepcontrol.launch_dependents right after the wait was measured:
// no gain at any size, profiles/r01/midsize_probe.md -- the implicit trigger at
// grid completion already hides the launch.)
__device__ __forceinline__ void wait_for_producer_grid()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---- reductions with a fixed order ------------------------------------------
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        v += __shfl_xor_sync(kFullMask, v, off);
    }
    return v;
}

// Sum over the CTA; result valid in thread 0.  scratch: kWarps doubles.
__device__ __forceinline__ double block_sum(double v, double *scratch)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double total = 0.0;
    if (warp == 0) {
        double part = lane < kWarps ? scratch[lane] : 0.0;
#pragma unroll
        for (int off = kWarps / 2; off >= 1; off >>= 1) {
            part += __shfl_xor_sync(kFullMask, part, off);
        }
        total = part;
    }
    __syncthreads();
    return total;
}

// Transposing warp reduction: every lane holds R per-row partial sums v[0..R);
// afterwards v[0] of lane l is the warp-wide sum of row (l / (32/R)).
// 31 shuffles for R = 32 instead of 32*5: the halving butterfly sends the half
// of the rows a lane does not keep to its partner.
template <int R>
__device__ __forceinline__ void warp_transpose_sum(double (&v)[R], int lane)
{
    static_assert(R == 1 || R == 2 || R == 4 || R == 8 || R == 16 || R == 32, "R must be a power of two <= 32");
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int off = 16 >> s;
        const int alive = R >> s;
        if (alive > 1) {
            const bool upper = (lane & off) != 0;
            const int half = alive >> 1;
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const double give = upper ? v[k] : v[k + half];
                const double keep = upper ? v[k + half] : v[k];
                v[k] = keep + __shfl_xor_sync(kFullMask, give, off);
            }
        } else {
            v[0] += __shfl_xor_sync(kFullMask, v[0], off);
        }
    }
}

// ---- shared-memory mbarriers (TMA completion, producer / consumer hand-offs inside a CTA) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
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

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---- static work split shared by kernels and their finalisers ---------------
// U units are dealt to G CTAs as contiguous ranges [U*k/G, U*(k+1)/G), the
// reference's own block formula (cemit.py:195-196) one level down.
__host__ __device__ __forceinline__ long split_begin(long U, long G, long k)
{
    return (U * k) / G;
}

// the CTA whose range contains unit u (the largest k with split_begin(k) <= u)
__host__ __device__ __forceinline__ long split_owner(long U, long G, long u)
{
    return ((u + 1) * G - 1) / U;
}

}  // namespace bto
