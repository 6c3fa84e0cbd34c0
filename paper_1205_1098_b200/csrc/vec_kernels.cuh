// vec_kernels.cuh -- fused BLAS-1 sequences: AXPYDOT, VADD, WAXPBY.
//
// One pass, every vector element crosses HBM once (AXPYDOT: 3 reads + 1 write
// = 32 B per element).  The contracted temporary
// (t0 = alpha*v, fuse.py:660-688) lives in a register; the dot product is
// reduced warp -> CTA -> grid with a fixed order, the grid stage done by the
// last CTA to finish (ticket counter), so there is no second launch.
#pragma once
#include "common.cuh"

namespace bto {

enum VecOp : int { kVadd = 0, kWaxpby = 1, kAxpydot = 2 };

struct VecArgs {
    const double *a;      // axpydot: w   vadd: w   waxpby: x
    const double *b;      // axpydot: v   vadd: y   waxpby: y
    const double *c;      // axpydot: u   vadd: z   waxpby: unused
    double alpha, beta;
    double *out;          // axpydot: z   vadd: x   waxpby: w
    double *dot;          // axpydot: the scalar output `beta` (device)
    double *partials;     // [gridDim.x] per-CTA dot partials
    unsigned int *ticket; // zero on entry, reset to zero by the last CTA
    long n;
};

// Element function: the reference's statement order, each op rounded on its
// own (no FMA contraction) so `z`, `x`, `w` are bit-identical to the C path.
template <int OP>
__device__ __forceinline__ double vec_elem(const VecArgs &g, double a, double b,
                                           double c, double &acc)
{
    if (OP == kVadd) {                     // t0 = w + y ; x = t0 + z
        return __dadd_rn(__dadd_rn(a, b), c);
    } else if (OP == kWaxpby) {            // t0 = x*alpha ; t1 = y*beta ; w = t0 + t1
        return __dadd_rn(__dmul_rn(a, g.alpha), __dmul_rn(b, g.beta));
    } else {                               // t0 = v*alpha ; z = w - t0 ; beta += z*u
        const double z = __dsub_rn(a, __dmul_rn(b, g.alpha));
        acc = fma(z, c, acc);
        return z;
    }
}

template <int OP, int UNROLL, bool ALIGNED>
__global__ void __launch_bounds__(kThreads)
vec_kernel(const VecArgs g)
{
    constexpr bool kHasC = OP != kWaxpby;
    constexpr bool kDot = OP == kAxpydot;
    wait_for_producer_grid();
    const long tid = (long)blockIdx.x * kThreads + threadIdx.x;
    const long nthreads = (long)gridDim.x * kThreads;
    double acc = 0.0;

    if (ALIGNED) {
        // all four base pointers are 16 B aligned: stream double2
        const long pairs = g.n >> 1;
        long i = tid;
        for (; i + (UNROLL - 1) * nthreads < pairs; i += UNROLL * nthreads) {
            double2 a[UNROLL], b[UNROLL], c[UNROLL];
#pragma unroll
            for (int k = 0; k < UNROLL; ++k) {
                const long e = 2 * (i + k * nthreads);
                a[k] = ld_stream2(g.a + e);
                b[k] = ld_stream2(g.b + e);
                c[k] = kHasC ? ld_stream2(g.c + e) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int k = 0; k < UNROLL; ++k) {
                const long e = 2 * (i + k * nthreads);
                double2 r;
                r.x = vec_elem<OP>(g, a[k].x, b[k].x, c[k].x, acc);
                r.y = vec_elem<OP>(g, a[k].y, b[k].y, c[k].y, acc);
                st_stream2(g.out + e, r);
            }
        }
        for (; i < pairs; i += nthreads) {
            const long e = 2 * i;
            const double2 a = ld_stream2(g.a + e), b = ld_stream2(g.b + e);
            const double2 c = kHasC ? ld_stream2(g.c + e) : make_double2(0.0, 0.0);
            double2 r;
            r.x = vec_elem<OP>(g, a.x, b.x, c.x, acc);
            r.y = vec_elem<OP>(g, a.y, b.y, c.y, acc);
            st_stream2(g.out + e, r);
        }
        if ((g.n & 1) && tid == 0) {          // odd tail element
            const long e = g.n - 1;
            g.out[e] = vec_elem<OP>(g, g.a[e], g.b[e], kHasC ? g.c[e] : 0.0, acc);
        }
    } else {
        for (long e = tid; e < g.n; e += nthreads) {
            const double a = ld_stream1(g.a + e), b = ld_stream1(g.b + e);
            const double c = kHasC ? ld_stream1(g.c + e) : 0.0;
            st_stream1(g.out + e, vec_elem<OP>(g, a, b, c, acc));
        }
    }

    if (kDot) {
        __shared__ double scratch[kWarps];
        __shared__ bool is_last;
        const double cta_sum = block_sum(acc, scratch);
        if (threadIdx.x == 0) {
            g.partials[blockIdx.x] = cta_sum;
            __threadfence();
            const unsigned int t = atomicAdd(g.ticket, 1u);
            is_last = (t == gridDim.x - 1);
        }
        __syncthreads();
        if (is_last) {
            // grid stage: fixed order (thread t takes partials t, t+256, ...)
            __threadfence();
            double s = 0.0;
            for (unsigned int p = threadIdx.x; p < gridDim.x; p += kThreads) {
                s += ld_cg(g.partials + p);
            }
            const double total = block_sum(s, scratch);
            if (threadIdx.x == 0) {
                *g.dot = total;
                *g.ticket = 0u;
            }
        }
    }
}

}  // namespace bto
