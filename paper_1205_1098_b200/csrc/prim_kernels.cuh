// prim_kernels.cuh -- unfused building blocks for kernel specs that have no
// hand-written fused sequence (the generic executor, runtime.GenericKernel).
//
// The fused sequences are the product; these exist so that ANY valid `.bto`
// spec runs on the device (statement by statement, temporaries in HBM -- what
// the reference's unfused organism `initial_forest` does on the CPU).  The two
// matrix-vector products reuse the tile engine (mv_kernels.cuh); everything
// else is a grid-stride elementwise kernel or a fixed-order reduction.
#pragma once
#include "common.cuh"

namespace bto {

// out = alpha*x (+|-) beta*y, each product and the sum rounded on their own
// (cemit.py:112-136).  mode: 0 scale (y unused), 1 x*alpha + y*beta,
// 2 x + y, 3 x - y.
__global__ void __launch_bounds__(kThreads)
prim_axpby_kernel(double alpha, const double *x, double beta, const double *y, double *out,
                  long n, int mode)
{
    const long stride = (long)gridDim.x * kThreads;
    for (long i = (long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
        double r;
        if (mode == 0) r = __dmul_rn(x[i], alpha);
        else if (mode == 1) r = __dadd_rn(__dmul_rn(x[i], alpha), __dmul_rn(y[i], beta));
        else if (mode == 2) r = __dadd_rn(x[i], y[i]);
        else r = __dsub_rn(x[i], y[i]);
        out[i] = r;
    }
}

// out[i,j] = u[i] * v[j]   (row-major M x N)
__global__ void __launch_bounds__(kThreads)
prim_outer_kernel(const double *u, const double *v, double *out, long M, long N)
{
    const long total = M * N, stride = (long)gridDim.x * kThreads;
    for (long e = (long)blockIdx.x * kThreads + threadIdx.x; e < total; e += stride) {
        out[e] = __dmul_rn(u[e / N], v[e % N]);
    }
}

// partials[b] = sum over the CTA's grid-stride share of x[i]*y[i]; the last CTA
// adds the partials in order (same scheme as AXPYDOT's dot).
__global__ void __launch_bounds__(kThreads)
prim_dot_kernel(const double *x, const double *y, double *out, double *partials,
                unsigned int *ticket, long n)
{
    __shared__ double scratch[kWarps];
    __shared__ bool is_last;
    const long stride = (long)gridDim.x * kThreads;
    double acc = 0.0;
    for (long i = (long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
        acc = fma(x[i], y[i], acc);
    }
    const double cta_sum = block_sum(acc, scratch);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = cta_sum;
        __threadfence();
        is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        double s = 0.0;
        for (unsigned int p = threadIdx.x; p < gridDim.x; p += kThreads) s += ld_cg(partials + p);
        const double total = block_sum(s, scratch);
        if (threadIdx.x == 0) {
            *out = total;
            *ticket = 0u;
        }
    }
}

}  // namespace bto
