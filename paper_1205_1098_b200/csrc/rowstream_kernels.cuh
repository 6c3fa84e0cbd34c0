// rowstream_kernels.cuh -- N-products of wide matrices by streaming whole rows.
//
// mv_tile_kernel cuts a matrix into 512-column strips, which the T-product needs (a thread
// keeps its columns' sums in registers).  A pass with row dots only does not: a CTA can take a
// block of rows and stream each row end to end -- four rows at a time, every thread striding
// across the full row -- so DRAM sees a handful of long sequential streams per CTA instead of
// 4 KiB row segments.  The organism-driven emitter prints exactly this shape for GESUMMV and
// measured 7.3 TB/s at n = 24576 against 6.9-7.07 for the strip-tiled pass, which is why it
// exists here (profiles/r01/probes/emitted_rowstream_probe.py).  Row dots are reduced warp -> CTA in a fixed
// order once per four rows; the row epilogue is applied in the kernel: ONE launch, no partials.
#pragma once
#include "mv_kernels.cuh"

namespace bto {

constexpr int kRsThreads = 512;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsRows = 4;          // rows per batch
constexpr int kRsPairs = 2;         // double2 per thread, row and matrix in flight

struct RowStreamArgs {
    const double *A, *A2;     // A2: second matrix (TWO)
    const double *colw;       // [N]
    FinArgs fin;              // row epilogue (rmode, ralpha, rbeta, rowy, rowout)
    long M, N;
    long rows_per_cta;        // multiple of kRsRows
};

template <bool TWO>
__global__ void __launch_bounds__(kRsThreads, 1)
rowstream_kernel(const RowStreamArgs a)
{
    constexpr int R = kRsRows, U = kRsPairs, S = TWO ? 2 : 1;
    __shared__ double red[2][kRsWarps][R * S];

    wait_for_producer_grid();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long N = a.N;
    const long m0 = (long)blockIdx.x * a.rows_per_cta;
    const long m1 = m0 + a.rows_per_cta < a.M ? m0 + a.rows_per_cta : a.M;
    int buf = 0;

    for (long rb = m0; rb < m1; rb += R) {
        double acc[R * S];
#pragma unroll
        for (int k = 0; k < R * S; ++k) acc[k] = 0.0;
        // rows beyond m1 are read as row m1-1 and dropped (keeps the loads unconditional)
        long row[R];
#pragma unroll
        for (int i = 0; i < R; ++i) row[i] = rb + i < m1 ? rb + i : m1 - 1;

        long j = 2L * tid;
        for (; j + 2L * (U - 1) * kRsThreads + 1 < N; j += 2L * U * kRsThreads) {
            double2 x[U], e[R][U], f[TWO ? R : 1][U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long jj = j + 2L * u * kRsThreads;
                x[u] = make_double2(__ldg(a.colw + jj), __ldg(a.colw + jj + 1));   // (x may sit at any 8-byte offset)
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    e[i][u] = ld_stream2<true>(a.A + row[i] * N + jj);
                    if constexpr (TWO) f[i][u] = ld_stream2<true>(a.A2 + row[i] * N + jj);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    acc[i] = fma(e[i][u].x, x[u].x, acc[i]);
                    acc[i] = fma(e[i][u].y, x[u].y, acc[i]);
                    if constexpr (TWO) {
                        acc[R + i] = fma(f[i][u].x, x[u].x, acc[R + i]);
                        acc[R + i] = fma(f[i][u].y, x[u].y, acc[R + i]);
                    }
                }
            }
        }
        for (; j + 1 < N; j += 2L * kRsThreads) {           // what is left of the row (pairs)
            const double2 x = make_double2(__ldg(a.colw + j), __ldg(a.colw + j + 1));
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const double2 e = ld_stream2<true>(a.A + row[i] * N + j);
                acc[i] = fma(e.x, x.x, acc[i]);
                acc[i] = fma(e.y, x.y, acc[i]);
                if constexpr (TWO) {
                    const double2 f = ld_stream2<true>(a.A2 + row[i] * N + j);
                    acc[R + i] = fma(f.x, x.x, acc[R + i]);
                    acc[R + i] = fma(f.y, x.y, acc[R + i]);
                }
            }
        }
        // lanes -> warp (butterfly), warps -> CTA through shared memory, ascending warp order
#pragma unroll
        for (int k = 0; k < R * S; ++k) acc[k] = warp_sum(acc[k]);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < R * S; ++k) red[buf][warp][k] = acc[k];
        }
        __syncthreads();
        if (tid < R && rb + tid < m1) {
            double s = red[buf][0][tid], s2 = TWO ? red[buf][0][R + tid] : 0.0;
            for (int w = 1; w < kRsWarps; ++w) {
                s += red[buf][w][tid];
                if constexpr (TWO) s2 += red[buf][w][R + tid];
            }
            row_epilogue(a.fin, rb + tid, s, s2);
        }
        buf ^= 1;        // double-buffered: the next batch's barrier orders these reads
    }
}

}  // namespace bto
