// skinny_kernels.cuh -- the matrix passes for narrow matrices (N <= 256).
//
// mv_tile_kernel gives every thread two columns of a 512-column strip; a matrix with
// N = 32 columns would use 16 of the 256 threads (measured 0.47 TB/s).  Here a row is
// shared by L <= 32 lanes of one warp (each holding V column slots) and the CTA's 256/L row
// groups walk down interleaved rows, so a warp still reads contiguous memory:
//   * a row's dot product is complete inside its warp segment (xor butterfly): the row
//     result and its epilogue are written here, no row partials, no row side in the join;
//   * a thread keeps its column pair for the whole kernel, so the weighted column sums
//     live in two registers; the row groups are folded in shared memory at the end and
//     the CTA writes ONE partial row, joined by finalize_kernel in ascending CTA order;
//   * kFlagAtax weights the column sums with the row's own dot: single-pass ATAX.
// Same per-element arithmetic as mv_unit (rank-2 update with separately rounded
// operations, fma accumulation), fixed reduction order, bit-reproducible.
#pragma once
#include "mv_kernels.cuh"

namespace bto {

enum : int { kFlagAtax = 16 };
constexpr long kSkinnyMaxN = 512;
// Rows per thread and unit for V column slots: 8 loads per matrix in flight, 16 for V = 2, 4
// (measured: GEMVER 1M x 256 4.8 -> 5.8 TB/s, 2M x 100 4.3 -> 4.8; with V = 1 the wider unit
// spills, with V = 8 it is slower)
__host__ __device__ constexpr int skinny_rows(int V) { return ((V == 2 || V == 4) ? 16 : 8) / V; }

struct SkinnyArgs {
    MvArgs mv;                // operands; colpart is [grid][N]
    FinArgs fin;              // row epilogue (rmode, ralpha, rbeta, rowy, rowout)
    int L;                    // threads per row (power of two, <= 32: a row never leaves its warp)
    long rows_per_cta;        // multiple of skinny_rows(V) * (kThreads / L)
};

// V slots per thread and row: slot v of thread cp holds column(s) (cp + L*v) * W, W = 2 (PAIR:
// double2 loads, N even and 16-byte aligned operands) or 1.  V = 1 covers N <= 32*W, larger V
// (then L = 32) up to N = 512; rows per thread and step shrink with V (skinny_rows) so that a
// thread has 8 or 16 loads per matrix in flight.
// (eight slots of a rank-2 pass spill ~100 bytes at 128 registers; one CTA per SM instead was
// measured slower, 4.4 vs 4.8 TB/s at N = 500)
template <int FLAGS, bool PAIR, int V>
__global__ void __launch_bounds__(kThreads, 2)
mv_skinny_kernel(const SkinnyArgs s)
{
    constexpr bool kN = (FLAGS & kFlagN) != 0;
    constexpr bool kN2 = (FLAGS & kFlagN2) != 0;
    constexpr bool kT = (FLAGS & kFlagT) != 0;
    constexpr bool kRank2 = (FLAGS & kFlagRank2) != 0;
    constexpr bool kAtax = (FLAGS & kFlagAtax) != 0;
    static_assert(!kN2 || kN, "the second N-product rides on the first");
    static_assert(!kAtax || (kN && kT), "ATAX weights the column sums with the row dots");
    static_assert(V == 1 || V == 2 || V == 4 || V == 8, "slots per thread");
    constexpr int R = skinny_rows(V);
    constexpr int W = PAIR ? 2 : 1;
    // loads bypass L1 here (measured: 4M x 32 BiCGK 4.8 TB/s with the bypass, 4.4 without)

    __shared__ double fold[V][kThreads][2];

    wait_for_producer_grid();
    const MvArgs &a = s.mv;
    const int tid = threadIdx.x;
    const int L = s.L, G = kThreads / L;
    const int cp = tid & (L - 1), g = tid / L;
    const long M = a.M, N = a.N;
    const long m0 = (long)blockIdx.x * s.rows_per_cta;
    const long m1 = m0 + s.rows_per_cta < M ? m0 + s.rows_per_cta : M;

    long col[V];
    bool ok0[V], ok1[V];
    double2 cw[V], b1[V], b2[V], cs[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        col[v] = (long)(cp + L * v) * W;
        ok0[v] = col[v] < N;
        ok1[v] = PAIR && col[v] + 1 < N;
        cs[v] = make_double2(0.0, 0.0);
        cw[v] = b1[v] = b2[v] = make_double2(0.0, 0.0);
        if constexpr (kN) {
            cw[v].x = ok0[v] ? __ldg(a.colw + col[v]) : 0.0;
            cw[v].y = ok1[v] ? __ldg(a.colw + col[v] + 1) : 0.0;
        }
        if constexpr (kRank2) {
            b1[v].x = ok0[v] ? __ldg(a.v1 + col[v]) : 0.0;
            b1[v].y = ok1[v] ? __ldg(a.v1 + col[v] + 1) : 0.0;
            b2[v].x = ok0[v] ? __ldg(a.v2 + col[v]) : 0.0;
            b2[v].y = ok1[v] ? __ldg(a.v2 + col[v] + 1) : 0.0;
        }
    }

    for (long rb = m0; rb < m1; rb += (long)R * G) {
        double2 e[R][V], e2[kN2 ? R : 1][V];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const long row = rb + (long)i * G + g;
            const bool rv = row < m1;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const bool ld = rv && ok0[v];
                const double *p = a.A + row * N + col[v];
                if constexpr (PAIR) {
                    e[i][v] = ld ? ld_stream2<true>(p) : make_double2(0.0, 0.0);
                    if constexpr (kN2) {
                        e2[i][v] = ld ? ld_stream2<true>(a.A2 + row * N + col[v]) : make_double2(0.0, 0.0);
                    }
                } else {
                    e[i][v] = make_double2(ld ? ld_stream1<true>(p) : 0.0, 0.0);
                    if constexpr (kN2) {
                        e2[i][v] = make_double2(ld ? ld_stream1<true>(a.A2 + row * N + col[v]) : 0.0, 0.0);
                    }
                }
            }
        }
        double rw[(kT && !kAtax) ? R : 1], ru1[kRank2 ? R : 1], ru2[kRank2 ? R : 1];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const long row = rb + (long)i * G + g;
            const bool rv = row < m1;
            if constexpr (kT && !kAtax) rw[i] = rv ? __ldg(a.roww + row) : 0.0;
            if constexpr (kRank2) {
                ru1[i] = rv ? __ldg(a.u1 + row) : 0.0;
                ru2[i] = rv ? __ldg(a.u2 + row) : 0.0;
            }
        }
        double dot[kN ? R : 1], dot2[kN2 ? R : 1];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const long row = rb + (long)i * G + g;
            const bool rv = row < m1;
            double d = 0.0, d2 = 0.0;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if constexpr (kRank2) {
                    // t0 = u1*v1 ; t1 = A + t0 ; t2 = u2*v2 ; B = t1 + t2
                    e[i][v].x = __dadd_rn(__dadd_rn(e[i][v].x, __dmul_rn(ru1[i], b1[v].x)),
                                          __dmul_rn(ru2[i], b2[v].x));
                    e[i][v].y = __dadd_rn(__dadd_rn(e[i][v].y, __dmul_rn(ru1[i], b1[v].y)),
                                          __dmul_rn(ru2[i], b2[v].y));
                    double *dst = a.Bout + row * N + col[v];
                    if constexpr (PAIR) {
                        if (rv && ok0[v]) st_stream2(dst, e[i][v]);
                    } else {
                        if (rv && ok0[v]) st_stream1(dst, e[i][v].x);
                    }
                }
                if constexpr (kN) {
                    d = fma(e[i][v].x, cw[v].x, d);
                    d = fma(e[i][v].y, cw[v].y, d);
                    if constexpr (kN2) {
                        d2 = fma(e2[i][v].x, cw[v].x, d2);
                        d2 = fma(e2[i][v].y, cw[v].y, d2);
                    }
                }
            }
            if constexpr (kN) dot[i] = d;
            if constexpr (kN2) dot2[i] = d2;
        }
        if constexpr (kN) {
            // the L lanes of a row -> every one of them holds the row's dot product
            for (int off = L >> 1; off >= 1; off >>= 1) {
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    dot[i] += __shfl_xor_sync(kFullMask, dot[i], off);
                    if constexpr (kN2) dot2[i] += __shfl_xor_sync(kFullMask, dot2[i], off);
                }
            }
            if (cp == 0 && s.fin.rmode != kRowNone) {
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    const long row = rb + (long)i * G + g;
                    if (row < m1) row_epilogue(s.fin, row, dot[i], kN2 ? dot2[kN2 ? i : 0] : 0.0);
                }
            }
        }
        if constexpr (kT) {
#pragma unroll
            for (int i = 0; i < R; ++i) {
                double wgt;
                if constexpr (kAtax) wgt = dot[i]; else wgt = rw[i];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    cs[v].x = fma(e[i][v].x, wgt, cs[v].x);
                    cs[v].y = fma(e[i][v].y, wgt, cs[v].y);
                }
            }
        }
    }
    if constexpr (kT) {
        // fold the row groups (ascending) and write this CTA's partial row
#pragma unroll
        for (int v = 0; v < V; ++v) {
            fold[v][tid][0] = cs[v].x;
            fold[v][tid][1] = cs[v].y;
        }
        __syncthreads();
        if (g == 0) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                double t0 = fold[v][cp][0], t1 = fold[v][cp][1];
                for (int gg = 1; gg < G; ++gg) {
                    t0 += fold[v][gg * L + cp][0];
                    t1 += fold[v][gg * L + cp][1];
                }
                double *dst = a.colpart + (long)blockIdx.x * N + col[v];
                if (ok0[v]) st_partial1(dst, t0);
                if (ok1[v]) st_partial1(dst + 1, t1);
            }
        }
    }
}

}  // namespace bto
