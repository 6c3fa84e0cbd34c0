// mv_kernels.cuh -- the matrix-streaming engine behind BiCGK, ATAX, GESUMMV,
// GEMVER (and DGEMV / DGEMVT / BATAX).
//
// One templated kernel streams a row-major fp64 matrix once and evaluates, on
// the tile it holds in registers, any combination of
//   N-product   rowdot[i] += A[i,j] * colw[j]      (q = A p, A x, B x)
//   N2-product  the same on a second matrix         (GESUMMV's B x)
//   T-product   colsum[j] += A[i,j] * roww[i]       (s = A' r, B' y)
//   rank-2      B[i,j] = (A[i,j] + u1[i] v1[j]) + u2[i] v2[j], stored once,
//               the T-product then runs on B        (GEMVER pass 1)
// which is what "fusing the loops" of the reference's organisms means here
// ({_i{_j 1 2}} for BiCGK, {_i{_j 1 3} ..} for GESUMMV,
// {_i{_j 1 2 3 4 5}} for GEMVER).
//
// Decomposition.  The matrix is cut into column strips of SW = 512*V columns;
// a strip is cut into units of R rows.  A thread owns 2*V columns of the strip
// (one or two double2 per row -> every warp load is 512 contiguous bytes) and
// walks DOWN the strip, so
//   * column sums stay in 2*V registers for as long as the CTA stays in the
//     strip and are flushed once per (CTA, strip) into `colpart`;
//   * the column weights colw[j] are loaded once per strip (no re-read of x);
//   * row dots are reduced per unit: warp_transpose_sum across the lanes,
//     shared memory across the 8 warps, one partial per (strip, row) into
//     `rowpart`.
// Units are numbered strip-major and dealt to the G resident CTAs as equal
// contiguous ranges (split_begin), i.e. the grid is persistent, perfectly
// balanced, and a CTA touches at most a couple of strips.  A second tiny
// kernel (finalize_kernel) adds the partials in a fixed order -- the
// reference's "serial ascending-block join" (cemit.py:204-222).
//
// Overheads on top of the algorithmic bytes: rowpart = nstrips*M doubles
// (N/SW of a vector per row: 1/(64*V) of the matrix), colpart <= slots*N.
#pragma once
#include "common.cuh"

namespace bto {

enum : int { kFlagN = 1, kFlagN2 = 2, kFlagT = 4, kFlagRank2 = 8 };

struct MvArgs {
    const double *A;        // matrix streamed (M x N row-major)
    const double *A2;       // second matrix (kFlagN2)
    double *Bout;           // rank-2 result (kFlagRank2)
    const double *colw;     // [N] weights of the N-products
    const double *roww;     // [M] weights of the T-product
    const double *u1, *v1, *u2, *v2;   // rank-2 update vectors
    double *rowpart;        // [nstrips][M]
    double *rowpart2;       // [nstrips][M] (kFlagN2)
    double *colpart;        // [slots][N]
    long M, N;
    long units_per_strip;   // ceil(M / R)
    long total_units;       // nstrips * units_per_strip
    int nstrips;
};

// Column epilogue of a pass (the same four cases as FinArgs::cmode below), for the kernels that
// finish a column inside the producer (DIRECT mode of mv_tile_walk).
struct ColEpilogue {
    double *out;              // [N]
    const double *z;          // mode 2: out = sum*scale + z
    double scale;
    int mode;                 // 1 plain, 2 axpz, 3 scale
    int vector_store;         // out is 16-byte aligned: one 128-bit store per column pair
};

__device__ __forceinline__ double apply_col_epilogue(const ColEpilogue &e, long j, double s)
{
    if (e.mode == 2) return __dadd_rn(__dmul_rn(s, e.scale), e.z[j]);   // t4 = t3*beta ; x = t4 + z
    if (e.mode == 3) return __dmul_rn(s, e.scale);                       // y = t1*beta
    return s;
}

template <bool ALIGNED, bool BYPASS_L1>
__device__ __forceinline__ double2 mv_load(const double *base, long row, long N,
                                           long j, bool ok0, bool ok1)
{
    const double *p = base + row * N + j;
    if constexpr (ALIGNED) {
        return ok0 ? ld_stream2<BYPASS_L1>(p) : make_double2(0.0, 0.0);
    }
    double2 v;
    v.x = ok0 ? ld_stream1<BYPASS_L1>(p) : 0.0;
    v.y = ok1 ? ld_stream1<BYPASS_L1>(p + 1) : 0.0;
    return v;
}

// Per-thread view of the strip the CTA is walking down.
template <int V>
struct StripState {
    long jcol[V];                     // first of the two columns of each double2; 0 for a thread
                                      // whose columns are outside the matrix (its loads stay
                                      // unconditional and in bounds, the values are dropped)
    bool ok0[V], ok1[V];              // column j / j+1 inside the matrix
    double2 cw[V], cv1[V], cv2[V];    // colw, v1, v2 at those columns
    double2 csum[V];                  // running column sums (T-product)
};

// One unit = R rows of the strip.  INTERIOR units (all R rows inside the matrix)
// load without predicates, so every load is issued before the first use -- in a
// ragged last strip the threads beyond column N read column 0 instead and drop
// the values; units that run past row M are guarded.
// MODE: 0 guarded, 1 interior (rows and strip inside), 2 interior rows of a ragged strip
template <int FLAGS, int R, int V, bool ALIGNED, int MODE>
__device__ __forceinline__ void mv_unit(const MvArgs &a, StripState<V> &st, long r0,
                                        double (&rp)[R],
                                        double (&rp2)[(FLAGS & kFlagN2) ? R : 1])
{
    constexpr bool kN = (FLAGS & kFlagN) != 0;
    constexpr bool kN2 = (FLAGS & kFlagN2) != 0;
    constexpr bool kT = (FLAGS & kFlagT) != 0;
    constexpr bool kRank2 = (FLAGS & kFlagRank2) != 0;
#ifndef BTO_N2_BYPASS
#define BTO_N2_BYPASS 1
#endif
    constexpr bool kBypass = kN2 && BTO_N2_BYPASS;   // L1 bypass only for the two-matrix pass (common.cuh)
    constexpr bool kInterior = MODE != 0;
    constexpr bool kRagged = MODE == 2;
    const long M = a.M, N = a.N;
    long (&jcol)[V] = st.jcol;
    bool (&ok0)[V] = st.ok0;
    bool (&ok1)[V] = st.ok1;
    double2 (&cw)[V] = st.cw;
    double2 (&cv1)[V] = st.cv1;
    double2 (&cv2)[V] = st.cv2;
    double2 (&csum)[V] = st.csum;
    double2 t[R][V], t2[kN2 ? R : 1][V];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const bool rv = kInterior || (r0 + i < M);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if constexpr (kInterior && ALIGNED) {
                t[i][v] = ld_stream2<kBypass>(a.A + (r0 + i) * N + jcol[v]);
                if constexpr (kN2) t2[i][v] = ld_stream2<kBypass>(a.A2 + (r0 + i) * N + jcol[v]);
            } else {
                t[i][v] = mv_load<ALIGNED, kBypass>(a.A, r0 + i, N, jcol[v],
                                           rv && ok0[v], rv && ok1[v]);
                if constexpr (kN2) {
                    t2[i][v] = mv_load<ALIGNED, kBypass>(a.A2, r0 + i, N, jcol[v],
                                                rv && ok0[v], rv && ok1[v]);
                }
            }
        }
    }
    if constexpr (kRagged) {              // drop what the threads outside the matrix loaded
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if (!ok0[v]) {
                    t[i][v] = make_double2(0.0, 0.0);
                    if constexpr (kN2) t2[i][v] = make_double2(0.0, 0.0);
                }
            }
        }
    }
    double rw[kT ? R : 1], ru1[kRank2 ? R : 1], ru2[kRank2 ? R : 1];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const bool rv = kInterior || (r0 + i < M);
        if constexpr (kT) rw[i] = rv ? __ldg(a.roww + r0 + i) : 0.0;
        if constexpr (kRank2) {
            ru1[i] = rv ? __ldg(a.u1 + r0 + i) : 0.0;
            ru2[i] = rv ? __ldg(a.u2 + r0 + i) : 0.0;
        }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const long row = r0 + i;
        const bool rv = kInterior || (row < M);
        double dot = 0.0, dot2 = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            double2 e = t[i][v];
            if constexpr (kRank2) {
                // t0 = u1*v1 ; t1 = A + t0 ; t2 = u2*v2 ; B = t1 + t2
                e.x = __dadd_rn(__dadd_rn(e.x, __dmul_rn(ru1[i], cv1[v].x)),
                                __dmul_rn(ru2[i], cv2[v].x));
                e.y = __dadd_rn(__dadd_rn(e.y, __dmul_rn(ru1[i], cv1[v].y)),
                                __dmul_rn(ru2[i], cv2[v].y));
                double *dst = a.Bout + row * N + jcol[v];
                if constexpr (ALIGNED) {
                    if (MODE == 1 || (rv && ok0[v])) st_stream2(dst, e);
                } else {
                    if (rv && ok0[v]) st_stream1(dst, e.x);
                    if (rv && ok1[v]) st_stream1(dst + 1, e.y);
                }
            }
            if constexpr (kN) {
                dot = fma(e.x, cw[v].x, dot);
                dot = fma(e.y, cw[v].y, dot);
            }
            if constexpr (kN2) {
                dot2 = fma(t2[i][v].x, cw[v].x, dot2);
                dot2 = fma(t2[i][v].y, cw[v].y, dot2);
            }
            if constexpr (kT) {
                csum[v].x = fma(e.x, rw[i], csum[v].x);
                csum[v].y = fma(e.y, rw[i], csum[v].y);
            }
        }
        rp[i] = dot;
        if constexpr (kN2) rp2[i] = dot2;
    }
}

// MINB: minimum resident CTAs per SM the register allocator must leave room
// for (__launch_bounds__); trades registers per thread (loads in flight per
// thread) against warps per SM.
// The walk of one CTA over its unit range.
// DIRECT (short, very wide matrices: thousands of strips, a handful of units each): CTAs are dealt
// WHOLE strips, so a strip's column sums are complete when the CTA leaves it -- the column epilogue
// is applied here and the result stored; no column partials, no column side in the join.
template <int FLAGS, int R, int V, bool ALIGNED, bool DIRECT = false>
__device__ __forceinline__ void mv_tile_walk(const MvArgs &a, const ColEpilogue *direct = nullptr)
{
    constexpr bool kN = (FLAGS & kFlagN) != 0;
    constexpr bool kN2 = (FLAGS & kFlagN2) != 0;
    constexpr bool kT = (FLAGS & kFlagT) != 0;
    constexpr bool kRank2 = (FLAGS & kFlagRank2) != 0;
    static_assert(!kN2 || kN, "the second N-product rides on the first");
    constexpr int kRowSets = kN2 ? 2 : 1;
    constexpr int kLanesPerRow = 32 / R;
    constexpr long kStripWidth = (long)kThreads * 2 * V;
    // Ragged last strip, rows inside: unconditional loads with clamped columns (mv_unit MODE 2).
    // Tall tiles only: their guarded unit is the slow one -- GEMVER pass 1 at N = 2500 ran at
    // 3.8 TB/s, 5.8 with this; in the 8-row kernels the extra path costs more than it gives
    // (GESUMMV spills at its 64-register budget, -2.5 %; BiCGK -0.6 % at bench size).
    constexpr bool kRaggedMode = ALIGNED && !kN2 && R >= 16;

    __shared__ double red[2][kRowSets][kWarps][R];

    wait_for_producer_grid();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long G = gridDim.x, cta = blockIdx.x;
    const long u_begin = DIRECT ? split_begin(a.nstrips, G, cta) * a.units_per_strip
                                : split_begin(a.total_units, G, cta);
    const long u_end = DIRECT ? split_begin(a.nstrips, G, cta + 1) * a.units_per_strip
                              : split_begin(a.total_units, G, cta + 1);
    const long M = a.M, N = a.N;

    long strip = -1;
    bool strip_inside = false;
    StripState<V> st;
    long (&jcol)[V] = st.jcol;
    bool (&ok0)[V] = st.ok0;
    bool (&ok1)[V] = st.ok1;
    double2 (&cw)[V] = st.cw;
    double2 (&cv1)[V] = st.cv1;
    double2 (&cv2)[V] = st.cv2;
    double2 (&csum)[V] = st.csum;
    int buf = 0;

    auto flush_colsums = [&]() {
        if constexpr (DIRECT) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if (!ok0[v]) continue;         // (N is even on this path: ok1 == ok0)
                double2 r;
                r.x = apply_col_epilogue(*direct, jcol[v], csum[v].x);
                r.y = apply_col_epilogue(*direct, jcol[v] + 1, csum[v].y);
                if (direct->vector_store) {
                    st_partial2(direct->out + jcol[v], r);
                } else {                       // the caller's vector sits at an odd 8-byte offset
                    direct->out[jcol[v]] = r.x;
                    direct->out[jcol[v] + 1] = r.y;
                }
            }
            return;
        }
        // this CTA's slot among the CTAs that share the strip
        const long first = split_owner(a.total_units, G, strip * a.units_per_strip);
        double *dst = a.colpart + (cta - first) * N;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if constexpr (ALIGNED) {
                if (ok0[v]) st_partial2(dst + jcol[v], csum[v]);
            } else {
                if (ok0[v]) st_partial1(dst + jcol[v], csum[v].x);
                if (ok1[v]) st_partial1(dst + jcol[v] + 1, csum[v].y);
            }
        }
    };

    for (long u = u_begin; u < u_end; ++u) {
        const long c = u / a.units_per_strip;
        const long r0 = (u - c * a.units_per_strip) * R;
        if (c != strip) {
            if (kT && strip >= 0) flush_colsums();
            strip = c;
            strip_inside = (c + 1) * kStripWidth <= N;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const long j = c * kStripWidth + (long)v * (kThreads * 2) + 2 * tid;
                jcol[v] = (kRaggedMode && j >= N) ? 0 : j;
                ok0[v] = j < N;
                ok1[v] = j + 1 < N;
                csum[v] = make_double2(0.0, 0.0);
                if constexpr (kN || kN2) {
                    cw[v].x = ok0[v] ? __ldg(a.colw + j) : 0.0;
                    cw[v].y = ok1[v] ? __ldg(a.colw + j + 1) : 0.0;
                }
                if constexpr (kRank2) {
                    cv1[v].x = ok0[v] ? __ldg(a.v1 + j) : 0.0;
                    cv1[v].y = ok1[v] ? __ldg(a.v1 + j + 1) : 0.0;
                    cv2[v].x = ok0[v] ? __ldg(a.v2 + j) : 0.0;
                    cv2[v].y = ok1[v] ? __ldg(a.v2 + j + 1) : 0.0;
                }
            }
        }

        double rp[R], rp2[kN2 ? R : 1];
        // Interior units (all R rows and the whole strip inside the matrix) take
        // a predicate-free path so that every load of the unit is issued before
        // the first use; edge units take the guarded path.
        if (strip_inside && r0 + R <= M) {
            mv_unit<FLAGS, R, V, ALIGNED, 1>(a, st, r0, rp, rp2);
        } else if (kRaggedMode && r0 + R <= M) {
            mv_unit<FLAGS, R, V, ALIGNED, kRaggedMode ? 2 : 0>(a, st, r0, rp, rp2);
        } else {
            mv_unit<FLAGS, R, V, ALIGNED, 0>(a, st, r0, rp, rp2);
        }

        if constexpr (kN) {
            // lanes -> one value per row, then the 8 warps through shared memory
            warp_transpose_sum<R>(rp, lane);
            if ((lane % kLanesPerRow) == 0) red[buf][0][warp][lane / kLanesPerRow] = rp[0];
            if constexpr (kN2) {
                warp_transpose_sum<R>(rp2, lane);
                if ((lane % kLanesPerRow) == 0)
                    red[buf][kRowSets - 1][warp][lane / kLanesPerRow] = rp2[0];
            }
            __syncthreads();
            if (tid < R * kRowSets) {
                const int set = tid / R, i = tid % R;
                double s = red[buf][set][0][i];
#pragma unroll
                for (int w = 1; w < kWarps; ++w) s += red[buf][set][w][i];
                if (r0 + i < M) {
                    double *dst = set == 1 ? a.rowpart2 : a.rowpart;
                    st_partial1(dst + strip * M + r0 + i, s);
                }
            }
            // red[] is double-buffered: the next unit writes the other half and
            // its __syncthreads orders this unit's reads before buf is reused.
            // (Round 2 replaced this barrier by an mbarrier hand-off -- producers arrive, only the
            //  consumer warp waits, the rest go on to the next unit's loads: BiCGK 7.07 -> 6.96 TB/s,
            //  GEMVER 6.61 -> 6.58, profiles/r02/ab/ab_mv_handoff.log.  The barrier stays.  Dealing the
            //  8-warp sums to all warps instead of warp 0's first threads: BiCGK 7.07 -> 7.00,
            //  ab_mv_spread.log.)
            buf ^= 1;
        }
    }
    if (kT && strip >= 0) flush_colsums();
}

template <int FLAGS, int R, int V, bool ALIGNED, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
mv_tile_kernel(const MvArgs a)
{
    mv_tile_walk<FLAGS, R, V, ALIGNED>(a);
}

struct MvDirectArgs {
    MvArgs mv;
    ColEpilogue col;
};

template <int FLAGS, int R, int V, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
mv_tile_direct_kernel(const MvDirectArgs d)
{
    mv_tile_walk<FLAGS, R, V, true, true>(d.mv, &d.col);
}

// ---- finaliser: fixed-order join of the partials + the sequence's epilogue ----
enum ColMode : int { kColNone = 0, kColPlain = 1, kColAxpz = 2, kColScale = 3 };
enum RowMode : int { kRowNone = 0, kRowPlain = 1, kRowGesummv = 2, kRowScale = 3,
                     kRowDgemv = 4 };

struct FinArgs {
    // column side: out[j] = f( sum_k colpart[k][j] )
    const double *colpart;
    double *colout;
    const double *colz;       // kColAxpz: x = sum*cscale + z
    double cscale;
    int cmode;
    long N;
    long units_per_strip, total_units, grid;   // geometry of the producer launch
    long strip_width;
    // row side: out[i] = f( sum_c rowpart[c][i] )
    const double *rowpart, *rowpart2;
    double *rowout;
    const double *rowy;       // kRowDgemv: z = sum*alpha + y*beta
    double ralpha, rbeta;
    int rmode;
    long M;
    int nstrips;
    int col_blocks;           // CTAs [0, col_blocks) do columns, the rest rows
    int row_group;            // threads that share one row's join: 1, 32 (a warp) or 256 (the CTA)
    int col_cols;             // columns per column CTA: kJoinCols (8 warps share a column's partials)
                              // or kThreads (a thread per column: few partials, very many columns)
};

constexpr int kJoinCols = 32;  // columns per column CTA of finalize_kernel

// Sum of `count` partials `stride` apart in a FIXED order that exposes 8
// independent load/add chains (the partials sit in L2; a single dependent chain
// would pay the L2 latency `count` times): lane k takes partials k, k+8, ..;
// the eight lane sums are added pairwise.
__device__ __forceinline__ double strided_sum(const double *p, long count, long stride)
{
    double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    long k = 0;
    for (; k + 8 <= count; k += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += p[(k + u) * stride];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {          // tail, predicated so acc[] stays in registers
        if (k + u < count) acc[u] += p[(k + u) * stride];
    }
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// ascending join of the column partials of column j (no epilogue)
__device__ __forceinline__ double join_column(const FinArgs &f, long j)
{
    const long strip = j / f.strip_width;
    const long first = split_owner(f.total_units, f.grid, strip * f.units_per_strip);
    const long last = split_owner(f.total_units, f.grid, (strip + 1) * f.units_per_strip - 1);
    return strided_sum(f.colpart + j, last - first + 1, f.N);
}

__device__ __forceinline__ double column_epilogue(const FinArgs &f, long j, double s)
{
    if (f.cmode == kColAxpz) {            // t4 = t3*beta ; x = t4 + z
        s = __dadd_rn(__dmul_rn(s, f.cscale), f.colz[j]);
    } else if (f.cmode == kColScale) {    // y = t1*beta
        s = __dmul_rn(s, f.cscale);
    }
    return s;
}

// The same join done by a whole CTA for kJoinCols adjacent columns: lane = column,
// warp w sums the w-th eighth of the partials (strided_sum order inside), the eight
// warp sums are added pairwise by warp 0.  A fixed order again, but the dependent
// L2 round trips per thread drop from count/8 to count/64 -- what a mid-size call
// (n ~ 2-8 K, 100+ partials per column, a 20 us tile kernel) spends its time on.
__device__ __forceinline__ void join_columns_cta(const FinArgs &f, long j0)
{
    __shared__ double warp_part[kWarps][kJoinCols];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long j = j0 + lane;
    if (j < f.N) {
        const long strip = j / f.strip_width;
        const long first = split_owner(f.total_units, f.grid, strip * f.units_per_strip);
        const long last = split_owner(f.total_units, f.grid, (strip + 1) * f.units_per_strip - 1);
        const long count = last - first + 1;
        const long k0 = (count * warp) / kWarps, k1 = (count * (warp + 1)) / kWarps;
        warp_part[warp][lane] = strided_sum(f.colpart + j + k0 * f.N, k1 - k0, f.N);
    }
    __syncthreads();
    if (warp == 0 && j < f.N) {
        static_assert(kWarps == 8, "pairwise tree below is written for 8 warps");
        const double s = ((warp_part[0][lane] + warp_part[1][lane]) +
                          (warp_part[2][lane] + warp_part[3][lane])) +
                         ((warp_part[4][lane] + warp_part[5][lane]) +
                          (warp_part[6][lane] + warp_part[7][lane]));
        st_partial1(f.colout + j, column_epilogue(f, j, s));
    }
}

// epilogue of row i given its joined sum(s)
__device__ __forceinline__ void row_epilogue(const FinArgs &f, long i, double s, double s2)
{
    if (f.rmode == kRowGesummv) {         // t1 = t0*alpha ; t3 = t2*beta ; y = t1 + t3
        s = __dadd_rn(__dmul_rn(s, f.ralpha), __dmul_rn(s2, f.rbeta));
    } else if (f.rmode == kRowScale) {    // w = t5*alpha
        s = __dmul_rn(s, f.ralpha);
    } else if (f.rmode == kRowDgemv) {    // t1 = t0*alpha ; t2 = y*beta ; z = t1 + t2
        s = __dadd_rn(__dmul_rn(s, f.ralpha), __dmul_rn(f.rowy[i], f.rbeta));
    }
    st_partial1(f.rowout + i, s);
}

// Row side of the join for row CTA `rblock`.  One partial per strip and row: a square
// matrix has 64 strips and a thread per row is right; a short, very wide one has thousands
// (N / 512) and few rows, so a warp or the whole CTA shares a row -- thread k adds strips
// k, k + G, .. in strided_sum order, then the fixed-order warp / CTA reduction.
// (its own kernel: the wide variant is the rare one and must not set the register count of the
// join every square matrix runs)
__global__ void __launch_bounds__(kThreads)
finalize_rows_wide_kernel(const FinArgs f)
{
    wait_for_producer_grid();
    const long rblock = blockIdx.x;
    const bool two = f.rmode == kRowGesummv;
    const int G = f.row_group;
    const int k = G == 32 ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
    const long i = G == 32 ? rblock * kWarps + (threadIdx.x >> 5) : rblock;
    const bool live = i < f.M;                                    // uniform per warp (G = 32) / CTA
    const long mine = live && k < f.nstrips ? (f.nstrips - k + G - 1) / G : 0;
    const long first = (live ? i : 0) + (long)k * f.M;
    double s = strided_sum(f.rowpart + first, mine, (long)G * f.M);
    double s2 = two ? strided_sum(f.rowpart2 + first, mine, (long)G * f.M) : 0.0;
    if (G == 32) {
        s = warp_sum(s);
        if (two) s2 = warp_sum(s2);
    } else {
        __shared__ double scratch[kWarps];
        s = block_sum(s, scratch);
        if (two) s2 = block_sum(s2, scratch);
    }
    if (live && k == 0) row_epilogue(f, i, s, s2);
}

__device__ __forceinline__ void finalize_rows_cta(const FinArgs &f, long rblock)
{
    const long i = rblock * kThreads + threadIdx.x;
    if (i < f.M) {
        const double s = strided_sum(f.rowpart + i, f.nstrips, f.M);
        const double s2 = f.rmode == kRowGesummv ? strided_sum(f.rowpart2 + i, f.nstrips, f.M) : 0.0;
        row_epilogue(f, i, s, s2);
    }
}

__global__ void __launch_bounds__(kThreads)
finalize_kernel(const FinArgs f)
{
    wait_for_producer_grid();
    if ((int)blockIdx.x < f.col_blocks) {
        if (f.col_cols == kThreads) {
            const long j = (long)blockIdx.x * kThreads + threadIdx.x;
            if (j < f.N) st_partial1(f.colout + j, column_epilogue(f, j, join_column(f, j)));
        } else {
            join_columns_cta(f, (long)blockIdx.x * kJoinCols);
        }
    } else {
        finalize_rows_cta(f, (long)blockIdx.x - f.col_blocks);
    }
}

// (Round 2 tried folding the join into the producer for mid-size matrices -- the last CTA to arrive
// at a strip / row unit adds its partials, ticket pattern of vec_kernels.cuh -- and measured it
// SLOWER than this second launch: BiCGK n = 2048 16.2 us against 9.5 us, n = 4096 41.8 against
// 29.7 (profiles/r02/midsize_join_in_producer.log).  One CTA per strip then adds ~74 partials per
// column as a chain of L2 round trips, where finalize_kernel spreads the same loads over N/32 CTAs;
// the launch it saves costs ~3.5 us under PDL.  Not kept.)

// ---- join fused with the cross-GPU exchange (row-sharded runtime) ------------
//
// Every rank owns a row shard and therefore a PARTIAL of each column-indexed
// result (s = A'r, y = A'(Ax), B'y, the AXPYDOT scalar).  Instead of joining
// locally and then calling a library all-reduce, the join kernel itself does
// the exchange over NVLink peer memory (one-shot, for vectors of a few
// hundred KiB the latency-optimal scheme):
//   A  join my columns into MY exchange buffer (symmetric memory, mapped by
//      every peer), double-buffered by call parity;
//   B  publish: one flag per (source rank, CTA) in every peer's flag array,
//      st.release.sys after a system fence; then wait until every peer's flag
//      for this CTA shows this call's epoch (ld.acquire.sys);
//   C  add the `world` partials of my columns in RANK ORDER straight from the
//      peers' buffers -- every rank computes the same bits -- apply the
//      sequence's epilogue, store the result.
// A CTA only depends on the same-numbered CTA of the peers, so no grid-wide
// barrier is needed; row-side joins ride in the same launch as extra CTAs.
// `phases` (bit 0: A+publish, bit 1: wait+C) exists so that one GPU can stand in
// for all ranks in tests: publish for every rank first, then reduce for every
// rank -- one kernel over all ranks' data, nobody ever waits.
constexpr int kExchCtas = 64;

// Device-resident exchange state of a rank (what must survive CUDA-graph replay cannot sit in
// kernel arguments): state[0] = exchanges completed so far (the epoch), state[1] = ticket of the
// column CTAs that have finished the current exchange, state[2] = error word (kExchTimedOut).
enum : unsigned int { kExchTimedOut = 1u };
constexpr unsigned long long kExchTimeoutNs = 20ull * 1000ull * 1000ull * 1000ull;   // 20 s

struct ExchArgs {
    FinArgs fin;                   // local partials + epilogue + row side
    double *const *exch;           // [world] every rank's exchange buffer (peer-mapped)
    unsigned int *const *flags;    // [world] every rank's flags [world][kExchCtas]
    unsigned int *state;           // this rank's exchange state (see above)
    long half;                     // doubles per parity half of the exchange buffer
    int rank, world;
    int phases;
};

__device__ __forceinline__ void st_release_sys(unsigned int *p, unsigned int v)
{
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ double ld_relaxed_sys(const double *p)
{
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long global_timer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kThreads)
join_exchange_kernel(const ExchArgs e)
{
    wait_for_producer_grid();
    const FinArgs &f = e.fin;
    if ((int)blockIdx.x >= kExchCtas) {          // row side: purely local
        finalize_rows_cta(f, (long)blockIdx.x - kExchCtas);
        return;
    }
    // The epoch of THIS exchange: one more than the exchanges completed.  Every column CTA
    // reads the counter before it takes its end-of-kernel ticket, and the counter moves only
    // when the last ticket has been taken, so all CTAs of a launch see the same value; a
    // replayed CUDA graph gets a fresh epoch each time.
    __shared__ unsigned int s_epoch;
    __shared__ bool s_timed_out;
    if (threadIdx.x == 0) {
        unsigned int done;
        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(done) : "l"(e.state) : "memory");
        s_epoch = done + 1u;
        s_timed_out = false;
    }
    __syncthreads();
    const unsigned int epoch = s_epoch;
    const long buf_offset = (long)(epoch & 1u) * e.half;
    const int cta = blockIdx.x;
    const long c_lo = (f.N * cta) / kExchCtas, c_hi = (f.N * (cta + 1)) / kExchCtas;
    if (e.phases & 1) {
        double *mine = e.exch[e.rank] + buf_offset;
        for (long j = c_lo + threadIdx.x; j < c_hi; j += kThreads) mine[j] = join_column(f, j);
        __syncthreads();
        if ((int)threadIdx.x < e.world) {
            __threadfence_system();
            st_release_sys(e.flags[threadIdx.x] + (long)e.rank * kExchCtas + cta, epoch);
        }
    }
    if (e.phases & 2) {
        if ((int)threadIdx.x < e.world) {
            // A peer may already be one exchange AHEAD (it needs our flag for epoch + 1 to get
            // any further, and epoch + 1 uses the other half of the buffers), so the test is
            // "has reached", not "equals": an equality test would spin forever on such a peer.
            const unsigned int *flag = e.flags[e.rank] + (long)threadIdx.x * kExchCtas + cta;
            const unsigned long long t0 = global_timer_ns();
            unsigned int spins = 0;
            while ((int)(ld_acquire_sys(flag) - epoch) < 0) {
                if ((++spins & 0x3ffu) == 0 && global_timer_ns() - t0 > kExchTimeoutNs) {
                    s_timed_out = true;             // a peer never arrived: fail loudly, do not hang
                    atomicOr(e.state + 2, kExchTimedOut);
                    break;
                }
            }
        }
        __syncthreads();
        const bool dead = s_timed_out;
        for (long j = c_lo + threadIdx.x; j < c_hi; j += kThreads) {
            double s = ld_relaxed_sys(e.exch[0] + buf_offset + j);
            for (int p = 1; p < e.world; ++p) s += ld_relaxed_sys(e.exch[p] + buf_offset + j);
            f.colout[j] = dead ? __longlong_as_double(0x7ff8000000000000ll) : column_epilogue(f, j, s);
        }
        // last column CTA out: the exchange is complete on this rank
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(e.state + 1, 1u) == kExchCtas - 1) {
                e.state[1] = 0u;
                __threadfence();
                e.state[0] = epoch;
            }
        }
    }
}

// x = colsum*beta + z on its own (the sharded GEMVER exchanges colsum first)
__global__ void __launch_bounds__(kThreads)
axpz_kernel(const double *colsum, double beta, const double *z, double *x, long n)
{
    const long j = (long)blockIdx.x * kThreads + threadIdx.x;
    if (j < n) x[j] = __dadd_rn(__dmul_rn(colsum[j], beta), z[j]);
}

}  // namespace bto
