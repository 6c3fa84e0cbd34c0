// host_plan.cuh -- launch planning: vector kernels, the matrix tile engine, joins
// Part of the host side of libbto_b200.so; included by api.cu (one translation unit).
#pragma once
#include "host_context.cuh"
#include "mv_kernels.cuh"
#include "skinny_kernels.cuh"
#include "rowstream_kernels.cuh"
#include "vec_kernels.cuh"

namespace bto_host {
namespace {          // internal linkage: nothing here is part of the C ABI

using namespace bto;

// ---------------------------------------------------------------------------
// vector kernels

using VecKernel = void (*)(const VecArgs);

template <int OP>
VecKernel vec_kernel_ptr(int unroll, bool aligned)
{
    if (!aligned) return vec_kernel<OP, 1, false>;
    switch (unroll) {
        case 1: return vec_kernel<OP, 1, true>;
        case 2: return vec_kernel<OP, 2, true>;
        default: return vec_kernel<OP, 4, true>;
    }
}

template <int OP>
int launch_vec(DeviceCtx &c, VecArgs g, cudaStream_t stream)
{
    if (g.n < 1) return fail(BTO_ERR_INVALID, "extent M=%ld must be >= 1", g.n);
    const bool aligned = aligned16(g.a) && aligned16(g.b) && aligned16(g.out) &&
                         (OP == kWaxpby || aligned16(g.c));
    VecKernel fn = vec_kernel_ptr<OP>((int)g_tuning.vec_unroll, aligned);
    int occ = 1;
    BTO_TRY(occupancy_of(c, fn, &occ));
    const long per_sm = g_tuning.vec_grid_per_sm > 0 ? g_tuning.vec_grid_per_sm : occ;
    long grid = (long)c.sm_count * per_sm;
    const long work = ((aligned ? (g.n + 1) / 2 : g.n) + kThreads - 1) / kThreads;
    if (grid > work) grid = work;
    if (grid < 1) grid = 1;
    if (OP == kAxpydot) {
        WsLayout lay;
        const size_t off = lay.take((size_t)grid);
        BTO_TRY(reserve_ws(c, stream, lay.total));
        g.partials = reinterpret_cast<double *>(c.ws + off);
        g.ticket = c.tickets;
    }
    char what[64];
    snprintf(what, sizeof(what), "vec_kernel<%d,%d,%d>", OP, aligned ? (int)g_tuning.vec_unroll : 1,
             aligned ? 1 : 0);
    return launch_dependent(fn, (unsigned)grid, g, stream, what);
}

// ---------------------------------------------------------------------------
// matrix kernels

using MvKernel = void (*)(const MvArgs);
using MvDirectKernel = void (*)(const MvDirectArgs);

struct MvPlan {
    int R = 8, V = 1;
    bool aligned = true;
    long strip_width = 512;
    int nstrips = 1;
    long units_per_strip = 1, total_units = 1;
    long grid = 1;
    long slots = 1;        // max CTAs sharing one strip
    int flags = 0, minb = 1;   // template arguments of `fn` (for the launch record)
    MvKernel fn = nullptr;
    MvDirectKernel direct_fn = nullptr;   // set: whole strips per CTA, columns finished in the producer

};

template <int FLAGS, int R, int V>
MvKernel mv_kernel_minb(int minb)
{
    switch (minb) {
        case 2: return mv_tile_kernel<FLAGS, R, V, true, 2>;
        case 3: return mv_tile_kernel<FLAGS, R, V, true, 3>;
        case 4: return mv_tile_kernel<FLAGS, R, V, true, 4>;
        case 6: return mv_tile_kernel<FLAGS, R, V, true, 6>;
        default: return mv_tile_kernel<FLAGS, R, V, true, 1>;
    }
}

// Supported tile shapes: (rows, double2 per thread) = (8,1) always; (16,1) for
// single-matrix kinds; (32,1) for kinds without row dots; (8,2) for A x alone.
template <int FLAGS>
bool mv_shape_ok(int R, int V)
{
    if (R == 8 && V == 1) return true;
    if (FLAGS & kFlagN2) return false;
    if (R == 16 && V == 1) return true;
    if (R == 32 && V == 1) return (FLAGS & kFlagN) == 0;
    if (R == 8 && V == 2) return FLAGS == kFlagN || FLAGS == (kFlagT | kFlagRank2) || FLAGS == (kFlagN | kFlagT);
    return false;
}

template <int FLAGS>
MvKernel mv_kernel_ptr(int R, int V, bool aligned, int minb)
{
    if (!aligned) return mv_tile_kernel<FLAGS, 8, 1, false, 1>;
    if constexpr ((FLAGS & kFlagN2) == 0) {
        if (R == 16 && V == 1) return mv_kernel_minb<FLAGS, 16, 1>(minb);
        if constexpr ((FLAGS & kFlagN) == 0) {
            if (R == 32 && V == 1) return mv_kernel_minb<FLAGS, 32, 1>(minb);
        }
        if constexpr (FLAGS == kFlagN || FLAGS == (kFlagT | kFlagRank2) || FLAGS == (kFlagN | kFlagT)) {
            if (R == 8 && V == 2) return mv_kernel_minb<FLAGS, 8, 2>(minb);
        }
    }
    return mv_kernel_minb<FLAGS, 8, 1>(minb);
}

// Launch defaults per pass kind, from the B200 sweep at n = 32768
// (profiles/r01/sweep2_passes.json): {rows per unit, double2 per thread, CTAs per SM
// (0 = what the occupancy calculator allows)}.
struct MvDefault { int rows, vec, grid_per_sm, minb; };

template <int FLAGS>
constexpr MvDefault mv_default()
{
    if (FLAGS == (kFlagN | kFlagT)) return {8, 2, 8, 2};        // BiCGK         7.07 TB/s (1024-column strips: half the barriers per byte)
    if (FLAGS == (kFlagN | kFlagN2)) return {8, 1, 4, 4};       // GESUMMV       7.04 TB/s
    if (FLAGS == (kFlagT | kFlagRank2)) return {16, 1, 2, 1};   // GEMVER pass 1 6.29 TB/s (r+w)
    if (FLAGS == (kFlagN | kFlagRank2)) return {8, 1, 4, 2};    // column-major GEMVER pass 1 6.38 TB/s (r+w)
    if (FLAGS == kFlagT) return {32, 1, 2, 1};                  // A' y          7.17 TB/s
    return {8, 2, 8, 2};                                        // A x           7.20 TB/s
}

// The column-direct variant exists for the passes with column sums, in the tile shapes of
// mv_shape_ok at the pass kind's default MINB.
template <int FLAGS>
MvDirectKernel mv_direct_kernel_ptr(int R, int V)
{
    if constexpr ((FLAGS & kFlagT) != 0) {
        constexpr int minb = mv_default<FLAGS>().minb;
        if (R == 8 && V == 1) return mv_tile_direct_kernel<FLAGS, 8, 1, minb>;
        if (R == 16 && V == 1) return mv_tile_direct_kernel<FLAGS, 16, 1, minb>;
        if constexpr ((FLAGS & kFlagN) == 0) {
            if (R == 32 && V == 1) return mv_tile_direct_kernel<FLAGS, 32, 1, minb>;
        }
        if constexpr (FLAGS == (kFlagT | kFlagRank2) || FLAGS == (kFlagN | kFlagT)) {
            if (R == 8 && V == 2) return mv_tile_direct_kernel<FLAGS, 8, 2, minb>;
        }
    }
    return nullptr;
}

template <int FLAGS>
int plan_mv(DeviceCtx &c, long M, long N, bool aligned, MvPlan *p)
{
    constexpr MvDefault dflt = mv_default<FLAGS>();
    int R = g_tuning.mv_rows ? (int)g_tuning.mv_rows : dflt.rows;
    int V = g_tuning.mv_vec ? (int)g_tuning.mv_vec : dflt.vec;
    int minb = g_tuning.mv_minb ? (int)g_tuning.mv_minb : dflt.minb;
    if (!aligned || !mv_shape_ok<FLAGS>(R, V)) { R = 8; V = 1; }
    // A ragged last strip takes the guarded (predicated) unit, which is slow for tall tiles; when
    // it is a large share of the matrix (N = 1000: half of it) 8-row tiles win (GEMVER 3.9 -> 5.3 TB/s)
    if (!g_tuning.mv_rows && R > 8 && N % ((long)kThreads * 2 * V) != 0 && N < 4L * kThreads * 2 * V) R = 8;
    // fewer rows than a tall tile has: the rows beyond M would be predicated-off loads in every unit
    if (!g_tuning.mv_rows && aligned) {
        while (R > 8 && M <= R / 2) R /= 2;
    }
    // Mid-size matrices (profiles/r02/midsize_tune_before.log): the bench-size shapes leave too few
    // units to spread -- 1024-column strips need N > 2048 (BiCGK n = 2048: 9.4 -> 8.7 us with 512; n = 3072 is
    // better off with three 1024-column strips),
    // tall tiles need about eight units per resident CTA (GEMVER n = 2048: 20.0 -> 17.9 us with 8 rows)
    if (g_tuning.midsize && aligned) {
        if (!g_tuning.mv_vec && V == 2 && N <= 2048) V = 1;
        if (!g_tuning.mv_rows) {
            const long strips = (N + (long)kThreads * 2 * V - 1) / ((long)kThreads * 2 * V);
            while (R > 8 && strips * ((M + R - 1) / R) < 16L * c.sm_count) R /= 2;
        }
    }
    p->R = R;
    p->V = V;
    p->aligned = aligned;
    p->fn = mv_kernel_ptr<FLAGS>(R, V, aligned, minb);
    p->flags = FLAGS;
    p->minb = !aligned ? 1 : ((minb == 2 || minb == 3 || minb == 4 || minb == 6) ? minb : 1);
    p->strip_width = (long)kThreads * 2 * V;
    p->nstrips = (int)((N + p->strip_width - 1) / p->strip_width);
    p->units_per_strip = (M + R - 1) / R;
    p->total_units = p->units_per_strip * p->nstrips;
    int occ = 1;
    BTO_TRY(occupancy_of(c, p->fn, &occ));
    long per_sm = g_tuning.grid_per_sm > 0 ? g_tuning.grid_per_sm : dflt.grid_per_sm;
    if (per_sm <= 0) per_sm = occ;
    // More CTAs than are resident only pay (tail balance) while each still walks a few dozen units:
    // every CTA adds a column partial per strip to the join (BiCGK n = 8192: 89.5 -> 81.4 us with
    // the resident 2 per SM instead of 8; at n >= 16384 the sweep of round 1 stands)
    if (g_tuning.midsize && !g_tuning.grid_per_sm && (FLAGS & kFlagT)) {
        const long resident = occ < per_sm ? occ : per_sm;
        while (per_sm > resident && p->total_units < 24L * c.sm_count * per_sm) per_sm /= 2;
        if (per_sm < resident) per_sm = resident;
    }
    long grid = (long)c.sm_count * per_sm;
    // small matrices: about 3 units or more per CTA (the prologue and the partial a CTA
    // writes per strip are fixed costs), in whole multiples of the SM count so that every
    // SM carries the same number of CTAs; below one CTA per SM, 2 units per CTA
    const long per_cta = 3;
    if (grid * per_cta > p->total_units) {
        const long waves = p->total_units / (per_cta * c.sm_count);
        grid = waves >= 1 ? waves * c.sm_count : (p->total_units + 1) / 2;
        if (grid > c.sm_count && waves < 1) grid = c.sm_count;
    }
    if (grid < 1) grid = 1;
    p->grid = grid;
    long slots = 1;
    for (int s = 0; s < p->nstrips; ++s) {
        const long first = split_owner(p->total_units, grid, (long)s * p->units_per_strip);
        const long last = split_owner(p->total_units, grid,
                                      (long)(s + 1) * p->units_per_strip - 1);
        if (last - first + 1 > slots) slots = last - first + 1;
    }
    p->slots = slots;
    // Short and very wide: at least 4 whole strips per CTA -> deal strips, finish columns in the producer
    // (no column partials: at M = 8 they are a quarter of the matrix bytes, and their join is N / 256 CTAs)
    p->direct_fn = nullptr;
    if (aligned && (FLAGS & kFlagT) && g_tuning.direct_cols != 0 && !c.exch_active &&
        p->minb == mv_default<FLAGS>().minb && (long)p->nstrips >= 4L * c.sm_count) {
        p->direct_fn = mv_direct_kernel_ptr<FLAGS>(R, V);
        if (p->direct_fn) {
            long g = (long)c.sm_count * per_sm;
            while (g > c.sm_count && (long)p->nstrips < 4 * g) g -= c.sm_count;
            p->grid = g;
            p->slots = 0;                  // no column partials
        }
    }
    return BTO_OK;
}

void fill_geometry(const MvPlan &p, MvArgs *a, long M, long N)
{
    a->M = M;
    a->N = N;
    a->units_per_strip = p.units_per_strip;
    a->total_units = p.total_units;
    a->nstrips = p.nstrips;
}

int launch_mv(const MvPlan &p, const MvArgs &a, cudaStream_t stream)
{
    char what[64];
    snprintf(what, sizeof(what), "mv_tile_kernel<%d,%d,%d,%d,%d>", p.flags, p.R, p.V, p.aligned ? 1 : 0,
             p.minb);
    return launch_dependent(p.fn, (unsigned)p.grid, a, stream, what);
}

// Launch the join of `f` (geometry already filled in).  While a sharded
// entry point is active and the join has a column side, the cross-GPU exchange
// is fused into it (join_exchange_kernel); otherwise the plain local join runs.
int launch_join(DeviceCtx &c, FinArgs f, cudaStream_t stream)
{
    // threads per row of the row-side join: a thread (in the join kernel itself), or a warp /
    // the whole CTA in finalize_rows_wide_kernel when a row has hundreds of strip partials
    f.row_group = f.nstrips <= 128 ? 1 : (f.nstrips <= 4096 ? 32 : kThreads);
    if (f.rmode != kRowNone && f.row_group > 1) {
        const long rows_per_cta = kThreads / f.row_group;
        const long rb = (f.M + rows_per_cta - 1) / rows_per_cta;
        BTO_TRY(launch_dependent(finalize_rows_wide_kernel, (unsigned)rb, f, stream,
                                 "finalize_rows_wide_kernel"));
        f.rmode = kRowNone;
        if (f.cmode == kColNone) return BTO_OK;
    }
    const long rb = f.rmode != kRowNone ? (f.M + kThreads - 1) / kThreads : 0;
    if (c.exch_active && f.cmode != kColNone) {
        if (2 * f.N > c.exch_capacity) {
            return fail(BTO_ERR_INVALID, "exchange buffer holds %ld doubles, need %ld",
                        c.exch_capacity, 2 * f.N);
        }
        ExchArgs e{};
        e.fin = f;
        e.exch = c.exch_bufs;
        e.flags = c.exch_flags;
        e.state = c.exch_state;
        e.half = c.exch_capacity / 2;
        e.rank = c.exch_rank;
        e.world = c.exch_world;
        e.phases = (int)g_tuning.exchange_phases;
        return launch_dependent(join_exchange_kernel, (unsigned)(kExchCtas + rb), e, stream,
                                "join_exchange_kernel");
    }
    // few partials per column (a short, wide matrix: about grid / nstrips of them): a thread per
    // column; otherwise 8 warps share the partials of 32 columns
    const long per_col = f.nstrips > 0 ? f.grid / f.nstrips + 2 : f.grid;
    f.col_cols = per_col <= 8 ? kThreads : kJoinCols;
    const long cb = f.cmode != kColNone ? (f.N + f.col_cols - 1) / f.col_cols : 0;
    f.col_blocks = (int)cb;
    return launch_dependent(finalize_kernel, (unsigned)(cb + rb), f, stream, "finalize_kernel");
}

int launch_finalize(DeviceCtx &c, const MvPlan &p, FinArgs f, long M, long N, cudaStream_t stream)
{
    f.M = M;
    f.N = N;
    f.units_per_strip = p.units_per_strip;
    f.total_units = p.total_units;
    f.grid = p.grid;
    f.strip_width = p.strip_width;
    f.nstrips = p.nstrips;
    return launch_join(c, f, stream);
}

int check_mn(long M, long N)
{
    if (M < 1 || N < 1) {
        return fail(BTO_ERR_INVALID, "extents M=%ld N=%ld must be >= 1", M, N);
    }
    return BTO_OK;
}

bool mat_aligned(long N, const void *a, const void *b = nullptr, const void *c = nullptr)
{
    return (N % 2 == 0) && aligned16(a) && aligned16(b) && aligned16(c);
}

// One streaming pass producing row dots and/or column sums, then the join.
// prepare() plans the launch and books its partial buffers in the sequence's
// workspace layout; run() launches after the workspace has been sized once,
// so no pointer handed out earlier in the sequence can move.
// ---- narrow matrices (skinny_kernels.cuh) --------------------------------------------

struct SkinnyPlan {
    bool pair = true;          // column pairs (double2) or single columns per thread
    int V = 1;                 // column slots per thread
    int L = 1;                 // threads per row (<= 32)
    long grid = 0;             // 0: not in use
    long rows_per_cta = 0;
};

// column pairs cover N <= 512; single columns (odd N or unaligned operands) N <= 256
bool skinny_applies(long N, bool aligned)
{
    return g_tuning.skinny != 0 && (N <= 256 || (N <= kSkinnyMaxN && aligned));
}

SkinnyPlan plan_skinny(DeviceCtx &c, long M, long N, bool aligned)
{
    SkinnyPlan p;
    p.pair = aligned && (N % 2 == 0);
    const long width = p.pair ? N / 2 : N;                        // column slots in a row
    p.V = 1;
    while (32L * p.V < width && p.V < 8) p.V *= 2;                // 8 slots x 32 lanes x 2 = 512 columns
    if (!p.pair && p.V == 2) p.V = 4;                             // (singles are built for V = 1, 4, 8)
    p.L = 1;
    while ((long)p.L * p.V < width) p.L *= 2;
    const long unit = (long)skinny_rows(p.V) * (kThreads / p.L);      // rows one CTA covers per step
    const long per_sm = g_tuning.grid_per_sm > 0 ? g_tuning.grid_per_sm : 4;
    const long target = (long)c.sm_count * per_sm;
    long rows = (M + target - 1) / target;
    rows = ((rows + unit - 1) / unit) * unit;
    // a few units per CTA at least: the fold of the column sums and the partial row are per CTA
    if (rows < 4 * unit) rows = 4 * unit;
    p.rows_per_cta = rows;
    p.grid = (M + rows - 1) / rows;
    return p;
}

// the join of the per-CTA column partials of a skinny pass (and its sharded exchange)
int launch_join(DeviceCtx &c, FinArgs f, cudaStream_t stream);

template <int FLAGS>
int run_skinny(DeviceCtx &c, const SkinnyPlan &p, const MvArgs &a, FinArgs f, cudaStream_t stream)
{
    SkinnyArgs s{};
    s.mv = a;
    s.fin = f;
    s.L = p.L;
    s.rows_per_cta = p.rows_per_cta;
    void (*fn)(const SkinnyArgs) = nullptr;
    if (p.pair) {
        fn = p.V == 1 ? mv_skinny_kernel<FLAGS, true, 1>
                      : (p.V == 2 ? mv_skinny_kernel<FLAGS, true, 2>
                                  : (p.V == 4 ? mv_skinny_kernel<FLAGS, true, 4> : mv_skinny_kernel<FLAGS, true, 8>));
    } else {
        fn = p.V == 1 ? mv_skinny_kernel<FLAGS, false, 1>
                      : (p.V == 4 ? mv_skinny_kernel<FLAGS, false, 4> : mv_skinny_kernel<FLAGS, false, 8>);
    }
    char what[64];
    snprintf(what, sizeof(what), "mv_skinny_kernel<%d,%d,%d>", FLAGS, p.pair ? 1 : 0, p.V);
    BTO_TRY(launch_dependent(fn, (unsigned)p.grid, s, stream, what));
    if (f.cmode == kColNone) return BTO_OK;
    f.colpart = a.colpart;
    f.M = a.M;
    f.N = a.N;
    f.strip_width = a.N;               // one "strip": every column has the same contributors
    f.units_per_strip = p.grid;        // owner(u) = u when units == CTAs
    f.total_units = p.grid;
    f.grid = p.grid;
    f.nstrips = 1;
    f.rmode = kRowNone;
    return launch_join(c, f, stream);
}

template <int FLAGS>
struct Pass {
    MvPlan plan;
    SkinnyPlan skinny;             // used instead of `plan` for narrow matrices
    size_t off_row = 0, off_row2 = 0, off_col = 0;
    long M = 0, N = 0;

    bool rowstream = false;        // whole-row streaming (rowstream_kernels.cuh), N-products only

    int prepare(DeviceCtx &c, long m, long n, bool aligned, WsLayout *lay)
    {
        M = m;
        N = n;
        // two-matrix row dots of a wide matrix: stream whole rows (7.3 vs 6.9-7.07 TB/s at n = 24576)
        // ... and of a narrow one: one launch and no partials beat the strips up to N = 2048 (graph
        // replay, profiles/r02/gesummv_rowstream_mid.log: n = 2000 -- the reference's acceptance size --
        // 15.2 -> 12.3 us, 1536 9.2 -> 8.1, 2048 13.1 -> 12.0; at 2500 / 3072 the strips win, 22.0 vs 24.6 us)
        const bool wide_or_narrow = n >= g_tuning.rowstream_min_n || (g_tuning.midsize && n <= 2048);
        rowstream = (FLAGS == (kFlagN | kFlagN2) || (FLAGS == kFlagN && g_tuning.rowstream == 2)) &&
                    aligned && g_tuning.rowstream != 0 && wide_or_narrow && m >= 4L * c.sm_count;
        if (rowstream) return BTO_OK;
        // (a full 512-column strip of a rank-2 pass is mv_tile_kernel's best case: 5.9 vs 4.9 TB/s)
        if (skinny_applies(N, aligned) && !((FLAGS & kFlagRank2) && N == kSkinnyMaxN)) {
            skinny = plan_skinny(c, M, N, aligned);
            if (FLAGS & kFlagT) off_col = lay->take((size_t)skinny.grid * N);
            return BTO_OK;
        }
        BTO_TRY(plan_mv<FLAGS>(c, M, N, aligned, &plan));
        if (FLAGS & kFlagN) off_row = lay->take((size_t)plan.nstrips * M);
        if (FLAGS & kFlagN2) off_row2 = lay->take((size_t)plan.nstrips * M);
        if ((FLAGS & kFlagT) && plan.slots > 0) off_col = lay->take((size_t)plan.slots * N);
        return BTO_OK;
    }

    // Row results go to f.rowout through f.rmode, column results to f.colout
    // through f.cmode.
    int run(DeviceCtx &c, MvArgs a, FinArgs f, cudaStream_t stream) const
    {
        if constexpr (FLAGS == (kFlagN | kFlagN2) || FLAGS == kFlagN) {
            if (rowstream) {
                RowStreamArgs r{};
                r.A = a.A; r.A2 = a.A2; r.colw = a.colw; r.fin = f; r.M = M; r.N = N;
                // One 512-thread CTA per SM is resident and every CTA does the same work, so the
                // grid runs in waves of sm_count.  4 CTAs per SM unless fewer fill the last wave much
                // better (M = 8192: 512 CTAs = 3.5 waves of 16 rows, 86 % full -> 293 CTAs of 28 rows,
                // 99 %: 157 -> 150 us).  A small gain in fullness does not pay: M = 24576 measured
                // 7.40 TB/s with 559 CTAs (94 %) and 7.25 with 439 (99 %) -- more CTAs in flight
                // keep more rows streaming.
                long rows = 0, grid = 0;
                double best = -1.0;
                for (long per_sm = 4; per_sm >= 2; --per_sm) {
                    if (g_tuning.grid_per_sm > 0 && per_sm != 4) break;
                    const long target = (long)c.sm_count * (g_tuning.grid_per_sm > 0 ? g_tuning.grid_per_sm : per_sm);
                    long rr = (M + target - 1) / target;
                    rr = ((rr + kRsRows - 1) / kRsRows) * kRsRows;
                    const long gg = (M + rr - 1) / rr;
                    const long waves = (gg + c.sm_count - 1) / c.sm_count;
                    const double eff = (double)M / ((double)waves * (double)rr * (double)c.sm_count);
                    if (eff > best + 0.08 || !g_tuning.midsize) {
                        best = eff;
                        rows = rr;
                        grid = gg;
                    }
                    if (!g_tuning.midsize) break;
                }
                r.rows_per_cta = rows;
                cudaLaunchConfig_t cfg;
                memset(&cfg, 0, sizeof(cfg));
                cfg.gridDim = dim3((unsigned)grid, 1, 1);
                cfg.blockDim = dim3(kRsThreads, 1, 1);
                cfg.stream = stream;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = g_tuning.pdl ? 1 : 0;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                CUDA_TRY(cudaLaunchKernelEx(&cfg, rowstream_kernel<(FLAGS & kFlagN2) != 0>, r));
                return check_launch((FLAGS & kFlagN2) ? "rowstream_kernel<1>" : "rowstream_kernel<0>", reinterpret_cast<const void *>(
                                                            rowstream_kernel<(FLAGS & kFlagN2) != 0>));
            }
        }
        if (skinny.grid > 0) {
            a.M = M;
            a.N = N;
            a.colpart = reinterpret_cast<double *>(c.ws + off_col);
            if (!(FLAGS & kFlagN)) f.rmode = kRowNone;
            if (!(FLAGS & kFlagT)) f.cmode = kColNone;
            return run_skinny<FLAGS>(c, skinny, a, f, stream);
        }
        fill_geometry(plan, &a, M, N);
        a.rowpart = reinterpret_cast<double *>(c.ws + off_row);
        a.rowpart2 = reinterpret_cast<double *>(c.ws + off_row2);
        a.colpart = reinterpret_cast<double *>(c.ws + off_col);
        f.rowpart = a.rowpart;
        f.rowpart2 = a.rowpart2;
        f.colpart = a.colpart;
        if (!(FLAGS & kFlagN)) f.rmode = kRowNone;
        if (!(FLAGS & kFlagT)) f.cmode = kColNone;
        if (plan.direct_fn) {
            MvDirectArgs d{};
            d.mv = a;
            d.col.out = f.colout;
            d.col.z = f.colz;
            d.col.scale = f.cscale;
            d.col.mode = f.cmode;
            d.col.vector_store = aligned16(f.colout) ? 1 : 0;
            char what[72];
            snprintf(what, sizeof(what), "mv_tile_direct_kernel<%d,%d,%d,%d>", plan.flags, plan.R, plan.V,
                     plan.minb);
            BTO_TRY(launch_dependent(plan.direct_fn, (unsigned)plan.grid, d, stream, what));
            f.cmode = kColNone;
            if (f.rmode == kRowNone) return BTO_OK;          // T-only pass: nothing left to join
            return launch_finalize(c, plan, f, M, N, stream);
        }
        BTO_TRY(launch_mv(plan, a, stream));
        return launch_finalize(c, plan, f, M, N, stream);
    }
};

// size (and bind) the workspace of the stream the sequence is enqueued on
int size_ws(DeviceCtx &c, const WsLayout &lay, cudaStream_t stream)
{
    return reserve_ws(c, stream, lay.total);
}


}  // namespace
}  // namespace bto_host
