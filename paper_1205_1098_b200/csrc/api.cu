// api.cu -- the C ABI of libbto_b200.so (declared in include/bto_b200.h).
//
// Host side of the drop-in boundary: argument checking, host/device pointer
// staging (the part of runtime.run_kernel, runtime.py:99-150, that moves
// buffers), the cached partial-sum workspace (replaces the per-call
// malloc/free of cemit.py:183-202), launch planning, and the kernel sequences
// for the ten corpus kernels.  No CPU fallback: without a device every entry
// point fails with BTO_ERR_NO_DEVICE / BTO_ERR_CUDA.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "atax_cluster.cuh"
#include "bto_b200.h"
#include "mv_kernels.cuh"
#include "prim_kernels.cuh"
#include "vec_kernels.cuh"

namespace {

using namespace bto;

// ---------------------------------------------------------------------------
// error channel

thread_local int g_err = BTO_OK;
thread_local char g_errmsg[512] = "";
std::atomic<long> g_launches{0};

int fail(int code, const char *fmt, ...)
{
    g_err = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_errmsg, sizeof(g_errmsg), fmt, ap);
    va_end(ap);
    return code;
}

#define CUDA_TRY(expr)                                                         \
    do {                                                                       \
        cudaError_t e_ = (expr);                                               \
        if (e_ != cudaSuccess)                                                 \
            return fail(BTO_ERR_CUDA, "%s failed: %s", #expr,                  \
                        cudaGetErrorString(e_));                               \
    } while (0)

#define BTO_TRY(expr)                                                          \
    do {                                                                       \
        int rc_ = (expr);                                                      \
        if (rc_ != BTO_OK) return rc_;                                         \
    } while (0)

// ---------------------------------------------------------------------------
// per-device context

struct Tuning {
    long mv_rows = 0;        // rows per unit (0 = per-kind default | 8 | 16)
    long mv_vec = 0;         // double2 per thread per row (0 = per-kind default | 1 | 2)
    long grid_per_sm = 0;    // CTAs per SM for the matrix kernels (0 = per-kind default)
    long mv_minb = 0;        // __launch_bounds__ min CTAs/SM variant (0 = default | 1 2 3 4 6)
    long vec_unroll = 2;     // independent double2 triples in flight (1 | 2 | 4)
    long vec_grid_per_sm = 0;
    long atax_fused = 1;     // 1: single-pass cluster kernel when applicable, 0: two passes
    long atax_cluster = 0;   // cluster size of the fused ATAX (0 = auto | 1 | 2 | 4 | 8 | 16)
    long atax_stages = 0;    // TMA ring depth (0 = as many as fit, at most 8)
    long atax_rows = 0;      // 0: 16 double2 per thread per panel, 1: half-height panels
    long pdl = 1;            // joins launched as programmatic dependents of their producer
    long debug = 0;          // print launch plans to stderr
    long exchange_phases = 3;    // bit 0 publish, bit 1 wait+reduce (tests emulate ranks with 1, 2)
    long host_pipeline = 1;  // overlap H2D / compute / D2H in row panels for host operands
    long host_panel_mib = 256;   // panel size of that pipeline
};

struct DeviceCtx {
    bool ready = false;
    int device = -1;
    int sm_count = 0;
    int max_threads_per_sm = 0;
    long l2_bytes = 0;
    long global_bytes = 0;
    char *ws = nullptr;            // partial sums
    size_t ws_bytes = 0;
    unsigned int *tickets = nullptr;
    char *arena = nullptr;         // device staging for host arguments
    size_t arena_bytes = 0;
    cudaStream_t stream = nullptr; // stream of the section-1 entry points
    std::map<const void *, int> occupancy;
    std::map<const void *, int> max_clusters;
    std::map<const void *, size_t> static_smem;
    // NVLink exchange fused into the join (row-sharded runtime)
    bool exch_ready = false, exch_active = false;
    int exch_rank = 0, exch_world = 1;
    long exch_capacity = 0;            // doubles per rank, both parity halves together
    double **exch_bufs = nullptr;      // device array [world] of peer-mapped buffers
    unsigned int **exch_flags = nullptr;
    unsigned int exch_epoch = 0;
    // host-pointer pipeline: copy-in and copy-out streams, reusable events
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    std::vector<cudaEvent_t> events;
};

std::mutex g_mu;
DeviceCtx g_ctx[64];
Tuning g_tuning;

int get_ctx(DeviceCtx **out)
{
    static bool have_device = false;     // guarded by g_mu (every caller holds it)
    if (!have_device) {
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) {
            return fail(BTO_ERR_NO_DEVICE, "no CUDA device: %s",
                        e == cudaSuccess ? "device count is 0" : cudaGetErrorString(e));
        }
        have_device = true;
    }
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(BTO_ERR_INVALID, "device index %d", dev);
    DeviceCtx &c = g_ctx[dev];
    if (!c.ready) {
        cudaDeviceProp prop;
        CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
        if (prop.major < 10) {
            return fail(BTO_ERR_NO_DEVICE,
                        "device %d is sm_%d%d; this library is built for sm_100a only",
                        dev, prop.major, prop.minor);
        }
        c.device = dev;
        c.sm_count = prop.multiProcessorCount;
        c.max_threads_per_sm = prop.maxThreadsPerMultiProcessor;
        c.l2_bytes = prop.l2CacheSize;
        c.global_bytes = (long)prop.totalGlobalMem;
        CUDA_TRY(cudaMalloc(&c.tickets, 64 * sizeof(unsigned int)));
        CUDA_TRY(cudaMemset(c.tickets, 0, 64 * sizeof(unsigned int)));
        c.ready = true;
    }
    *out = &c;
    return BTO_OK;
}

int grow(char **buf, size_t *have, size_t want, const char *what)
{
    if (want <= *have) return BTO_OK;
    // nothing of ours may still be running on the old buffer
    CUDA_TRY(cudaDeviceSynchronize());
    if (*buf) CUDA_TRY(cudaFree(*buf));
    *buf = nullptr;
    *have = 0;
    size_t bytes = want + want / 8 + (1u << 20);
    cudaError_t e = cudaMalloc(buf, bytes);
    if (e != cudaSuccess) {
        bytes = want;
        e = cudaMalloc(buf, bytes);
    }
    if (e != cudaSuccess) {
        return fail(BTO_ERR_ALLOC, "cannot allocate %zu bytes of %s: %s", want, what,
                    cudaGetErrorString(e));
    }
    *have = bytes;
    return BTO_OK;
}

// bump allocator over the workspace; sizes first, pointers after ensure()
struct WsLayout {
    size_t total = 0;
    size_t take(size_t doubles)
    {
        const size_t off = total;
        total += ((doubles * sizeof(double) + 255) / 256) * 256;
        return off;
    }
};

template <typename K>
int occupancy_of(DeviceCtx &c, K kernel, int *occ)
{
    const void *key = reinterpret_cast<const void *>(kernel);
    auto it = c.occupancy.find(key);
    if (it == c.occupancy.end()) {
        int n = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kThreads, 0));
        if (n < 1) n = 1;
        it = c.occupancy.emplace(key, n).first;
    }
    *occ = it->second;
    return BTO_OK;
}

int check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        return fail(BTO_ERR_CUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return BTO_OK;
}

// Launch `kernel(arg)` as a programmatic dependent of the previous kernel in the
// stream (the kernel itself calls griddepcontrol.wait before touching memory).
template <typename Arg>
int launch_dependent(void (*kernel)(const Arg), unsigned grid, const Arg &arg,
                     cudaStream_t stream, const char *what)
{
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_tuning.pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, arg));
    return check_launch(what);
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

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
        BTO_TRY(grow(&c.ws, &c.ws_bytes, lay.total, "workspace"));
        g.partials = reinterpret_cast<double *>(c.ws + off);
        g.ticket = c.tickets;
    }
    return launch_dependent(fn, (unsigned)grid, g, stream, "vec_kernel");
}

// ---------------------------------------------------------------------------
// matrix kernels

using MvKernel = void (*)(const MvArgs);

struct MvPlan {
    int R = 8, V = 1;
    bool aligned = true;
    long strip_width = 512;
    int nstrips = 1;
    long units_per_strip = 1, total_units = 1;
    long grid = 1;
    long slots = 1;        // max CTAs sharing one strip
    MvKernel fn = nullptr;
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
    if (R == 8 && V == 2) return FLAGS == kFlagN || FLAGS == (kFlagT | kFlagRank2);
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
        if constexpr (FLAGS == kFlagN || FLAGS == (kFlagT | kFlagRank2)) {
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
    if (FLAGS == (kFlagN | kFlagT)) return {8, 1, 8, 4};        // BiCGK         7.10 TB/s
    if (FLAGS == (kFlagN | kFlagN2)) return {8, 1, 4, 4};       // GESUMMV       7.04 TB/s
    if (FLAGS == (kFlagT | kFlagRank2)) return {16, 1, 2, 1};   // GEMVER pass 1 6.29 TB/s (r+w)
    if (FLAGS == kFlagT) return {32, 1, 2, 1};                  // A' y          7.17 TB/s
    return {8, 2, 8, 2};                                        // A x           7.20 TB/s
}

template <int FLAGS>
int plan_mv(DeviceCtx &c, long M, long N, bool aligned, MvPlan *p)
{
    constexpr MvDefault dflt = mv_default<FLAGS>();
    int R = g_tuning.mv_rows ? (int)g_tuning.mv_rows : dflt.rows;
    int V = g_tuning.mv_vec ? (int)g_tuning.mv_vec : dflt.vec;
    int minb = g_tuning.mv_minb ? (int)g_tuning.mv_minb : dflt.minb;
    if (!aligned || !mv_shape_ok<FLAGS>(R, V)) { R = 8; V = 1; }
    p->R = R;
    p->V = V;
    p->aligned = aligned;
    p->fn = mv_kernel_ptr<FLAGS>(R, V, aligned, minb);
    p->strip_width = (long)kThreads * 2 * V;
    p->nstrips = (int)((N + p->strip_width - 1) / p->strip_width);
    p->units_per_strip = (M + R - 1) / R;
    p->total_units = p->units_per_strip * p->nstrips;
    int occ = 1;
    BTO_TRY(occupancy_of(c, p->fn, &occ));
    long per_sm = g_tuning.grid_per_sm > 0 ? g_tuning.grid_per_sm : dflt.grid_per_sm;
    if (per_sm <= 0) per_sm = occ;
    long grid = (long)c.sm_count * per_sm;
    // small matrices: at least 4 units per CTA, so that few CTAs share a strip and
    // the join (one partial per CTA and strip) stays short
    const long by_work = (p->total_units + 3) / 4;
    if (grid > by_work) grid = by_work;
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
    return launch_dependent(p.fn, (unsigned)p.grid, a, stream, "mv_tile_kernel");
}

// Launch the join of `f` (geometry already filled in).  While a sharded
// entry point is active and the join has a column side, the cross-GPU exchange
// is fused into it (join_exchange_kernel); otherwise the plain local join runs.
int launch_join(DeviceCtx &c, FinArgs f, cudaStream_t stream)
{
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
        e.epoch = ++c.exch_epoch;
        e.buf_offset = (long)(e.epoch & 1u) * (c.exch_capacity / 2);
        e.rank = c.exch_rank;
        e.world = c.exch_world;
        e.phases = (int)g_tuning.exchange_phases;
        return launch_dependent(join_exchange_kernel, (unsigned)(kExchCtas + rb), e, stream,
                                "join_exchange_kernel");
    }
    const long cb = f.cmode != kColNone ? (f.N + kThreads - 1) / kThreads : 0;
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
template <int FLAGS>
struct Pass {
    MvPlan plan;
    size_t off_row = 0, off_row2 = 0, off_col = 0;
    long M = 0, N = 0;

    int prepare(DeviceCtx &c, long m, long n, bool aligned, WsLayout *lay)
    {
        M = m;
        N = n;
        BTO_TRY(plan_mv<FLAGS>(c, M, N, aligned, &plan));
        if (FLAGS & kFlagN) off_row = lay->take((size_t)plan.nstrips * M);
        if (FLAGS & kFlagN2) off_row2 = lay->take((size_t)plan.nstrips * M);
        if (FLAGS & kFlagT) off_col = lay->take((size_t)plan.slots * N);
        return BTO_OK;
    }

    // Row results go to f.rowout through f.rmode, column results to f.colout
    // through f.cmode.
    int run(DeviceCtx &c, MvArgs a, FinArgs f, cudaStream_t stream) const
    {
        fill_geometry(plan, &a, M, N);
        a.rowpart = reinterpret_cast<double *>(c.ws + off_row);
        a.rowpart2 = reinterpret_cast<double *>(c.ws + off_row2);
        a.colpart = reinterpret_cast<double *>(c.ws + off_col);
        BTO_TRY(launch_mv(plan, a, stream));
        f.rowpart = a.rowpart;
        f.rowpart2 = a.rowpart2;
        f.colpart = a.colpart;
        if (!(FLAGS & kFlagN)) f.rmode = kRowNone;
        if (!(FLAGS & kFlagT)) f.cmode = kColNone;
        return launch_finalize(c, plan, f, M, N, stream);
    }
};

int size_ws(DeviceCtx &c, const WsLayout &lay)
{
    return grow(&c.ws, &c.ws_bytes, lay.total, "workspace");
}

// ---------------------------------------------------------------------------
// kernel sequences (device pointers, asynchronous)

int seq_axpydot(DeviceCtx &c, const double *w, const double *v, const double *u,
                double alpha, double *z, double *beta, long M, cudaStream_t st)
{
    VecArgs g{};
    g.a = w; g.b = v; g.c = u; g.alpha = alpha; g.out = z; g.dot = beta; g.n = M;
    return launch_vec<kAxpydot>(c, g, st);
}

int seq_vadd(DeviceCtx &c, const double *w, const double *y, const double *z,
             double *x, long M, cudaStream_t st)
{
    VecArgs g{};
    g.a = w; g.b = y; g.c = z; g.out = x; g.n = M;
    return launch_vec<kVadd>(c, g, st);
}

int seq_waxpby(DeviceCtx &c, double alpha, const double *x, double beta,
               const double *y, double *w, long M, cudaStream_t st)
{
    VecArgs g{};
    g.a = x; g.b = y; g.alpha = alpha; g.beta = beta; g.out = w; g.n = M;
    return launch_vec<kWaxpby>(c, g, st);
}

int seq_bicgk(DeviceCtx &c, const double *A, const double *p, const double *r,
              double *q, double *s, long M, long N, cudaStream_t st)
{
    BTO_TRY(check_mn(M, N));
    WsLayout lay;
    Pass<kFlagN | kFlagT> pass;
    BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, A), &lay));
    BTO_TRY(size_ws(c, lay));
    MvArgs a{};
    a.A = A; a.colw = p; a.roww = r;
    FinArgs f{};
    f.cmode = kColPlain; f.colout = s;
    f.rmode = kRowPlain; f.rowout = q;
    return pass.run(c, a, f, st);
}

// ---- fused single-pass ATAX (atax_cluster.cuh) -----------------------------------

using AtaxKernel = void (*)(const AtaxArgs);

struct AtaxPlan {
    AtaxKernel fn = nullptr;     // nullptr: not applicable, use the two-pass sequence
    int C = 1, KMAX = 1, RG = 1, W = 0, S = 0;
    size_t smem = 0;
    int nclusters = 0;
};

// TR (rows per panel) is 16 / KMAX capped at 8: a panel is 16 double2 per thread.
// `small` halves it (fewer registers per tile, more panels per byte).
template <int C>
AtaxKernel atax_kernel_ptr(int kmax, bool small)
{
    switch (kmax) {
        case 1: return small ? atax_cluster_kernel<C, 1, 4> : atax_cluster_kernel<C, 1, 8>;
        case 2: return small ? atax_cluster_kernel<C, 2, 4> : atax_cluster_kernel<C, 2, 8>;
        case 4: return small ? atax_cluster_kernel<C, 4, 2> : atax_cluster_kernel<C, 4, 4>;
        case 8: return small ? atax_cluster_kernel<C, 8, 1> : atax_cluster_kernel<C, 8, 2>;
        case 16: return atax_cluster_kernel<C, 16, 1>;
    }
    return nullptr;
}

int atax_rows_of(int kmax, bool small)
{
    const int full = (16 / kmax) < kAtaxMaxRows ? (16 / kmax) : kAtaxMaxRows;
    if (!small || kmax == 16) return full;
    return kmax == 1 ? 4 : full / 2;
}

AtaxKernel atax_kernel_ptr(int c, int kmax, bool small)
{
    switch (c) {
        case 1: return atax_kernel_ptr<1>(kmax, small);
        case 2: return atax_kernel_ptr<2>(kmax, small);
        case 4: return atax_kernel_ptr<4>(kmax, small);
        case 8: return atax_kernel_ptr<8>(kmax, small);
        case 16: return atax_kernel_ptr<16>(kmax, small);
    }
    return nullptr;
}

int fill_launch_config(const AtaxPlan &p, cudaLaunchConfig_t *cfg, cudaLaunchAttribute *attr,
                       cudaStream_t stream)
{
    memset(cfg, 0, sizeof(*cfg));
    cfg->gridDim = dim3((unsigned)(p.nclusters > 0 ? p.nclusters * p.C : p.C), 1, 1);
    cfg->blockDim = dim3(kAtaxThreads, 1, 1);
    cfg->dynamicSmemBytes = p.smem;
    cfg->stream = stream;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_tuning.pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)p.C;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg->attrs = attr;
    cfg->numAttrs = p.C > 1 ? 2 : 1;
    return BTO_OK;
}

// Picks cluster size, per-thread column count, ring depth and the number of
// co-resident clusters.  Leaves p->fn == nullptr when the fused kernel does not
// apply (odd N / unaligned operands / a row too long for 16 CTAs).
int plan_atax(DeviceCtx &c, const double *A, const double *x, long M, long N, AtaxPlan *p)
{
    p->fn = nullptr;
    if (!g_tuning.atax_fused || (N % 2) || !aligned16(A) || !aligned16(x)) return BTO_OK;
    int C = (int)g_tuning.atax_cluster;
    if (C == 0) {
        // smallest cluster whose per-CTA slice fits 8 double2 per thread (4096 columns)
        C = 1;
        while (C < 16 && (N + C - 1) / C > 4096) C *= 2;
    }
    long W = (N + C - 1) / C;
    W += W & 1;
    int kmax = 1;
    while ((long)kmax * 2 * kThreads < W) kmax *= 2;
    if (kmax > 16) return BTO_OK;
    if ((long)(C - 1) * W >= N && C > 1) return BTO_OK;   // a CTA would own no column
    const bool small = g_tuning.atax_rows == 1;     // 1: half-height panels
    AtaxKernel fn = atax_kernel_ptr(C, kmax, small);
    if (!fn) return BTO_OK;
    const int rg = atax_rows_of(kmax, small);
    const size_t stage = (size_t)rg * W * sizeof(double);
    auto sm = c.static_smem.find(reinterpret_cast<const void *>(fn));
    if (sm == c.static_smem.end()) {
        cudaFuncAttributes fattr;
        CUDA_TRY(cudaFuncGetAttributes(&fattr, fn));
        sm = c.static_smem.emplace(reinterpret_cast<const void *>(fn), fattr.sharedSizeBytes).first;
    }
    // 227 KiB per CTA on sm_100, minus the kernel's static shared memory
    const size_t budget = ((227 * 1024 - sm->second) / 1024) * 1024;
    int S = (int)(budget / stage);
    if (S > 8) S = 8;
    if (g_tuning.atax_stages > 0 && g_tuning.atax_stages < S) S = (int)g_tuning.atax_stages;
    if (S < 2) return BTO_OK;
    p->C = C;
    p->KMAX = kmax;
    p->RG = rg;
    p->W = (int)W;
    p->S = S;
    p->smem = stage * S;
    auto it = c.max_clusters.find(reinterpret_cast<const void *>(fn));
    if (it == c.max_clusters.end()) {
        CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)budget));
        if (C > 8) {
            CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
        int n = 0;
        if (C > 1) {
            AtaxPlan probe = *p;
            probe.nclusters = c.sm_count / C;
            probe.smem = budget;
            cudaLaunchConfig_t cfg;
            cudaLaunchAttribute attr[2];
            fill_launch_config(probe, &cfg, attr, nullptr);
            CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, fn, &cfg));
        } else {
            n = c.sm_count;
        }
        if (n < 1) n = 1;
        it = c.max_clusters.emplace(reinterpret_cast<const void *>(fn), n).first;
    }
    long ncl = it->second;
    const long groups = (M + rg - 1) / rg;
    if (ncl > groups) ncl = groups;
    p->nclusters = (int)ncl;
    p->fn = fn;
    return BTO_OK;
}

int seq_atax_fused(DeviceCtx &c, const AtaxPlan &p, const double *A, const double *x,
                   double *y, long M, long N, bool scaled, double beta, cudaStream_t st)
{
    WsLayout lay;
    const size_t off = lay.take((size_t)p.nclusters * N);
    BTO_TRY(size_ws(c, lay));
    AtaxArgs a{};
    a.A = A; a.x = x; a.M = M; a.N = N;
    a.ypart = reinterpret_cast<double *>(c.ws + off);
    a.W = p.W; a.stages = p.S; a.nclusters = p.nclusters;
    if (g_tuning.debug) {
        fprintf(stderr, "[bto] atax fused: C=%d KMAX=%d rows=%d W=%d stages=%d smem=%zu clusters=%d\n",
                p.C, p.KMAX, p.RG, p.W, p.S, p.smem, p.nclusters);
    }
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[2];
    fill_launch_config(p, &cfg, attr, st);
    CUDA_TRY(cudaLaunchKernelEx(&cfg, p.fn, a));
    BTO_TRY(check_launch("atax_cluster_kernel"));
    // join the per-cluster partials in ascending cluster order
    FinArgs f{};
    f.colpart = a.ypart;
    f.colout = y;
    f.cmode = scaled ? kColScale : kColPlain;
    f.cscale = beta;
    f.N = N;
    f.M = M;
    f.strip_width = N;                 // one "strip": every column has the same contributors
    f.units_per_strip = p.nclusters;   // owner(0) = 0, owner(U-1) = G-1 when U == G
    f.total_units = p.nclusters;
    f.grid = p.nclusters;
    f.rmode = kRowNone;
    return launch_join(c, f, st);
}

// y = [beta *] A'(A x): pass 1 contracts t = A x into a workspace vector (it
// never reaches the caller), pass 2 streams A again for A' t.
int seq_atax(DeviceCtx &c, const double *A, const double *x, double *y, long M,
             long N, bool scaled, double beta, cudaStream_t st)
{
    BTO_TRY(check_mn(M, N));
    AtaxPlan fused;
    BTO_TRY(plan_atax(c, A, x, M, N, &fused));
    if (fused.fn) return seq_atax_fused(c, fused, A, x, y, M, N, scaled, beta, st);
    const bool al = mat_aligned(N, A);
    WsLayout lay;
    const size_t off_t = lay.take((size_t)M);
    Pass<kFlagN> dots;
    Pass<kFlagT> sums;
    BTO_TRY(dots.prepare(c, M, N, al, &lay));
    BTO_TRY(sums.prepare(c, M, N, al, &lay));
    BTO_TRY(size_ws(c, lay));
    double *t = reinterpret_cast<double *>(c.ws + off_t);
    {
        MvArgs a{};
        a.A = A; a.colw = x;
        FinArgs f{};
        f.rmode = kRowPlain; f.rowout = t;
        BTO_TRY(dots.run(c, a, f, st));
    }
    MvArgs a{};
    a.A = A; a.roww = t;
    FinArgs f{};
    f.cmode = scaled ? kColScale : kColPlain; f.cscale = beta; f.colout = y;
    return sums.run(c, a, f, st);
}

int seq_gesummv(DeviceCtx &c, double alpha, double beta, const double *A,
                const double *B, const double *x, double *y, long M, long N,
                cudaStream_t st)
{
    BTO_TRY(check_mn(M, N));
    WsLayout lay;
    Pass<kFlagN | kFlagN2> pass;
    BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, A, B), &lay));
    BTO_TRY(size_ws(c, lay));
    MvArgs a{};
    a.A = A; a.A2 = B; a.colw = x;
    FinArgs f{};
    f.rmode = kRowGesummv; f.ralpha = alpha; f.rbeta = beta; f.rowout = y;
    return pass.run(c, a, f, st);
}

int seq_dgemv(DeviceCtx &c, double alpha, const double *A, const double *x,
              double beta, const double *y, double *z, long M, long N,
              cudaStream_t st)
{
    BTO_TRY(check_mn(M, N));
    WsLayout lay;
    Pass<kFlagN> pass;
    BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, A), &lay));
    BTO_TRY(size_ws(c, lay));
    MvArgs a{};
    a.A = A; a.colw = x;
    FinArgs f{};
    f.rmode = kRowDgemv; f.ralpha = alpha; f.rbeta = beta; f.rowy = y; f.rowout = z;
    return pass.run(c, a, f, st);
}

// GEMVER / DGEMVT pass 1: colsum = B' y with B = A + u1 v1' + u2 v2' stored
// (u1 == nullptr: DGEMVT, colsum = A' y, nothing stored).  f.cmode decides
// what lands in f.colout (the sum itself, or x = sum*beta + z).
int seq_pass1(DeviceCtx &c, const double *A, const double *u1, const double *v1,
              const double *u2, const double *v2, const double *y, double *B,
              FinArgs f, long M, long N, cudaStream_t st)
{
    WsLayout lay;
    MvArgs a{};
    a.A = A; a.roww = y;
    if (u1 == nullptr) {
        Pass<kFlagT> pass;
        BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, A), &lay));
        BTO_TRY(size_ws(c, lay));
        return pass.run(c, a, f, st);
    }
    a.u1 = u1; a.v1 = v1; a.u2 = u2; a.v2 = v2; a.Bout = B;
    Pass<kFlagT | kFlagRank2> pass;
    BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, A, B), &lay));
    BTO_TRY(size_ws(c, lay));
    return pass.run(c, a, f, st);
}

int seq_pass2(DeviceCtx &c, const double *B, const double *x, double alpha,
              double *w, long M, long N, cudaStream_t st)
{
    WsLayout lay;
    Pass<kFlagN> pass;
    BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, B), &lay));
    BTO_TRY(size_ws(c, lay));
    MvArgs a{};
    a.A = B; a.colw = x;
    FinArgs f{};
    f.rmode = kRowScale; f.ralpha = alpha; f.rowout = w;
    return pass.run(c, a, f, st);
}

// The two passes run back to back on one stream and no workspace pointer
// outlives its pass (x and colsum are caller buffers), so each pass may size
// the workspace for itself.
int seq_gemver(DeviceCtx &c, const double *A, const double *u1, const double *v1,
               const double *u2, const double *v2, double alpha, double beta,
               const double *y, const double *z, double *B, double *x, double *w,
               long M, long N, cudaStream_t st)
{
    BTO_TRY(check_mn(M, N));
    if (u1 == nullptr || v1 == nullptr || u2 == nullptr || v2 == nullptr) {
        return fail(BTO_ERR_INVALID, "gemver: null rank-2 vector");
    }
    FinArgs f{};
    f.cmode = kColAxpz; f.cscale = beta; f.colz = z; f.colout = x;
    BTO_TRY(seq_pass1(c, A, u1, v1, u2, v2, y, B, f, M, N, st));
    return seq_pass2(c, B, x, alpha, w, M, N, st);
}

int seq_dgemvt(DeviceCtx &c, double alpha, double beta, const double *A,
               const double *y, const double *z, double *x, double *w, long M,
               long N, cudaStream_t st)
{
    BTO_TRY(check_mn(M, N));
    FinArgs f{};
    f.cmode = kColAxpz; f.cscale = beta; f.colz = z; f.colout = x;
    BTO_TRY(seq_pass1(c, A, nullptr, nullptr, nullptr, nullptr, y, nullptr, f, M, N, st));
    return seq_pass2(c, A, x, alpha, w, M, N, st);
}

// ---------------------------------------------------------------------------
// host/device argument staging for the section-1 entry points

bool host_memory(const void *p)
{
    if (!p) return false;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return !(attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged);
}

class Call {
public:
    Call() : lock_(g_mu)
    {
        g_err = BTO_OK;
        g_errmsg[0] = 0;
        rc_ = get_ctx(&ctx_);
    }
    bool ok() const { return rc_ == BTO_OK; }
    DeviceCtx &ctx() { return *ctx_; }
    cudaStream_t stream() const { return ctx_->stream; }
    void status(int rc) { if (rc_ == BTO_OK) rc_ = rc; }

    void in(const double **slot, long count) { add(const_cast<double **>(slot), count, false); }
    void out(double **slot, long count) { add(slot, count, true); }
    // Streamed operands: device space is reserved for them, but the caller moves
    // the data itself in panels (see gemver_streamed / axpydot_streamed).
    void in_streamed(const double **slot, long count)
    {
        add(const_cast<double **>(slot), count, false);
        args_.back().streamed = true;
    }
    void out_streamed(double **slot, long count)
    {
        add(slot, count, true);
        args_.back().streamed = true;
    }
    // device scratch that lives as long as the call (host-operand calls only)
    void scratch(double **slot, long count)
    {
        *slot = nullptr;
        add(slot, count, true);
        args_.back().scratch = true;
    }
    // the caller's host pointer behind a staged argument (nullptr: it was device memory)
    double *host_of(const double *dev) const
    {
        for (const Arg &a : args_) {
            if (a.on_host && *a.slot == dev) return a.host;
        }
        return nullptr;
    }
    bool any_host() const { return any_host_; }

    // classify, allocate staging, copy inputs host -> device
    void prepare()
    {
        if (!ok()) return;
        size_t need = 0;
        for (Arg &a : args_) {
            if (a.scratch) {
                a.on_host = true;
                a.offset = need;
                need += ((size_t)a.count * sizeof(double) + 255) / 256 * 256;
                continue;
            }
            if (*a.slot == nullptr || a.count < 1) {
                status(fail(BTO_ERR_INVALID, "null pointer or empty array argument"));
                return;
            }
            cudaPointerAttributes attr;
            cudaError_t e = cudaPointerGetAttributes(&attr, *a.slot);
            if (e != cudaSuccess) {
                cudaGetLastError();
                attr.type = cudaMemoryTypeUnregistered;
            }
            a.on_host = !(attr.type == cudaMemoryTypeDevice ||
                          attr.type == cudaMemoryTypeManaged);
            if (a.on_host) {
                a.offset = need;
                need += ((size_t)a.count * sizeof(double) + 255) / 256 * 256;
                any_host_ = true;
            }
        }
        if (!any_host_) return;
        status(grow(&ctx_->arena, &ctx_->arena_bytes, need, "staging arena"));
        if (!ok()) return;
        for (Arg &a : args_) {
            if (!a.on_host) continue;
            a.host = *a.slot;
            *a.slot = reinterpret_cast<double *>(ctx_->arena + a.offset);
            if (!a.is_out && !a.streamed) {
                cudaError_t e = cudaMemcpyAsync(*a.slot, a.host, (size_t)a.count * sizeof(double),
                                                cudaMemcpyHostToDevice, stream());
                if (e != cudaSuccess) {
                    status(fail(BTO_ERR_CUDA, "host->device copy failed: %s",
                                cudaGetErrorString(e)));
                    return;
                }
            }
        }
    }

    // copy outputs device -> host and wait (only when something was staged)
    void finish()
    {
        if (!any_host_) return;
        if (ok()) {
            for (Arg &a : args_) {
                if (!a.on_host || !a.is_out || a.streamed || a.scratch) continue;
                cudaError_t e = cudaMemcpyAsync(a.host, *a.slot, (size_t)a.count * sizeof(double),
                                                cudaMemcpyDeviceToHost, stream());
                if (e != cudaSuccess) {
                    status(fail(BTO_ERR_CUDA, "device->host copy failed: %s",
                                cudaGetErrorString(e)));
                    break;
                }
            }
        }
        cudaError_t e = cudaStreamSynchronize(stream());
        if (e != cudaSuccess && ok()) {
            status(fail(BTO_ERR_CUDA, "kernel sequence failed: %s", cudaGetErrorString(e)));
        }
    }

private:
    struct Arg {
        double **slot;
        long count;
        bool is_out;
        bool on_host = false;
        bool streamed = false;
        bool scratch = false;
        size_t offset = 0;
        double *host = nullptr;
    };
    void add(double **slot, long count, bool is_out)
    {
        Arg a;
        a.slot = slot;
        a.count = count;
        a.is_out = is_out;
        args_.push_back(a);
    }
    std::lock_guard<std::mutex> lock_;
    DeviceCtx *ctx_ = nullptr;
    int rc_ = BTO_OK;
    bool any_host_ = false;
    std::vector<Arg> args_;
};

// ---------------------------------------------------------------------------
// host operands: panel pipeline over three streams
//
// PCIe is full duplex and the kernels are ~50x faster than the link, so for
// the sequences with matrix- or vector-sized OUTPUTS the copy-out of panel p
// overlaps the copy-in of panel p+1.. and the total is max(in, out) instead of
// in + out.  Row panels are the reference's row blocks once more
// (cemit.py:195-196); per-panel partial sums are joined in ascending order.

int pipe_setup(DeviceCtx &c, size_t nevents)
{
    if (!c.copy_in) CUDA_TRY(cudaStreamCreateWithFlags(&c.copy_in, cudaStreamNonBlocking));
    if (!c.copy_out) CUDA_TRY(cudaStreamCreateWithFlags(&c.copy_out, cudaStreamNonBlocking));
    while (c.events.size() < nevents) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c.events.push_back(e);
    }
    return BTO_OK;
}

long panel_count(double bytes_total)
{
    const double panel = (double)g_tuning.host_panel_mib * 1048576.0;
    long p = (long)(bytes_total / panel + 0.999);
    if (p < 2) p = 2;
    if (p > 64) p = 64;
    return p;
}

// ascending join of `count` length-n partial vectors (+ optional x = sum*beta + z)
int join_partials(const double *parts, long count, long n, int cmode, double scale,
                  const double *z, double *out, cudaStream_t st)
{
    FinArgs f{};
    f.colpart = parts;
    f.colout = out;
    f.cmode = cmode;
    f.cscale = scale;
    f.colz = z;
    f.N = n;
    f.strip_width = n;
    f.units_per_strip = count;
    f.total_units = count;
    f.grid = count;
    f.rmode = kRowNone;
    f.col_blocks = (int)((n + kThreads - 1) / kThreads);
    return launch_dependent(finalize_kernel, (unsigned)f.col_blocks, f, st, "finalize_kernel");
}

// GEMVER with A and B in host memory.  d* are device copies (dA, dB reserved but
// not filled), h* the caller's buffers; vectors are already on the device.
int gemver_streamed(DeviceCtx &c, cudaStream_t main, const double *hA, double *dA,
                    const double *u1, const double *v1, const double *u2, const double *v2,
                    double alpha, double beta, const double *y, const double *z, double *hB,
                    double *dB, double *x, double *w, double *panel_sums, long P, long M, long N)
{
    BTO_TRY(pipe_setup(c, (size_t)(2 * P + 2)));
    cudaEvent_t ready = c.events[2 * P], done = c.events[2 * P + 1];
    // the copy streams start after whatever the main stream has queued (vector H2D)
    CUDA_TRY(cudaEventRecord(ready, main));
    CUDA_TRY(cudaStreamWaitEvent(c.copy_in, ready, 0));
    CUDA_TRY(cudaStreamWaitEvent(c.copy_out, ready, 0));
    for (long p = 0; p < P; ++p) {
        const long r0 = (M * p) / P, r1 = (M * (p + 1)) / P;
        if (r1 == r0) {
            CUDA_TRY(cudaMemsetAsync(panel_sums + p * N, 0, (size_t)N * sizeof(double), main));
            continue;
        }
        const size_t off = (size_t)r0 * N, bytes = (size_t)(r1 - r0) * N * sizeof(double);
        CUDA_TRY(cudaMemcpyAsync(dA + off, hA + off, bytes, cudaMemcpyHostToDevice, c.copy_in));
        CUDA_TRY(cudaEventRecord(c.events[2 * p], c.copy_in));
        CUDA_TRY(cudaStreamWaitEvent(main, c.events[2 * p], 0));
        FinArgs f{};
        f.cmode = kColPlain;
        f.colout = panel_sums + p * N;
        BTO_TRY(seq_pass1(c, dA + off, u1 + r0, v1, u2 + r0, v2, y + r0, dB + off, f, r1 - r0, N,
                          main));
        CUDA_TRY(cudaEventRecord(c.events[2 * p + 1], main));
        CUDA_TRY(cudaStreamWaitEvent(c.copy_out, c.events[2 * p + 1], 0));
        CUDA_TRY(cudaMemcpyAsync(hB + off, dB + off, bytes, cudaMemcpyDeviceToHost, c.copy_out));
    }
    BTO_TRY(join_partials(panel_sums, P, N, kColAxpz, beta, z, x, main));
    BTO_TRY(seq_pass2(c, dB, x, alpha, w, M, N, main));
    // the caller's finish() copies x and w on `main`; B must have landed too
    CUDA_TRY(cudaEventRecord(done, c.copy_out));
    CUDA_TRY(cudaStreamWaitEvent(main, done, 0));
    return BTO_OK;
}

// AXPYDOT with all four vectors in host memory: chunks in, z chunks out.
int axpydot_streamed(DeviceCtx &c, cudaStream_t main, const double *hw, double *dw,
                     const double *hv, double *dv, const double *hu, double *du, double alpha,
                     double *hz, double *dz, double *dbeta, double *chunk_dots, long P, long M)
{
    BTO_TRY(pipe_setup(c, (size_t)(2 * P + 2)));
    cudaEvent_t ready = c.events[2 * P], done = c.events[2 * P + 1];
    CUDA_TRY(cudaEventRecord(ready, main));
    CUDA_TRY(cudaStreamWaitEvent(c.copy_in, ready, 0));
    CUDA_TRY(cudaStreamWaitEvent(c.copy_out, ready, 0));
    for (long p = 0; p < P; ++p) {
        // even chunk starts keep the double2 path aligned
        long k0 = ((M * p) / P) & ~1L, k1 = p + 1 == P ? M : (((M * (p + 1)) / P) & ~1L);
        if (k1 == k0) {
            CUDA_TRY(cudaMemsetAsync(chunk_dots + p, 0, sizeof(double), main));
            continue;
        }
        const size_t bytes = (size_t)(k1 - k0) * sizeof(double);
        CUDA_TRY(cudaMemcpyAsync(dw + k0, hw + k0, bytes, cudaMemcpyHostToDevice, c.copy_in));
        CUDA_TRY(cudaMemcpyAsync(dv + k0, hv + k0, bytes, cudaMemcpyHostToDevice, c.copy_in));
        CUDA_TRY(cudaMemcpyAsync(du + k0, hu + k0, bytes, cudaMemcpyHostToDevice, c.copy_in));
        CUDA_TRY(cudaEventRecord(c.events[2 * p], c.copy_in));
        CUDA_TRY(cudaStreamWaitEvent(main, c.events[2 * p], 0));
        BTO_TRY(seq_axpydot(c, dw + k0, dv + k0, du + k0, alpha, dz + k0, chunk_dots + p, k1 - k0,
                            main));
        CUDA_TRY(cudaEventRecord(c.events[2 * p + 1], main));
        CUDA_TRY(cudaStreamWaitEvent(c.copy_out, c.events[2 * p + 1], 0));
        CUDA_TRY(cudaMemcpyAsync(hz + k0, dz + k0, bytes, cudaMemcpyDeviceToHost, c.copy_out));
    }
    BTO_TRY(join_partials(chunk_dots, P, 1, kColPlain, 0.0, nullptr, dbeta, main));
    CUDA_TRY(cudaEventRecord(done, c.copy_out));
    CUDA_TRY(cudaStreamWaitEvent(main, done, 0));
    return BTO_OK;
}

// async entry points share this prologue
struct AsyncCall {
    AsyncCall() : lock(g_mu)
    {
        g_err = BTO_OK;
        g_errmsg[0] = 0;
        rc = get_ctx(&ctx);
    }
    std::lock_guard<std::mutex> lock;
    DeviceCtx *ctx = nullptr;
    int rc = BTO_OK;
};

bool extents_ok(Call &c, long M, long N)
{
    if (!c.ok()) return false;
    if (M < 1 || N < 1) {
        c.status(fail(BTO_ERR_INVALID, "extents M=%ld N=%ld must be >= 1", M, N));
        return false;
    }
    return true;
}

}  // namespace

// ===========================================================================
// exported symbols

extern "C" {

int bto_last_error(void) { return g_err; }
const char *bto_last_error_string(void) { return g_errmsg; }
void bto_clear_error(void) { g_err = BTO_OK; g_errmsg[0] = 0; }
int bto_abi_version(void) { return BTO_B200_ABI_VERSION; }
long bto_kernel_launches(void) { return g_launches.load(); }

// ---- section 1: the reference's signatures ---------------------------------

void axpydot(const double *w, const double *v, const double *u, double alpha,
             double *z, double *beta, long M)
{
    Call c;
    if (!extents_ok(c, M, 1)) return;
    const long P = panel_count(8.0 * (double)M);
    const bool stream_it = g_tuning.host_pipeline && M >= (1L << 22) && host_memory(w) &&
                           host_memory(v) && host_memory(u) && host_memory(z);
    if (stream_it) {
        double *dots = nullptr;
        c.in_streamed(&w, M); c.in_streamed(&v, M); c.in_streamed(&u, M);
        c.out_streamed(&z, M); c.out(&beta, 1); c.scratch(&dots, P);
        c.prepare();
        if (c.ok()) {
            c.status(axpydot_streamed(c.ctx(), c.stream(), c.host_of(w), const_cast<double *>(w),
                                      c.host_of(v), const_cast<double *>(v), c.host_of(u),
                                      const_cast<double *>(u), alpha, c.host_of(z), z, beta, dots,
                                      P, M));
        }
        c.finish();
        return;
    }
    c.in(&w, M); c.in(&v, M); c.in(&u, M); c.out(&z, M); c.out(&beta, 1);
    c.prepare();
    if (c.ok()) c.status(seq_axpydot(c.ctx(), w, v, u, alpha, z, beta, M, c.stream()));
    c.finish();
}

void vadd(const double *w, const double *y, const double *z, double *x, long M)
{
    Call c;
    if (!extents_ok(c, M, 1)) return;
    c.in(&w, M); c.in(&y, M); c.in(&z, M); c.out(&x, M);
    c.prepare();
    if (c.ok()) c.status(seq_vadd(c.ctx(), w, y, z, x, M, c.stream()));
    c.finish();
}

void waxpby(double alpha, const double *x, double beta, const double *y,
            double *w, long M)
{
    Call c;
    if (!extents_ok(c, M, 1)) return;
    c.in(&x, M); c.in(&y, M); c.out(&w, M);
    c.prepare();
    if (c.ok()) c.status(seq_waxpby(c.ctx(), alpha, x, beta, y, w, M, c.stream()));
    c.finish();
}

void bicgk(const double *A, const double *p, const double *r, double *q,
           double *s, long M, long N)
{
    Call c;
    if (!extents_ok(c, M, N)) return;
    c.in(&A, M * N); c.in(&p, N); c.in(&r, M); c.out(&q, M); c.out(&s, N);
    c.prepare();
    if (c.ok()) c.status(seq_bicgk(c.ctx(), A, p, r, q, s, M, N, c.stream()));
    c.finish();
}

void atax(const double *A, const double *x, double *y, long M, long N)
{
    Call c;
    if (!extents_ok(c, M, N)) return;
    c.in(&A, M * N); c.in(&x, N); c.out(&y, N);
    c.prepare();
    if (c.ok()) c.status(seq_atax(c.ctx(), A, x, y, M, N, false, 1.0, c.stream()));
    c.finish();
}

void batax(const double *x, double beta, const double *A, double *y, long M, long N)
{
    Call c;
    if (!extents_ok(c, M, N)) return;
    c.in(&x, N); c.in(&A, M * N); c.out(&y, N);
    c.prepare();
    if (c.ok()) c.status(seq_atax(c.ctx(), A, x, y, M, N, true, beta, c.stream()));
    c.finish();
}

void gesummv(double alpha, double beta, const double *A, const double *B,
             const double *x, double *y, long M, long N)
{
    Call c;
    if (!extents_ok(c, M, N)) return;
    c.in(&A, M * N); c.in(&B, M * N); c.in(&x, N); c.out(&y, M);
    c.prepare();
    if (c.ok()) c.status(seq_gesummv(c.ctx(), alpha, beta, A, B, x, y, M, N, c.stream()));
    c.finish();
}

void dgemv(double alpha, const double *A, const double *x, double beta,
           const double *y, double *z, long M, long N)
{
    Call c;
    if (!extents_ok(c, M, N)) return;
    c.in(&A, M * N); c.in(&x, N); c.in(&y, M); c.out(&z, M);
    c.prepare();
    if (c.ok()) c.status(seq_dgemv(c.ctx(), alpha, A, x, beta, y, z, M, N, c.stream()));
    c.finish();
}

void gemver(const double *A, const double *u1, const double *v1, const double *u2,
            const double *v2, double alpha, double beta, const double *y,
            const double *z, double *B, double *x, double *w, long M, long N)
{
    Call c;
    if (!extents_ok(c, M, N)) return;
    if (g_tuning.host_pipeline && (double)M * (double)N >= (double)(1L << 22) && M >= 2 &&
        host_memory(A) && host_memory(B) && u1 && v1 && u2 && v2) {
        const long P = panel_count(8.0 * (double)M * (double)N) < M
                           ? panel_count(8.0 * (double)M * (double)N) : M;
        double *sums = nullptr;
        c.in(&u1, M); c.in(&v1, N); c.in(&u2, M); c.in(&v2, N); c.in(&y, M); c.in(&z, N);
        c.in_streamed(&A, M * N); c.out_streamed(&B, M * N); c.out(&x, N); c.out(&w, M);
        c.scratch(&sums, P * N);
        c.prepare();
        if (c.ok()) {
            c.status(gemver_streamed(c.ctx(), c.stream(), c.host_of(A), const_cast<double *>(A),
                                     u1, v1, u2, v2, alpha, beta, y, z, c.host_of(B), B, x, w,
                                     sums, P, M, N));
        }
        c.finish();
        return;
    }
    c.in(&A, M * N); c.in(&u1, M); c.in(&v1, N); c.in(&u2, M); c.in(&v2, N);
    c.in(&y, M); c.in(&z, N); c.out(&B, M * N); c.out(&x, N); c.out(&w, M);
    c.prepare();
    if (c.ok()) {
        c.status(seq_gemver(c.ctx(), A, u1, v1, u2, v2, alpha, beta, y, z, B, x, w,
                            M, N, c.stream()));
    }
    c.finish();
}

void dgemvt(double alpha, double beta, const double *A, const double *y,
            const double *z, double *x, double *w, long M, long N)
{
    Call c;
    if (!extents_ok(c, M, N)) return;
    c.in(&A, M * N); c.in(&y, M); c.in(&z, N); c.out(&x, N); c.out(&w, M);
    c.prepare();
    if (c.ok()) c.status(seq_dgemvt(c.ctx(), alpha, beta, A, y, z, x, w, M, N, c.stream()));
    c.finish();
}

// ---- section 2: asynchronous, device pointers --------------------------------

#define ASYNC_PROLOGUE()                                                        \
    AsyncCall ac;                                                               \
    if (ac.rc != BTO_OK) return ac.rc;                                          \
    cudaStream_t st = static_cast<cudaStream_t>(stream)

int bto_axpydot_async(const double *w, const double *v, const double *u,
                      double alpha, double *z, double *beta, long M,
                      bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_axpydot(*ac.ctx, w, v, u, alpha, z, beta, M, st);
}

int bto_vadd_async(const double *w, const double *y, const double *z, double *x,
                   long M, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_vadd(*ac.ctx, w, y, z, x, M, st);
}

int bto_waxpby_async(double alpha, const double *x, double beta, const double *y,
                     double *w, long M, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_waxpby(*ac.ctx, alpha, x, beta, y, w, M, st);
}

int bto_bicgk_async(const double *A, const double *p, const double *r, double *q,
                    double *s, long M, long N, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_bicgk(*ac.ctx, A, p, r, q, s, M, N, st);
}

int bto_atax_async(const double *A, const double *x, double *y, long M, long N,
                   bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_atax(*ac.ctx, A, x, y, M, N, false, 1.0, st);
}

int bto_batax_async(const double *x, double beta, const double *A, double *y,
                    long M, long N, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_atax(*ac.ctx, A, x, y, M, N, true, beta, st);
}

int bto_gesummv_async(double alpha, double beta, const double *A, const double *B,
                      const double *x, double *y, long M, long N,
                      bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_gesummv(*ac.ctx, alpha, beta, A, B, x, y, M, N, st);
}

int bto_dgemv_async(double alpha, const double *A, const double *x, double beta,
                    const double *y, double *z, long M, long N, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_dgemv(*ac.ctx, alpha, A, x, beta, y, z, M, N, st);
}

int bto_gemver_async(const double *A, const double *u1, const double *v1,
                     const double *u2, const double *v2, double alpha, double beta,
                     const double *y, const double *z, double *B, double *x,
                     double *w, long M, long N, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_gemver(*ac.ctx, A, u1, v1, u2, v2, alpha, beta, y, z, B, x, w, M, N, st);
}

int bto_dgemvt_async(double alpha, double beta, const double *A, const double *y,
                     const double *z, double *x, double *w, long M, long N,
                     bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    return seq_dgemvt(*ac.ctx, alpha, beta, A, y, z, x, w, M, N, st);
}

// ---- section 3: row-sharded pieces ---------------------------------------------

int bto_gemver_pass1_async(const double *A, const double *u1, const double *v1,
                           const double *u2, const double *v2, const double *y,
                           double *B, double *colsum, long M, long N,
                           bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    BTO_TRY(check_mn(M, N));
    FinArgs f{};
    f.cmode = kColPlain; f.colout = colsum;
    return seq_pass1(*ac.ctx, A, u1, v1, u2, v2, y, B, f, M, N, st);
}

int bto_gemver_xupdate_async(const double *colsum, double beta, const double *z,
                             double *x, long N, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    if (N < 1) return fail(BTO_ERR_INVALID, "extent N=%ld must be >= 1", N);
    axpz_kernel<<<(unsigned)((N + kThreads - 1) / kThreads), kThreads, 0, st>>>(
        colsum, beta, z, x, N);
    return check_launch("axpz_kernel");
}

int bto_gemver_pass2_async(const double *B, const double *x, double alpha,
                           double *w, long M, long N, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    BTO_TRY(check_mn(M, N));
    return seq_pass2(*ac.ctx, B, x, alpha, w, M, N, st);
}

// ---- section 5: exchange fused into the join (NVLink peer memory) -----------------

int bto_exchange_init(int rank, int world, void *const *exch_ptrs, void *const *flag_ptrs,
                      long capacity_doubles, unsigned int epoch0)
{
    AsyncCall ac;
    if (ac.rc != BTO_OK) return ac.rc;
    DeviceCtx &c = *ac.ctx;
    if (world < 1 || world > 64 || rank < 0 || rank >= world || !exch_ptrs || !flag_ptrs ||
        capacity_doubles < 2) {
        return fail(BTO_ERR_INVALID, "exchange: bad rank/world/pointers/capacity");
    }
    for (int p = 0; p < world; ++p) {
        if (!exch_ptrs[p] || !flag_ptrs[p]) return fail(BTO_ERR_INVALID, "exchange: null peer pointer");
    }
    CUDA_TRY(cudaDeviceSynchronize());
    if (!c.exch_bufs) {
        CUDA_TRY(cudaMalloc(&c.exch_bufs, 64 * sizeof(double *)));
        CUDA_TRY(cudaMalloc(&c.exch_flags, 64 * sizeof(unsigned int *)));
    }
    CUDA_TRY(cudaMemcpy(c.exch_bufs, exch_ptrs, (size_t)world * sizeof(void *), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c.exch_flags, flag_ptrs, (size_t)world * sizeof(void *), cudaMemcpyHostToDevice));
    c.exch_rank = rank;
    c.exch_world = world;
    c.exch_capacity = (capacity_doubles / 2) * 2;
    c.exch_epoch = epoch0;
    c.exch_ready = true;
    return BTO_OK;
}

int bto_exchange_shutdown(void)
{
    AsyncCall ac;
    if (ac.rc != BTO_OK) return ac.rc;
    CUDA_TRY(cudaDeviceSynchronize());
    ac.ctx->exch_ready = false;
    return BTO_OK;
}

int bto_exchange_flag_bytes(int world) { return world * kExchCtas * (int)sizeof(unsigned int); }

namespace {
// marks the sequence as sharded for the joins it launches
struct ExchangeScope {
    explicit ExchangeScope(DeviceCtx &c) : ctx(c)
    {
        // a reduce-only call (tests) re-uses the epoch of the publish it pairs with
        if (!(g_tuning.exchange_phases & 1)) --ctx.exch_epoch;
        ctx.exch_active = true;
    }
    ~ExchangeScope() { ctx.exch_active = false; }
    DeviceCtx &ctx;
};
}  // namespace

#define SHARDED_PROLOGUE()                                                      \
    ASYNC_PROLOGUE();                                                           \
    if (!ac.ctx->exch_ready) return fail(BTO_ERR_INVALID, "bto_exchange_init has not been called"); \
    ExchangeScope scope(*ac.ctx)

int bto_axpydot_sharded_async(const double *w, const double *v, const double *u, double alpha,
                              double *z, double *beta, long M, bto_stream_t stream)
{
    SHARDED_PROLOGUE();
    DeviceCtx &c = *ac.ctx;
    if (M < 1) return fail(BTO_ERR_INVALID, "extent M=%ld must be >= 1", M);
    // local dot into a workspace scalar (kept clear of the kernel's own partials)
    WsLayout lay;
    lay.take((size_t)c.sm_count * 64);
    const size_t off = lay.take(1);
    BTO_TRY(size_ws(c, lay));
    double *local = reinterpret_cast<double *>(c.ws + off);
    c.exch_active = false;
    int rc = seq_axpydot(c, w, v, u, alpha, z, local, M, st);
    c.exch_active = true;
    BTO_TRY(rc);
    FinArgs f{};
    f.colpart = local;
    f.colout = beta;
    f.cmode = kColPlain;
    f.N = 1;
    f.M = 1;
    f.strip_width = 1;
    f.units_per_strip = 1;
    f.total_units = 1;
    f.grid = 1;
    f.rmode = kRowNone;
    return launch_join(c, f, st);
}

int bto_bicgk_sharded_async(const double *A, const double *p, const double *r, double *q,
                            double *s, long M, long N, bto_stream_t stream)
{
    SHARDED_PROLOGUE();
    return seq_bicgk(*ac.ctx, A, p, r, q, s, M, N, st);
}

int bto_atax_sharded_async(const double *A, const double *x, double *y, long M, long N,
                           bto_stream_t stream)
{
    SHARDED_PROLOGUE();
    return seq_atax(*ac.ctx, A, x, y, M, N, false, 1.0, st);
}

int bto_gemver_sharded_async(const double *A, const double *u1, const double *v1,
                             const double *u2, const double *v2, double alpha, double beta,
                             const double *y, const double *z, double *B, double *x, double *w,
                             long M, long N, bto_stream_t stream)
{
    SHARDED_PROLOGUE();
    return seq_gemver(*ac.ctx, A, u1, v1, u2, v2, alpha, beta, y, z, B, x, w, M, N, st);
}

// ---- section 6: unfused primitives (generic executor) -------------------------------

int bto_prim_matvec_async(const double *A, const double *x, double *out, long M, long N,
                          int transposed, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    BTO_TRY(check_mn(M, N));
    DeviceCtx &c = *ac.ctx;
    WsLayout lay;
    MvArgs a{};
    FinArgs f{};
    a.A = A;
    if (transposed) {                    // out[j] = sum_i A[i,j] x[i]
        Pass<kFlagT> pass;
        BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, A), &lay));
        BTO_TRY(size_ws(c, lay));
        a.roww = x;
        f.cmode = kColPlain; f.colout = out;
        return pass.run(c, a, f, st);
    }
    Pass<kFlagN> pass;                   // out[i] = sum_j A[i,j] x[j]
    BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, A), &lay));
    BTO_TRY(size_ws(c, lay));
    a.colw = x;
    f.rmode = kRowPlain; f.rowout = out;
    return pass.run(c, a, f, st);
}

int bto_prim_axpby_async(double alpha, const double *x, double beta, const double *y,
                         double *out, long n, int mode, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    if (n < 1 || mode < 0 || mode > 3 || !x || !out || (mode != 0 && !y)) {
        return fail(BTO_ERR_INVALID, "prim_axpby: bad arguments");
    }
    long grid = (n + kThreads - 1) / kThreads;
    const long cap = (long)ac.ctx->sm_count * 16;
    if (grid > cap) grid = cap;
    prim_axpby_kernel<<<(unsigned)grid, kThreads, 0, st>>>(alpha, x, beta, y, out, n, mode);
    return check_launch("prim_axpby_kernel");
}

int bto_prim_outer_async(const double *u, const double *v, double *out, long M, long N,
                         bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    BTO_TRY(check_mn(M, N));
    long grid = (M * N + kThreads - 1) / kThreads;
    const long cap = (long)ac.ctx->sm_count * 16;
    if (grid > cap) grid = cap;
    prim_outer_kernel<<<(unsigned)grid, kThreads, 0, st>>>(u, v, out, M, N);
    return check_launch("prim_outer_kernel");
}

int bto_prim_dot_async(const double *x, const double *y, double *out, long n, bto_stream_t stream)
{
    ASYNC_PROLOGUE();
    if (n < 1) return fail(BTO_ERR_INVALID, "extent %ld must be >= 1", n);
    DeviceCtx &c = *ac.ctx;
    long grid = (n + kThreads - 1) / kThreads;
    const long cap = (long)c.sm_count * 8;
    if (grid > cap) grid = cap;
    WsLayout lay;
    const size_t off = lay.take((size_t)grid);
    BTO_TRY(size_ws(c, lay));
    prim_dot_kernel<<<(unsigned)grid, kThreads, 0, st>>>(
        x, y, out, reinterpret_cast<double *>(c.ws + off), c.tickets + 1, n);
    return check_launch("prim_dot_kernel");
}

// ---- section 4: control ----------------------------------------------------------

int bto_set_stream(bto_stream_t stream)
{
    AsyncCall ac;
    if (ac.rc != BTO_OK) return ac.rc;
    ac.ctx->stream = static_cast<cudaStream_t>(stream);
    return BTO_OK;
}

static long *tuning_slot(const char *key)
{
    if (!key) return nullptr;
    if (!strcmp(key, "mv_rows")) return &g_tuning.mv_rows;
    if (!strcmp(key, "mv_vec")) return &g_tuning.mv_vec;
    if (!strcmp(key, "grid_per_sm")) return &g_tuning.grid_per_sm;
    if (!strcmp(key, "mv_minb")) return &g_tuning.mv_minb;
    if (!strcmp(key, "vec_unroll")) return &g_tuning.vec_unroll;
    if (!strcmp(key, "vec_grid_per_sm")) return &g_tuning.vec_grid_per_sm;
    if (!strcmp(key, "atax_fused")) return &g_tuning.atax_fused;
    if (!strcmp(key, "atax_cluster")) return &g_tuning.atax_cluster;
    if (!strcmp(key, "atax_stages")) return &g_tuning.atax_stages;
    if (!strcmp(key, "atax_rows")) return &g_tuning.atax_rows;
    if (!strcmp(key, "debug")) return &g_tuning.debug;
    if (!strcmp(key, "pdl")) return &g_tuning.pdl;
    if (!strcmp(key, "exchange_phases")) return &g_tuning.exchange_phases;
    if (!strcmp(key, "host_pipeline")) return &g_tuning.host_pipeline;
    if (!strcmp(key, "host_panel_mib")) return &g_tuning.host_panel_mib;
    return nullptr;
}

int bto_set_tuning(const char *key, long value)
{
    std::lock_guard<std::mutex> lock(g_mu);
    long *slot = tuning_slot(key);
    if (!slot) return fail(BTO_ERR_INVALID, "unknown tuning key %s", key ? key : "(null)");
    bool ok = value >= 0;
    if (slot == &g_tuning.mv_rows) ok = value == 0 || value == 8 || value == 16 || value == 32;
    if (slot == &g_tuning.mv_minb) ok = value == 0 || value == 1 || value == 2 || value == 3 || value == 4 || value == 6;
    if (slot == &g_tuning.mv_vec) ok = value == 0 || value == 1 || value == 2;
    if (slot == &g_tuning.vec_unroll) ok = value == 1 || value == 2 || value == 4;
    if (slot == &g_tuning.atax_fused || slot == &g_tuning.host_pipeline) ok = value == 0 || value == 1;
    if (slot == &g_tuning.host_panel_mib) ok = value >= 1 && value <= 4096;
    if (slot == &g_tuning.exchange_phases) ok = value >= 1 && value <= 3;
    if (slot == &g_tuning.atax_cluster) ok = value == 0 || value == 1 || value == 2 || value == 4 || value == 8 || value == 16;
    if (slot == &g_tuning.atax_stages) ok = value == 0 || (value >= 2 && value <= 8);
    if (slot == &g_tuning.atax_rows) ok = value == 0 || value == 1;
    if (slot == &g_tuning.grid_per_sm || slot == &g_tuning.vec_grid_per_sm) ok = value >= 0 && value <= 64;
    if (!ok) return fail(BTO_ERR_INVALID, "tuning %s=%ld is not supported", key, value);
    *slot = value;
    return BTO_OK;
}

long bto_get_tuning(const char *key)
{
    std::lock_guard<std::mutex> lock(g_mu);
    long *slot = tuning_slot(key);
    return slot ? *slot : -1;
}

double bto_bytes_min(const char *kernel, long M, long N)
{
    if (!kernel) return -1.0;
    const double m = (double)M, n = (double)N;
    if (!strcmp(kernel, "axpydot")) return 32.0 * m;
    if (!strcmp(kernel, "vadd")) return 32.0 * m;
    if (!strcmp(kernel, "waxpby")) return 24.0 * m;
    if (!strcmp(kernel, "bicgk")) return 8.0 * m * n + 16.0 * m + 16.0 * n;
    if (!strcmp(kernel, "atax")) return 8.0 * m * n + 16.0 * n;
    if (!strcmp(kernel, "batax")) return 8.0 * m * n + 16.0 * n;
    if (!strcmp(kernel, "gesummv")) return 16.0 * m * n + 8.0 * n + 8.0 * m;
    if (!strcmp(kernel, "dgemv")) return 8.0 * m * n + 8.0 * n + 16.0 * m;
    // read A, write B, re-read B; u1,u2,y (M) v1,v2,z (N) in; x out + re-read; w out
    if (!strcmp(kernel, "gemver")) return 24.0 * m * n + 32.0 * m + 40.0 * n;
    // A twice; y (M), z (N) in; x out + re-read (N); w out (M)
    if (!strcmp(kernel, "dgemvt")) return 16.0 * m * n + 16.0 * m + 24.0 * n;
    return -1.0;
}

int bto_device_info(int *sm_count, int *max_threads_per_sm, long *l2_bytes,
                    long *global_bytes)
{
    AsyncCall ac;
    if (ac.rc != BTO_OK) return ac.rc;
    if (sm_count) *sm_count = ac.ctx->sm_count;
    if (max_threads_per_sm) *max_threads_per_sm = ac.ctx->max_threads_per_sm;
    if (l2_bytes) *l2_bytes = ac.ctx->l2_bytes;
    if (global_bytes) *global_bytes = ac.ctx->global_bytes;
    return BTO_OK;
}

long bto_workspace_bytes(void)
{
    std::lock_guard<std::mutex> lock(g_mu);
    long total = 0;
    for (DeviceCtx &c : g_ctx) total += (long)(c.ws_bytes + c.arena_bytes);
    return total;
}

int bto_release_workspace(void)
{
    AsyncCall ac;
    if (ac.rc != BTO_OK) return ac.rc;
    CUDA_TRY(cudaDeviceSynchronize());
    DeviceCtx &c = *ac.ctx;
    if (c.ws) CUDA_TRY(cudaFree(c.ws));
    if (c.arena) CUDA_TRY(cudaFree(c.arena));
    c.ws = nullptr; c.ws_bytes = 0;
    c.arena = nullptr; c.arena_bytes = 0;
    return BTO_OK;
}

}  // extern "C"
