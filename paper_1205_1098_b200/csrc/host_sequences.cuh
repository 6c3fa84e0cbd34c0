// host_sequences.cuh -- the kernel sequences of the ten corpus kernels (device pointers, asynchronous)
// Part of the host side of libbto_b200.so; included by api.cu (one translation unit).
#pragma once
#include "atax_cluster.cuh"
#include "host_plan.cuh"

namespace bto_host {
namespace {          // internal linkage: nothing here is part of the C ABI

using namespace bto;

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
    BTO_TRY(size_ws(c, lay, st));
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
    int C = 1, KMAX = 1, RG = 1, W = 0, S = 0, minb = 1;
    size_t smem = 0;
    int nclusters = 0;
};

// TR (rows per panel): the largest power of two with TR * KMAX <= 16, capped at 8 -- a panel is at
// most 16 double2 per thread.  `small` halves it (fewer registers per tile, more panels per byte).
// KMAX need not be a power of two: a slice of 3072 columns (N = 24576 over 8 CTAs) in a KMAX = 8
// kernel runs 8 iterations for 6 of data, and the per-panel chain is what bounds the kernel --
// 5.4 TB/s where KMAX = 6 gives 7 (profiles/r02/atax_kmax.log).
constexpr int atax_tr(int kmax) { return kmax <= 2 ? 8 : kmax <= 4 ? 4 : kmax <= 8 ? 2 : 1; }

template <int C>
AtaxKernel atax_kernel_ptr(int kmax, bool small)
{
    switch (kmax) {
        case 1: return small ? atax_cluster_kernel<C, 1, 4> : atax_cluster_kernel<C, 1, 8>;
        case 2: return small ? atax_cluster_kernel<C, 2, 4> : atax_cluster_kernel<C, 2, 8>;
        case 3: return small ? atax_cluster_kernel<C, 3, 2> : atax_cluster_kernel<C, 3, 4>;
        case 4: return small ? atax_cluster_kernel<C, 4, 2> : atax_cluster_kernel<C, 4, 4>;
        case 5: return small ? atax_cluster_kernel<C, 5, 1> : atax_cluster_kernel<C, 5, 2>;
        case 6: return small ? atax_cluster_kernel<C, 6, 1> : atax_cluster_kernel<C, 6, 2>;
        case 7: return small ? atax_cluster_kernel<C, 7, 1> : atax_cluster_kernel<C, 7, 2>;
        case 8: return small ? atax_cluster_kernel<C, 8, 1> : atax_cluster_kernel<C, 8, 2>;
        case 16: return atax_cluster_kernel<C, 16, 1>;
    }
    return nullptr;
}

// Cluster sizes that exist only to give mid-size matrices full-width slices (N = 24576 over 6 CTAs
// = 4096 columns each, where 8 or 9 CTAs hold 3072 / 2736 and the panels get too small for their
// fixed cost): whole panels, one CTA per SM, slices of 5 .. 8 iterations.
template <int C>
AtaxKernel atax_kernel_ptr_wide(int kmax, bool small)
{
    if (small) return nullptr;
    switch (kmax) {
        case 5: return atax_cluster_kernel<C, 5, 2>;
        case 6: return atax_cluster_kernel<C, 6, 2>;
        case 7: return atax_cluster_kernel<C, 7, 2>;
        case 8: return atax_cluster_kernel<C, 8, 2>;
    }
    return nullptr;
}

int atax_rows_of(int kmax, bool small)
{
    const int full = atax_tr(kmax);
    if (!small || kmax == 16) return full;
    return kmax == 1 ? 4 : full / 2;
}

// two CTAs per SM, one register tile of 8 double2 per thread (atax_cluster.cuh, MINB = 2)
template <int C>
AtaxKernel atax_kernel_ptr_two(int kmax)
{
    switch (kmax) {
        case 1: return atax_cluster_kernel<C, 1, 8, 2>;
        case 2: return atax_cluster_kernel<C, 2, 4, 2>;
        case 4: return atax_cluster_kernel<C, 4, 2, 2>;
        case 8: return atax_cluster_kernel<C, 8, 1, 2>;
    }
    return nullptr;
}

int atax_rows_of_two(int kmax) { return kmax >= 8 ? 1 : 8 / kmax; }

AtaxKernel atax_kernel_ptr(int c, int kmax, bool small, bool two)
{
    if (two) {
        switch (c) {
            case 1: return atax_kernel_ptr_two<1>(kmax);
            case 2: return atax_kernel_ptr_two<2>(kmax);
            case 4: return atax_kernel_ptr_two<4>(kmax);
            case 8: return atax_kernel_ptr_two<8>(kmax);
            case 9: return atax_kernel_ptr_two<9>(kmax);
        }
        return nullptr;
    }
    switch (c) {
        case 1: return atax_kernel_ptr<1>(kmax, small);
        case 2: return atax_kernel_ptr<2>(kmax, small);
        case 3: return atax_kernel_ptr_wide<3>(kmax, small);
        case 4: return atax_kernel_ptr<4>(kmax, small);
        case 5: return atax_kernel_ptr_wide<5>(kmax, small);
        case 6: return atax_kernel_ptr_wide<6>(kmax, small);
        case 7: return atax_kernel_ptr_wide<7>(kmax, small);
        case 8: return atax_kernel_ptr<8>(kmax, small);
        case 9: return atax_kernel_ptr<9>(kmax, small);
        case 10: return atax_kernel_ptr_wide<10>(kmax, small);
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
int plan_atax_cluster(DeviceCtx &c, int C, long M, long N, AtaxPlan *p, long *max_clusters);

int plan_atax(DeviceCtx &c, const double *A, const double *x, long M, long N, AtaxPlan *p)
{
    p->fn = nullptr;
    if (!g_tuning.atax_fused || (N % 2) || !aligned16(A) || !aligned16(x)) return BTO_OK;
    int C = (int)g_tuning.atax_cluster;
    long cover = 0;
    if (C != 0) return plan_atax_cluster(c, C, M, N, p, &cover);
    // Every cluster size that is built, priced by what bounds the kernel (profiles/r02/atax_sustained.md):
    // a panel of TR rows costs a fixed ~1150 cycles (the exchange chain) + ~62 per row and
    // 512-column iteration, and a cluster works through M / clusters rows.  Slices close to the
    // 4096-column maximum amortise the fixed part; clusters live inside a GPC, so their number
    // depends on the size (profiles/r02/cluster_probe.log: 74 x 2, 45 x 3, 33 x 4, 26 x 5, 22 x 6,
    // 15 x 7 / 8 / 9, 11 x 10, 7 x 16).  N = 24576: 6 CTAs x 4096 columns on 22 clusters instead of 9 x 2736
    // on 15; N = 32768 stays at 9 (profiles/r02/atax_csize.log).
    static const int kSizes[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 16};
    double best = 0.0;
    for (int C : kSizes) {
        AtaxPlan q;
        long cover = 0;
        BTO_TRY(plan_atax_cluster(c, C, M, N, &q, &cover));
        if (!q.fn) continue;
        if (q.KMAX == 16 && C < 16) continue;       // 8192-column slices: one-row panels and no registers to spare
        const double panel = 1150.0 / q.RG + 62.5 * q.KMAX;            // cycles per row
        const double cost = panel / (double)q.nclusters;
        // (ties: more SMs pulling on HBM)
        if (!p->fn || cost < best * 0.999 || (cost < best * 1.001 && q.nclusters * q.C > p->nclusters * p->C)) {
            *p = q;
            best = cost;
        }
    }
    return BTO_OK;
}

// The plan for one cluster size; *max_clusters = co-resident clusters the device offers.
int plan_atax_cluster(DeviceCtx &c, int C, long M, long N, AtaxPlan *p, long *max_clusters)
{
    p->fn = nullptr;
    long W = (N + C - 1) / C;
    W += W & 1;
    // a slice that starts off a 128-byte line costs the TMA stream ~7 % (C = 9 at N = 32768:
    // 3642 columns -> 6.76 TB/s for the copies alone, 3648 -> as good as C = 8)
    if (((W + 15) / 16) * 16 * (long)(C - 1) < N) W = ((W + 15) / 16) * 16;
    int kmax = (int)((W + 2 * kThreads - 1) / (2 * kThreads));      // iterations of 512 columns a slice needs
    const bool two_per_sm = g_tuning.atax_per_sm == 2;
    if (kmax > 8 || two_per_sm) {                                   // 9 .. 16 and the two-per-SM variants: powers of two
        int p2 = 1;
        while (p2 < kmax) p2 *= 2;
        kmax = p2;
    }
    if (kmax > 16) return BTO_OK;
    if ((long)(C - 1) * W >= N && C > 1) return BTO_OK;   // a CTA would own no column
    const bool small = g_tuning.atax_rows == 1;     // 1: half-height panels
    const bool two = g_tuning.atax_per_sm == 2;     // two CTAs per SM, one register tile each
    AtaxKernel fn = atax_kernel_ptr(C, kmax, small, two);
    if (!fn) return BTO_OK;
    const int rg = two ? atax_rows_of_two(kmax) : atax_rows_of(kmax, small);
    const size_t stage = (size_t)rg * W * sizeof(double);
    auto sm = c.static_smem.find(reinterpret_cast<const void *>(fn));
    if (sm == c.static_smem.end()) {
        cudaFuncAttributes fattr;
        CUDA_TRY(cudaFuncGetAttributes(&fattr, fn));
        sm = c.static_smem.emplace(reinterpret_cast<const void *>(fn), fattr.sharedSizeBytes).first;
    }
    // 227 KiB per CTA on sm_100 (113 KiB each for two per SM: 228 KiB per SM, 1 KiB reserved per
    // CTA), minus the kernel's static shared memory
    const size_t budget = (((two ? 113 : 227) * 1024 - sm->second) / 1024) * 1024;
    int S = (int)(budget / stage);
    if (S > 8) S = 8;
    if (g_tuning.atax_stages > 0 && g_tuning.atax_stages < S) S = (int)g_tuning.atax_stages;
    if (S < 2) return BTO_OK;
    p->C = C;
    p->KMAX = kmax;
    p->RG = rg;
    p->W = (int)W;
    p->S = S;
    p->minb = two ? 2 : 1;
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
    *max_clusters = ncl;
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
    BTO_TRY(size_ws(c, lay, st));
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
    char what[64];
    snprintf(what, sizeof(what), "atax_cluster_kernel<%d,%d,%d,%d>", p.C, p.KMAX, p.RG, p.minb);
    BTO_TRY(check_launch(what, reinterpret_cast<const void *>(p.fn)));
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
    if (skinny_applies(N, mat_aligned(N, A))) {
        // a row lives inside one CTA segment: t_i = A_i . x is complete before A_i leaves the
        // registers, so y = A' t needs no second pass
        WsLayout lay;
        const SkinnyPlan sp = plan_skinny(c, M, N, mat_aligned(N, A));
        const size_t off = lay.take((size_t)sp.grid * N);
        BTO_TRY(size_ws(c, lay, st));
        MvArgs a{};
        a.A = A; a.colw = x; a.M = M; a.N = N;
        a.colpart = reinterpret_cast<double *>(c.ws + off);
        FinArgs f{};
        f.rmode = kRowNone;
        f.cmode = scaled ? kColScale : kColPlain; f.cscale = beta; f.colout = y;
        return run_skinny<kFlagN | kFlagT | kFlagAtax>(c, sp, a, f, st);
    }
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
    BTO_TRY(size_ws(c, lay, st));
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
    BTO_TRY(size_ws(c, lay, st));
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
    BTO_TRY(size_ws(c, lay, st));
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
        BTO_TRY(size_ws(c, lay, st));
        return pass.run(c, a, f, st);
    }
    a.u1 = u1; a.v1 = v1; a.u2 = u2; a.v2 = v2; a.Bout = B;
    Pass<kFlagT | kFlagRank2> pass;
    BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, A, B), &lay));
    BTO_TRY(size_ws(c, lay, st));
    return pass.run(c, a, f, st);
}

int seq_pass2(DeviceCtx &c, const double *B, const double *x, double alpha,
              double *w, long M, long N, cudaStream_t st)
{
    WsLayout lay;
    Pass<kFlagN> pass;
    BTO_TRY(pass.prepare(c, M, N, mat_aligned(N, B), &lay));
    BTO_TRY(size_ws(c, lay, st));
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


}  // namespace
}  // namespace bto_host
