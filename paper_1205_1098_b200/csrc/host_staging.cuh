// host_staging.cuh -- host/device argument staging and the host-operand panel pipeline
// Part of the host side of libbto_b200.so; included by api.cu (one translation unit).
#pragma once
#include "host_sequences.cuh"

namespace bto_host {
namespace {          // internal linkage: nothing here is part of the C ABI

using namespace bto;

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
}  // namespace bto_host
