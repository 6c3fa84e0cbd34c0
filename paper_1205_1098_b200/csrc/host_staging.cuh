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

// true for ordinary (pageable, unregistered) host memory
bool pageable_memory(const void *p)
{
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return attr.type == cudaMemoryTypeUnregistered;
}

// ---------------------------------------------------------------------------
// Pageable host operands.  cudaMemcpyAsync from pageable memory runs at
// ~11 GB/s on this platform (the driver bounces it through a small pinned
// buffer on one thread); the reference's own caller passes exactly such
// buffers (numpy arrays, runtime.py:99-150).  Large pageable operands are
// therefore copied by several host threads into three pinned 64 MiB slots
// that the copy engine drains (or fills, for outputs) concurrently.

constexpr size_t kBounceBytes = 64u << 20;
constexpr size_t kBounceMin = 16u << 20;       // smaller copies are not worth the threads

// slots [base, base+3)
cudaError_t bounce_setup(DeviceCtx &c, int base)
{
    for (int i = base; i < base + 3; ++i) {
        cudaError_t e = cudaSuccess;
        if (!c.bounce[i]) e = cudaHostAlloc(reinterpret_cast<void **>(&c.bounce[i]), kBounceBytes, cudaHostAllocDefault);
        if (e == cudaSuccess && !c.bounce_ev[i]) e = cudaEventCreateWithFlags(&c.bounce_ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

int host_copy_threads()
{
    if (g_tuning.host_threads > 0) return (int)g_tuning.host_threads;
    unsigned hw = std::thread::hardware_concurrency();
    int t = hw ? (int)hw : 4;
    if (t > 16) t = 16;
    return t;
}

// memcpy with non-temporal stores: the destination (a bounce slot the copy engine
// reads next, or a result the caller reads later) is not wanted in this core's cache,
// and skipping the read-for-ownership saves a third of the host memory traffic.
void stream_copy(char *dst, const char *src, size_t bytes)
{
#if defined(__SSE2__)
    if (g_tuning.host_nt && bytes >= 4096) {
        const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
        memcpy(dst, src, head);
        dst += head; src += head; bytes -= head;
        const size_t blocks = bytes / 64;
        for (size_t b = 0; b < blocks; ++b, dst += 64, src += 64) {
            const __m128i r0 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src));
            const __m128i r1 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + 16));
            const __m128i r2 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + 32));
            const __m128i r3 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + 48));
            _mm_stream_si128(reinterpret_cast<__m128i *>(dst), r0);
            _mm_stream_si128(reinterpret_cast<__m128i *>(dst + 16), r1);
            _mm_stream_si128(reinterpret_cast<__m128i *>(dst + 32), r2);
            _mm_stream_si128(reinterpret_cast<__m128i *>(dst + 48), r3);
        }
        _mm_sfence();
        memcpy(dst, src, bytes - blocks * 64);
        return;
    }
#endif
    memcpy(dst, src, bytes);
}

// dst[0 .. bytes) = the 8-byte pattern `bits`, non-temporal (bytes is a multiple of 8)
void stream_fill(char *dst, unsigned long long bits, size_t bytes)
{
    unsigned long long *p = reinterpret_cast<unsigned long long *>(dst);
    size_t n = bytes / 8;
#if defined(__SSE2__)
    while (n && (reinterpret_cast<uintptr_t>(p) & 15)) { *p++ = bits; --n; }
    const __m128i v = _mm_set1_epi64x((long long)bits);
    for (; n >= 8; n -= 8, p += 8) {
        _mm_stream_si128(reinterpret_cast<__m128i *>(p), v);
        _mm_stream_si128(reinterpret_cast<__m128i *>(p + 2), v);
        _mm_stream_si128(reinterpret_cast<__m128i *>(p + 4), v);
        _mm_stream_si128(reinterpret_cast<__m128i *>(p + 6), v);
    }
    _mm_sfence();
#endif
    while (n) { *p++ = bits; --n; }
}

// Persistent helpers for the bounce copies (a thread per piece and call cost ~0.5 ms of thread
// creation per 64 MiB chunk, a third of the chunk's copy time).  Pieces of concurrent calls
// (GEMVER fills inbound slots while its helper drains outbound ones) share one queue; a caller
// works on the queue too until its own pieces are done.  The pool is created on first use and
// never destroyed (its threads sleep on a condition variable and die with the process).
class CopyPool {
public:
    static CopyPool &get()
    {
        static CopyPool *pool = new CopyPool();
        return *pool;
    }

    // src == nullptr: fill dst with the 8-byte pattern `bits` instead of copying
    void copy(char *dst, const char *src, size_t bytes, int nt, unsigned long long bits = 0)
    {
        const size_t piece = ((bytes / nt) + 4095) & ~size_t(4095);
        std::atomic<int> left{0};
        {
            std::lock_guard<std::mutex> g(mu_);
            for (size_t lo = 0; lo < bytes; lo += piece) {
                const size_t len = lo + piece < bytes ? piece : bytes - lo;
                queue_.push_back({dst + lo, src ? src + lo : nullptr, len, &left, bits});
                left.fetch_add(1, std::memory_order_relaxed);
            }
            while ((int)workers_ < nt - 1) {
                std::thread([this] { serve(); }).detach();
                ++workers_;
            }
        }
        cv_.notify_all();
        while (left.load(std::memory_order_acquire) > 0) {
            Piece p;
            if (take(&p)) {
                run(p);
            } else {
                std::this_thread::yield();       // the last pieces are in other threads' hands
            }
        }
    }

private:
    struct Piece { char *dst; const char *src; size_t len; std::atomic<int> *left; unsigned long long bits; };

    bool take(Piece *p)
    {
        std::lock_guard<std::mutex> g(mu_);
        if (queue_.empty()) return false;
        *p = queue_.front();
        queue_.pop_front();
        return true;
    }

    static void run(const Piece &p)
    {
        if (p.src) {
            stream_copy(p.dst, p.src, p.len);
        } else {
            stream_fill(p.dst, p.bits, p.len);
        }
        p.left->fetch_sub(1, std::memory_order_release);
    }

    void serve()
    {
        for (;;) {
            Piece p;
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [this] { return !queue_.empty(); });
                p = queue_.front();
                queue_.pop_front();
            }
            run(p);
        }
    }

    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Piece> queue_;
    size_t workers_ = 0;
};

void parallel_memcpy(char *dst, const char *src, size_t bytes, int nt)
{
    if (nt <= 1 || bytes < (4u << 20)) {
        stream_copy(dst, src, bytes);
        return;
    }
    CopyPool::get().copy(dst, src, bytes, nt);
}

// host (pageable) -> device, enqueued on `s`; returns once `src` has been read.
// (cudaError_t, no fail(): the device->host twin also runs on a helper thread.)
cudaError_t h2d_bounced(DeviceCtx &c, void *dst, const void *src, size_t bytes, cudaStream_t s,
                        int nt)
{
    cudaError_t e = bounce_setup(c, 0);
    size_t off = 0;
    for (int i = 0; off < bytes && e == cudaSuccess; ++i, off += kBounceBytes) {
        const int slot = i % 3;
        const size_t len = bytes - off < kBounceBytes ? bytes - off : kBounceBytes;
        e = cudaEventSynchronize(c.bounce_ev[slot]);              // slot drained by its last copy
        if (e != cudaSuccess) break;
        parallel_memcpy(c.bounce[slot], static_cast<const char *>(src) + off, len, nt);
        e = cudaMemcpyAsync(static_cast<char *>(dst) + off, c.bounce[slot], len,
                            cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(c.bounce_ev[slot], s);
    }
    return e;
}

// device -> host (pageable); everything queued on `s` before the call is waited for
cudaError_t d2h_bounced(DeviceCtx &c, void *dst, const void *src, size_t bytes, cudaStream_t s,
                        int nt)
{
    cudaError_t e = bounce_setup(c, 3);
    if (e != cudaSuccess) return e;
    const size_t nchunks = (bytes + kBounceBytes - 1) / kBounceBytes;
    auto issue = [&](size_t i) -> cudaError_t {
        const int slot = 3 + (int)(i % 3);
        const size_t off = i * kBounceBytes;
        const size_t len = bytes - off < kBounceBytes ? bytes - off : kBounceBytes;
        cudaError_t r = cudaMemcpyAsync(c.bounce[slot], static_cast<const char *>(src) + off, len,
                                        cudaMemcpyDeviceToHost, s);
        return r == cudaSuccess ? cudaEventRecord(c.bounce_ev[slot], s) : r;
    };
    // two copies in flight while the third slot is emptied by the host threads
    for (size_t i = 0; i < nchunks && i < 2 && e == cudaSuccess; ++i) e = issue(i);
    for (size_t i = 0; i < nchunks && e == cudaSuccess; ++i) {
        const int slot = 3 + (int)(i % 3);
        const size_t off = i * kBounceBytes;
        const size_t len = bytes - off < kBounceBytes ? bytes - off : kBounceBytes;
        if (i + 2 < nchunks) e = issue(i + 2);                    // its slot was emptied at i-1
        if (e == cudaSuccess) e = cudaEventSynchronize(c.bounce_ev[slot]);
        if (e != cudaSuccess) break;
        parallel_memcpy(static_cast<char *>(dst) + off, c.bounce[slot], len, nt);
    }
    return e;
}

bool bounce_wanted(const void *host, size_t bytes)
{
    return g_tuning.host_bounce && bytes >= kBounceMin && pageable_memory(host);
}

// one host <-> device transfer on `s`, through the bounce slots when that pays
int copy_in(DeviceCtx &c, void *dst, const void *src, size_t bytes, cudaStream_t s, int nt = 0)
{
    if (bounce_wanted(src, bytes)) {
        CUDA_TRY(h2d_bounced(c, dst, src, bytes, s, nt ? nt : host_copy_threads()));
        return BTO_OK;
    }
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return BTO_OK;
}

int copy_out(DeviceCtx &c, void *dst, const void *src, size_t bytes, cudaStream_t s, int nt = 0)
{
    if (bounce_wanted(dst, bytes)) {
        CUDA_TRY(d2h_bounced(c, dst, src, bytes, s, nt ? nt : host_copy_threads()));
        return BTO_OK;
    }
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    return BTO_OK;
}

// Drains finished device panels into pageable host memory on a helper thread while the
// calling thread keeps feeding the other direction.  post() hands over a panel whose
// producer event has ALREADY been recorded; close() waits for the last one.
class PanelDrain {
public:
    PanelDrain(DeviceCtx &c, cudaStream_t s, int nt) : c_(c), s_(s), nt_(nt) {}
    ~PanelDrain() { close(); }
    void post(void *dst, const void *src, size_t bytes, cudaEvent_t produced)
    {
        if (!worker_.joinable()) worker_ = std::thread([this] { run(); });
        std::lock_guard<std::mutex> g(mu_);
        jobs_.push_back({dst, src, bytes, produced});
        cv_.notify_one();
    }
    cudaError_t close()
    {
        if (worker_.joinable()) {
            {
                std::lock_guard<std::mutex> g(mu_);
                closed_ = true;
                cv_.notify_one();
            }
            worker_.join();
        }
        return err_;
    }

private:
    struct Job { void *dst; const void *src; size_t bytes; cudaEvent_t produced; };
    void run()
    {
        err_ = cudaSetDevice(c_.device);
        for (size_t next = 0;; ++next) {
            Job j;
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return next < jobs_.size() || closed_; });
                if (next >= jobs_.size()) return;
                j = jobs_[next];
            }
            if (err_ != cudaSuccess) continue;                    // keep consuming, copy nothing
            err_ = cudaStreamWaitEvent(s_, j.produced, 0);
            if (err_ == cudaSuccess) err_ = d2h_bounced(c_, j.dst, j.src, j.bytes, s_, nt_);
        }
    }
    DeviceCtx &c_;
    cudaStream_t s_;
    int nt_;
    std::thread worker_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::vector<Job> jobs_;
    bool closed_ = false;
    cudaError_t err_ = cudaSuccess;
};

class Call {
public:
    Call() : lock_(g_mu)
    {
        g_err = BTO_OK;
        g_errmsg[0] = 0;
        reset_call_record();
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
                status(copy_in(*ctx_, *a.slot, a.host, (size_t)a.count * sizeof(double), stream()));
                if (!ok()) return;
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
                status(copy_out(*ctx_, a.host, *a.slot, (size_t)a.count * sizeof(double), stream()));
                if (!ok()) break;
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
    f.col_cols = kJoinCols;
    f.col_blocks = (int)((n + kJoinCols - 1) / kJoinCols);
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
    // pageable A / B: this thread fills the inbound bounce slots, a helper drains B
    const size_t panel_bytes = (size_t)(M / P) * N * sizeof(double);
    const bool drain_b = bounce_wanted(hB, panel_bytes);
    const int nt = host_copy_threads();
    const int nt_in = drain_b && bounce_wanted(hA, panel_bytes) ? (nt + 1) / 2 : nt;
    PanelDrain drain(c, c.copy_out, nt_in < nt ? nt - nt_in : nt);
    for (long p = 0; p < P; ++p) {
        const long r0 = (M * p) / P, r1 = (M * (p + 1)) / P;
        if (r1 == r0) {
            CUDA_TRY(cudaMemsetAsync(panel_sums + p * N, 0, (size_t)N * sizeof(double), main));
            continue;
        }
        const size_t off = (size_t)r0 * N, bytes = (size_t)(r1 - r0) * N * sizeof(double);
        BTO_TRY(copy_in(c, dA + off, hA + off, bytes, c.copy_in, nt_in));
        CUDA_TRY(cudaEventRecord(c.events[2 * p], c.copy_in));
        CUDA_TRY(cudaStreamWaitEvent(main, c.events[2 * p], 0));
        FinArgs f{};
        f.cmode = kColPlain;
        f.colout = panel_sums + p * N;
        BTO_TRY(seq_pass1(c, dA + off, u1 + r0, v1, u2 + r0, v2, y + r0, dB + off, f, r1 - r0, N,
                          main));
        CUDA_TRY(cudaEventRecord(c.events[2 * p + 1], main));
        if (drain_b) {
            drain.post(hB + off, dB + off, bytes, c.events[2 * p + 1]);
        } else {
            CUDA_TRY(cudaStreamWaitEvent(c.copy_out, c.events[2 * p + 1], 0));
            CUDA_TRY(cudaMemcpyAsync(hB + off, dB + off, bytes, cudaMemcpyDeviceToHost, c.copy_out));
        }
    }
    BTO_TRY(join_partials(panel_sums, P, N, kColAxpz, beta, z, x, main));
    BTO_TRY(seq_pass2(c, dB, x, alpha, w, M, N, main));
    CUDA_TRY(drain.close());
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
        reset_call_record();
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
