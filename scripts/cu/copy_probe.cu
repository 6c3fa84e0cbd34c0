// copy_probe.cu -- what a read+write stream can reach on this part, by mechanism:
//   0  ld.global.nc.v2 / st.global.cs.v2, grid-stride (what an elementwise kernel does)
//   1  the same with plain stores
//   2  TMA bulk load -> shared memory -> TMA bulk store (cp.async.bulk both ways), S-stage ring
//   3  ld.global -> registers -> shared memory -> TMA bulk store
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/cu/copy_probe.cu -o /tmp/copy_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CS>
__global__ void __launch_bounds__(256) copy_ldst(const double2 *__restrict__ a, double2 *__restrict__ b, long n2)
{
    const long stride = (long)gridDim.x * 256 * 4;
    for (long i = (long)blockIdx.x * 256 * 4 + threadIdx.x; i < n2; i += stride) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long j = i + u * 256;
            if (j < n2) asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(a + j));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long j = i + u * 256;
            if (j < n2) {
                if (CS) asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(b + j), "d"(v[u].x), "d"(v[u].y) : "memory");
                else b[j] = v[u];
            }
        }
    }
}

// TMA ring: one elected thread moves CHUNK bytes global -> smem -> global per stage
template <int CHUNK, int S>
__global__ void __launch_bounds__(128) copy_tma(const char *__restrict__ a, char *__restrict__ b, long nchunks)
{
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[S];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long first = blockIdx.x, step = gridDim.x;
    long issued = 0, done = 0;
    const long mine = first < nchunks ? (nchunks - first + step - 1) / step : 0;
    auto load = [&](long k) {
        const int s = (int)(k % S);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[s])), "r"(CHUNK) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s32(smem + (size_t)s * CHUNK)), "l"(a + (first + k * step) * CHUNK), "r"(CHUNK), "r"(s32(&full[s])) : "memory");
    };
    for (; issued < S - 1 && issued < mine; ++issued) load(issued);
    for (; done < mine; ++done) {
        const int s = (int)(done % S);
        const uint32_t par = (uint32_t)((done / S) & 1);
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D_%=;\nbra W_%=;\nD_%=:\n}\n"
                     ::"r"(s32(&full[s])), "r"(par) : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(b + (first + done * step) * CHUNK), "r"(s32(smem + (size_t)s * CHUNK)), "r"(CHUNK) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (issued < mine) {
            // the next load goes to the stage of chunk done - 1: wait until that store has READ it
            // (at most the store just committed may still be pending)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            load(issued);
            ++issued;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// loads through registers, stores through shared memory + TMA bulk store
template <int CHUNK, int S>
__global__ void __launch_bounds__(256) copy_ld_tmast(const char *__restrict__ a, char *__restrict__ b, long nchunks)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const long first = blockIdx.x, step = gridDim.x;
    long k = 0;
    for (long c = first; c < nchunks; c += step, ++k) {
        const int s = (int)(k % S);
        if (k >= S) {
            if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
            __syncthreads();
        }
        const double2 *src = reinterpret_cast<const double2 *>(a + c * CHUNK);
        double2 *dst = reinterpret_cast<double2 *>(smem + (size_t)s * CHUNK);
        constexpr int PER = CHUNK / 16 / 256;
        double2 v[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(src + threadIdx.x + u * 256));
#pragma unroll
        for (int u = 0; u < PER; ++u) dst[threadIdx.x + u * 256] = v[u];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(b + c * CHUNK), "r"(s32(dst)), "r"(CHUNK) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
static void run(const char *name, F launch, double gbytes)
{
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e9f, sum = 0.f;
    const int reps = 10;
    for (int i = 0; i < reps; ++i) {
        CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best; sum += ms;
    }
    CK(cudaGetLastError());
    printf("%-44s best %7.3f ms %7.0f GB/s   mean %7.3f ms %7.0f GB/s\n", name, best, gbytes / best * 1e3, sum / reps, gbytes / (sum / reps) * 1e3);
}

int main()
{
    const long bytes = 8L << 30;
    char *a, *b;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 1, bytes)); CK(cudaMemset(b, 0, bytes));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const double gb = 2.0 * bytes / 1e9;
    run("cudaMemcpy D2D", [&] { CK(cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice)); }, gb);
    for (int per : {4, 8, 16}) {
        char name[96];
        snprintf(name, sizeof name, "ld.nc / st.cs, %d CTAs per SM", per);
        run(name, [&] { copy_ldst<1><<<sms * per, 256>>>((const double2 *)a, (double2 *)b, bytes / 16); }, gb);
    }
    run("ld.nc / st (plain), 8 CTAs per SM", [&] { copy_ldst<0><<<sms * 8, 256>>>((const double2 *)a, (double2 *)b, bytes / 16); }, gb);
    {
        constexpr int CH = 32768, S = 6;
        CK(cudaFuncSetAttribute(copy_tma<CH, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * S));
        run("TMA load -> TMA store, 32 KiB x 6, 1 CTA/SM", [&] { copy_tma<CH, S><<<sms, 128, CH * S>>>(a, b, bytes / CH); }, gb);
    }
    {
        constexpr int CH = 16384, S = 6;
        CK(cudaFuncSetAttribute(copy_tma<CH, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * S));
        run("TMA load -> TMA store, 16 KiB x 6, 2 CTA/SM", [&] { copy_tma<CH, S><<<sms * 2, 128, CH * S>>>(a, b, bytes / CH); }, gb);
    }
    {
        constexpr int CH = 8192, S = 8;
        CK(cudaFuncSetAttribute(copy_tma<CH, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * S));
        run("TMA load -> TMA store, 8 KiB x 8, 3 CTA/SM", [&] { copy_tma<CH, S><<<sms * 3, 128, CH * S>>>(a, b, bytes / CH); }, gb);
    }
    {
        constexpr int CH = 32768, S = 3;
        CK(cudaFuncSetAttribute(copy_ld_tmast<CH, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * S));
        run("ld.nc -> smem -> TMA store, 32 KiB x 3, 2 CTA/SM", [&] { copy_ld_tmast<CH, S><<<sms * 2, 256, CH * S>>>(a, b, bytes / CH); }, gb);
    }
    {
        constexpr int CH = 16384, S = 3;
        CK(cudaFuncSetAttribute(copy_ld_tmast<CH, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * S));
        run("ld.nc -> smem -> TMA store, 16 KiB x 3, 4 CTA/SM", [&] { copy_ld_tmast<CH, S><<<sms * 4, 256, CH * S>>>(a, b, bytes / CH); }, gb);
    }
    // check
    unsigned char h[64];
    CK(cudaMemcpy(h, b + bytes - 64, 64, cudaMemcpyDeviceToHost));
    printf("tail byte %d (expect 1)\n", h[63]);
    return 0;
}
