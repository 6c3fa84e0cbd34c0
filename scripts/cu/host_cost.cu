// Host-side cost of one library call from C (no Python): bto_bicgk_async / bto_gemver_async /
// bto_axpydot_async on small operands, against bare launches of an empty kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/host_cost scripts/cu/host_cost.cu -ldl
//   ./build/host_cost paper_1205_1098_b200/libbto_b200.so
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <dlfcn.h>

__global__ void empty_kernel(int) {}

typedef int (*bicgk_fn)(const double *, const double *, const double *, double *, double *, long, long, void *);
typedef int (*gemver_fn)(const double *, const double *, const double *, const double *, const double *, double,
                         double, const double *, const double *, double *, double *, double *, long, long, void *);
typedef int (*axpydot_fn)(const double *, const double *, const double *, double, double *, double *, long, void *);

template <typename F>
double per_call_us(F fn, int reps)
{
    for (int i = 0; i < 200; ++i) fn();
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) fn();
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main(int argc, char **argv)
{
    void *lib = dlopen(argc > 1 ? argv[1] : "paper_1205_1098_b200/libbto_b200.so", RTLD_NOW);
    if (!lib) { printf("dlopen failed: %s\n", dlerror()); return 1; }
    bicgk_fn bicgk = (bicgk_fn)dlsym(lib, "bto_bicgk_async");
    gemver_fn gemver = (gemver_fn)dlsym(lib, "bto_gemver_async");
    axpydot_fn axpydot = (axpydot_fn)dlsym(lib, "bto_axpydot_async");
    const long M = 256, N = 512;
    double *A, *B, *v[8];
    cudaMalloc(&A, M * N * 8); cudaMalloc(&B, M * N * 8);
    cudaMemset(A, 0, M * N * 8);
    for (auto &p : v) { cudaMalloc(&p, 4096 * 8); cudaMemset(p, 0, 4096 * 8); }
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    const int reps = 20000;
    printf("bare launch x1            %6.2f us\n", per_call_us([&] { empty_kernel<<<148, 256, 0, st>>>(0); }, reps));
    printf("bare launch x2            %6.2f us\n", per_call_us([&] { empty_kernel<<<148, 256, 0, st>>>(0); empty_kernel<<<16, 256, 0, st>>>(0); }, reps));
    printf("bto_axpydot_async (1)     %6.2f us\n", per_call_us([&] { axpydot(v[0], v[1], v[2], 0.5, v[3], v[4], 4096, st); }, reps));
    printf("bto_bicgk_async   (2)     %6.2f us\n", per_call_us([&] { bicgk(A, v[0], v[1], v[2], v[3], M, N, st); }, reps));
    printf("bto_gemver_async  (4)     %6.2f us\n", per_call_us([&] { gemver(A, v[0], v[1], v[2], v[3], 0.5, 0.25, v[4], v[5], B, v[6], v[7], M, N, st); }, reps));
    return 0;
}
