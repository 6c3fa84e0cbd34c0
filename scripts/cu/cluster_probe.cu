// How many clusters of each size can be co-resident on this GPU (GPC structure), for a kernel
// with one CTA per SM (200 KB dynamic shared memory) and for a light kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o gpurun_out/cluster_probe scripts/cu/cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe_kernel(int *out) { extern __shared__ unsigned char s[]; if (out) out[0] = s[0]; }

int main()
{
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    printf("%s: %d SMs\n", prop.name, prop.multiProcessorCount);
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const size_t smems[3] = {200 * 1024, 100 * 1024, 1024};
    for (size_t smem : smems) {
        for (int threads : {256, 512}) {
            printf("smem %3zu KB, %d threads:", smem / 1024, threads);
            for (int c = 1; c <= 16; ++c) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(c * 64, 1, 1);
                cfg.blockDim = dim3(threads, 1, 1);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = c;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                int n = -1;
                cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_kernel, &cfg);
                if (e != cudaSuccess) { cudaGetLastError(); n = -1; }
                printf(" C%d:%d(%d)", c, n, n * c);
            }
            printf("\n");
        }
    }
    return 0;
}
