// Launch-to-completion cost of an (almost) empty kernel: plain 8-CTA grid vs
// an 8-CTA thread-block cluster, with and without 200 KB dynamic smem, chained
// back to back on one stream (CUDA events over 200 launches).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void plain(int* x) { if (threadIdx.x == 0 && x) x[blockIdx.x] += 1; }
__global__ void clustered(int* x) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    if (threadIdx.x == 0 && x) x[blockIdx.x] += 1;
}

template <class K>
float run(K k, bool cluster, size_t smem, int threads) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(8);
    c.blockDim = dim3(threads);
    c.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    c.attrs = cluster ? at : nullptr;
    c.numAttrs = cluster ? 1 : 0;
    int* x;
    cudaMalloc(&x, 64);
    for (int i = 0; i < 20; ++i) cudaLaunchKernelEx(&c, k, x);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 200; ++i) cudaLaunchKernelEx(&c, k, x);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000 / 200;
}

int main() {
    printf("plain 8 CTAs          : %.2f us/launch\n", run(plain, false, 0, 512));
    printf("plain 8 CTAs 200KB    : %.2f us/launch\n", run(plain, false, 200 << 10, 512));
    printf("cluster 8             : %.2f us/launch\n", run(clustered, true, 0, 512));
    printf("cluster 8 200KB       : %.2f us/launch\n", run(clustered, true, 200 << 10, 512));
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
