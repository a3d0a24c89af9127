// Microbenchmark of the small-matrix building blocks (rowalg.cuh) in one CTA:
// cycles per call of block_chol / rows_uinv / rows_utinv / gram_rows at the
// BASELINE shapes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I paper_2503_18759_b200/csrc tools/probes/rowalg_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "rowalg.cuh"

using namespace cpdb;

template <int NT>
__global__ void bench(int R, int rows, long long* out, double* sink) {
    extern __shared__ double sm[];
    const int ld = R + 1;
    double* g = sm;                 // R x R
    double* d = g + R * R;          // 64
    double* w = d + 64;             // rows x (R+1)
    Owned<NT> own;
    own.init(R);
    // SPD matrix: diag dominant
    for (int e = threadIdx.x; e < R * R; e += NT) {
        const int i = e / R, j = e % R;
        g[e] = (i == j) ? R + 1.0 : 1.0 / (1 + i + j);
    }
    for (int e = threadIdx.x; e < rows * ld; e += NT) w[e] = 1.0 + (e % 7) * 0.1;
    __syncthreads();
    long long t0 = clock64();
    bool ok = block_chol<NT>(g, R, R, d, own);
    __syncthreads();
    long long t1 = clock64();
    rows_uinv<NT>(w, ld, rows, g, R, d, R);
    __syncthreads();
    long long t2 = clock64();
    rows_utinv<NT>(w, ld, rows, g, R, d, R);
    __syncthreads();
    long long t3 = clock64();
    gram_rows<NT>(w, ld, rows, g, R, own);
    __syncthreads();
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t1;
        out[2] = t3 - t2;
        out[3] = t4 - t3;
        sink[0] = ok ? g[0] + w[0] : -1;
    }
}

int main() {
    long long* out;
    double* sink;
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 64);
    cudaFuncSetAttribute(bench<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int cases[][2] = {{10, 13}, {16, 16}, {20, 32}, {32, 64}, {64, 32}, {32, 128}};
    for (auto& c : cases) {
        const int R = c[0], rows = c[1];
        const size_t smem = (R * R + 64 + rows * (R + 1)) * 8;
        long long h[4];
        for (int rep = 0; rep < 3; ++rep) bench<256><<<1, 256, smem>>>(R, rows, out, sink);
        cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        printf("R=%2d rows=%3d  chol %7lld  uinv %7lld  utinv %7lld  gram %7lld cycles\n", R, rows,
               h[0], h[1], h[2], h[3]);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
