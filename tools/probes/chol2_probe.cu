// Cholesky latency inside one 256-thread CTA: block_chol (smem, one barrier
// per step) vs fast_chol (warp registers), R = 16 / 32 / 64.  clock64 cycles
// per factorisation (100 repetitions of factor + restore).
#include <cstdio>
#include <cuda_runtime.h>

#include "rowalg.cuh"

using namespace cpdb;

template <int RM, int MODE>
__global__ void __launch_bounds__(256) k(const double* g0, int R, long long* cyc, double* out) {
    __shared__ double g[RM * RM];
    __shared__ float keep_f[1];
    const double* keep = g0;
    (void)keep_f;

    __syncthreads();
    long long t0 = 0;
    for (int rep = 0; rep < 101; ++rep) {
        if (rep == 1) t0 = clock64();
        for (int e = threadIdx.x; e < R * R; e += 256) g[e] = keep[e];
        __syncthreads();
        if (MODE == 0) block_chol<256, (RM * RM + 255) / 256>(g, R, R);
        else reg_chol<256, RM>(g, R, R);
        __syncthreads();
    }
    if (threadIdx.x == 0) *cyc = (clock64() - t0) / 100;
    for (int e = threadIdx.x; e < R * R; e += 256) out[e] = g[e];
}

template <int RM>
void run(int R) {
    double* h = new double[R * R];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) h[i * R + j] = (i == j ? R : 0.0) + 1.0 / (1 + i + j);
    double *g, *o0, *o1;
    long long* c;
    cudaMalloc(&g, R * R * 8); cudaMalloc(&o0, R * R * 8); cudaMalloc(&o1, R * R * 8);
    cudaMalloc(&c, 16);
    cudaMemcpy(g, h, R * R * 8, cudaMemcpyHostToDevice);
    k<RM, 0><<<1, 256>>>(g, R, c, o0);
    k<RM, 1><<<1, 256>>>(g, R, c + 1, o1);
    long long hc[2];
    double a[4096], b[4096];
    cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(a, o0, R * R * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b, o1, R * R * 8, cudaMemcpyDeviceToHost);
    double md = 0;
    for (int e = 0; e < R * R; ++e) md = fmax(md, fabs(a[e] - b[e]));
    printf("R=%d block_chol %lld cycles  reg_chol %lld cycles  max|diff| %.3g  (%s)\n", R, hc[0],
           hc[1], md, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<16>(16);
    run<32>(20);
    run<32>(32);
    run<64>(64);
    return 0;
}
