// LaneRow (rowalg.cuh) row solves in isolation: cycles for `rows` rows, one CTA.
#include <cstdio>
#include <cuda_runtime.h>

#include "rowalg.cuh"

using namespace cpdb;

template <int RM, int NT>
__global__ void bench(int R, int rows, const double* vglobal, long long* out, double* sink) {
    using Row = LaneRow<RM>;
    constexpr int T = Row::T, G = NT / T;
    extern __shared__ double sm[];
    double* U = sm;
    double* dinv = U + RM * RM;
    double* w = dinv + RM;
    const int ld = R + 1;
    for (int e = threadIdx.x; e < RM * RM; e += NT) {
        const int i = e / RM, j = e % RM;
        U[e] = i == j ? 2.0 : (j > i ? 0.01 * (i + j) : 0.0);
    }
    for (int j = threadIdx.x; j < RM; j += NT) dinv[j] = 0.5;
    __syncthreads();
    const int grp = threadIdx.x / T, q = threadIdx.x % T;
    double acc = 0.0;
    long long t0 = clock64();
    for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
        const bool act = li < rows;
        Row x;
        x.load(vglobal + (act ? li : 0) * R, act ? R : 0, q);
        if (act) x.store(w + li * ld, R, q);
    }
    __syncthreads();
    long long t1 = clock64();
    for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
        const bool act = li < rows;
        Row x;
        x.load(w + (act ? li : 0) * ld, act ? R : 0, q);
        x.utinv(U, dinv, R, q);
        if (act) x.store(w + li * ld, R, q);
    }
    __syncthreads();
    long long t2 = clock64();
    for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
        const bool act = li < rows;
        Row x;
        x.load(w + (act ? li : 0) * ld, act ? R : 0, q);
        x.uinv(U, dinv, R, q);
        if (act) x.store(w + li * ld, R, q);
    }
    __syncthreads();
    long long t3 = clock64();
    for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
        const bool act = li < rows;
        Row x, wv;
        x.load(w + (act ? li : 0) * ld, act ? R : 0, q);
        wv.set_times_upper(x, U, R, q);
#pragma unroll
        for (int s = 0; s < Row::S; ++s) acc = fma(x.t[s], wv.t[s], acc);
    }
    __syncthreads();
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t1;
        out[2] = t3 - t2;
        out[3] = t4 - t3;
    }
    sink[threadIdx.x] = acc + w[0];
}

template <int RM, int NT>
void run(int R, int rows, const double* v, long long* out, double* sink) {
    const size_t smem = (RM * RM + RM + rows * (R + 1)) * 8;
    cudaFuncSetAttribute(bench<RM, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long h[4] = {0, 0, 0, 0};
    for (int rep = 0; rep < 3; ++rep) bench<RM, NT><<<1, NT, smem>>>(R, rows, v, out, sink);
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("RM=%d NT=%d R=%d rows=%d: gload %lld utinv %lld uinv %lld times_upper %lld (%s)\n", RM,
           NT, R, rows, h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long* out;
    double *sink, *v;
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 8192);
    cudaMalloc(&v, 1 << 20);
    cudaMemset(v, 0, 1 << 20);
    run<32, 512>(32, 64, v, out, sink);
    run<32, 256>(32, 64, v, out, sink);
    run<16, 512>(16, 16, v, out, sink);
    run<64, 512>(64, 32, v, out, sink);
    run<32, 512>(20, 32, v, out, sink);
    return 0;
}
