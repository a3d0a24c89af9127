// Calibrate basic latencies on B200 (cycles): dependent DFMA chain, dependent
// LDS.64 chain, __syncthreads with 256 threads, DMUL by reciprocal vs DDIV.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(long long* out, double* buf, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 1) % 1024;
    __syncthreads();
    double a = buf[0], b = buf[1], c = buf[2];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) c = fma(a, c, b);  // dependent DFMA
    long long t1 = clock64();
    int idx = threadIdx.x & 31;
    for (int i = 0; i < n; ++i) idx = int(sm[idx]) & 1023;  // dependent LDS.64 + cvt
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t3 = clock64();
    double d = c;
    for (int i = 0; i < n; ++i) d = d / (b + i);  // dependent DDIV
    long long t4 = clock64();
    double e = c;
    for (int i = 0; i < n; ++i) e = __drcp_rn(e + 1.0);
    long long t5 = clock64();
    double f = c;
    for (int i = 0; i < n; ++i) f = sqrt(f + 2.0);
    long long t6 = clock64();
    // independent DFMAs: 8 chains
    double x0 = a, x1 = b, x2 = c, x3 = a + 1, x4 = b + 1, x5 = c + 1, x6 = a + 2, x7 = b + 2;
    long long t7 = clock64();
    for (int i = 0; i < n; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    long long t8 = clock64();
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0);
        out[1] = (t2 - t1);
        out[2] = (t3 - t2);
        out[3] = (t4 - t3);
        out[4] = (t5 - t4);
        out[5] = (t6 - t5);
        out[6] = (t8 - t7);
    }
    buf[3 + threadIdx.x % 4] = c + idx + d + e + f + x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
    long long* out;
    double* buf;
    cudaMalloc(&out, 128);
    cudaMalloc(&buf, 128);
    double h[4] = {0.999, 0.001, 1.0, 0};
    cudaMemcpy(buf, h, 32, cudaMemcpyHostToDevice);
    const int n = 1000;
    for (int threads : {32, 256}) {
        long long r[8];
        for (int rep = 0; rep < 3; ++rep) probe<<<1, threads>>>(out, buf, n);
        cudaMemcpy(r, out, 56, cudaMemcpyDeviceToHost);
        printf("threads %3d per-op cycles: dfma-dep %.1f  lds-dep %.1f  syncthreads %.1f  ddiv %.1f"
               "  drcp %.1f  sqrt %.1f  8x-indep-dfma(per iter) %.1f\n",
               threads, r[0] / double(n), r[1] / double(n), r[2] / double(n), r[3] / double(n),
               r[4] / double(n), r[5] / double(n), r[6] / double(n));
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
