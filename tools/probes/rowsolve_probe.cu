// Row triangular solve x <- x U^-1 on `rows` rows: register-resident row
// (compile-time RM, unrolled, U in smem with stride RM) vs the smem T-lane
// version in rowalg.cuh.  Cycles per call, one CTA.
#include <cstdio>
#include <cuda_runtime.h>

#include "rowalg.cuh"

using namespace cpdb;

template <int RM, int ACC>
__device__ __forceinline__ void reg_uinv(double (&x)[RM], const double* U, const double* dinv,
                                         int R) {
#pragma unroll
    for (int j = 0; j < RM; ++j) {
        if (j < R) {
            double s[ACC];
#pragma unroll
            for (int a = 0; a < ACC; ++a) s[a] = 0.0;
#pragma unroll
            for (int p = 0; p < j; ++p) s[p % ACC] = fma(x[p], U[p * RM + j], s[p % ACC]);
            double t = x[j];
#pragma unroll
            for (int a = 0; a < ACC; ++a) t -= s[a];
            x[j] = t * dinv[j];
        }
    }
}

// right-looking: after x[j] is final, update all later partial sums (ILP)
template <int RM>
__device__ __forceinline__ void reg_uinv_right(double (&t)[RM], const double* U, const double* dinv,
                                               int R) {
#pragma unroll
    for (int j = 0; j < RM; ++j) {
        if (j < R) {
            t[j] *= dinv[j];
#pragma unroll
            for (int k = j + 1; k < RM; ++k) t[k] = fma(-t[j], U[j * RM + k], t[k]);
        }
    }
}

template <int RM, int NT, int ACC>
__global__ void bench(int R, int rows, long long* out, double* sink) {
    extern __shared__ double sm[];
    double* U = sm;                 // RM x RM
    double* d = U + RM * RM;        // RM
    double* w = d + RM;             // rows x (R+1)
    const int ld = R + 1;
    for (int e = threadIdx.x; e < RM * RM; e += NT) {
        const int i = e / RM, j = e % RM;
        U[e] = i == j ? 2.0 : (j > i ? 0.01 * (i + j) : 0.0);
    }
    for (int j = threadIdx.x; j < RM; j += NT) d[j] = 0.5;
    for (int e = threadIdx.x; e < rows * ld; e += NT) w[e] = 1.0 + (e % 5) * 0.1;
    __syncthreads();
    long long t0 = clock64();
    for (int li = threadIdx.x; li < rows; li += NT) {
        double x[RM];
#pragma unroll
        for (int j = 0; j < RM; ++j) x[j] = j < R ? w[li * ld + j] : 0.0;
        reg_uinv<RM, ACC>(x, U, d, R);
#pragma unroll
        for (int j = 0; j < RM; ++j)
            if (j < R) w[li * ld + j] = x[j];
    }
    __syncthreads();
    long long t1 = clock64();
    for (int li = threadIdx.x; li < rows; li += NT) {
        double x[RM];
#pragma unroll
        for (int j = 0; j < RM; ++j) x[j] = j < R ? w[li * ld + j] : 0.0;
        reg_uinv_right<RM>(x, U, d, R);
#pragma unroll
        for (int j = 0; j < RM; ++j)
            if (j < R) w[li * ld + j] = x[j];
    }
    __syncthreads();
    long long t2 = clock64();
    if (threadIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t1;
        sink[0] = w[0];
    }
}

template <int RM, int NT, int ACC>
void run(int R, int rows, long long* out, double* sink) {
    const size_t smem = (RM * RM + RM + rows * (R + 1)) * 8;
    cudaFuncSetAttribute(bench<RM, NT, ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long h[2] = {0, 0};
    for (int rep = 0; rep < 3; ++rep) bench<RM, NT, ACC><<<1, NT, smem>>>(R, rows, out, sink);
    cudaError_t e = cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("RM=%d NT=%d ACC=%d R=%d rows=%d: left %lld  right %lld cycles (%s)\n", RM, NT,
           ACC, R, rows, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    (void)e;
}

int main() {
    long long* out;
    double* sink;
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 64);
    run<32, 256, 2>(32, 64, out, sink);
    run<32, 256, 4>(32, 64, out, sink);
    run<32, 128, 4>(32, 64, out, sink);
    run<16, 256, 2>(16, 16, out, sink);
    run<32, 256, 4>(20, 32, out, sink);
    run<64, 128, 4>(64, 32, out, sink);
    run<64, 256, 4>(64, 32, out, sink);
    return 0;
}
