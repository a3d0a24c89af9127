// Cholesky of an R x R SPD matrix in one CTA: block-parallel owned entries
// (rowalg.cuh block_chol) vs one warp with columns in registers.
#include <cstdio>
#include <cuda_runtime.h>

#include "rowalg.cuh"

using namespace cpdb;

// one warp; lane l holds column l (and l+32); row j of U broadcast through smem
template <int RM>
__device__ bool warp_chol_cols(double* g, int R, double* rowbuf) {
    constexpr int C = RM > 32 ? 2 : 1;
    const int lane = threadIdx.x & 31;
    double col[C][RM];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int l = lane + 32 * c;
#pragma unroll
        for (int a = 0; a < RM; ++a) col[c][a] = (l < R && a < R) ? g[a * R + l] : 0.0;
    }
    bool ok = true;
#pragma unroll
    for (int j = 0; j < RM; ++j) {
        if (j < R) {
            const double d = __shfl_sync(0xffffffffu, col[j / 32][j], j % 32);
            ok = ok && d > 0.0;
            const double rs = rsqrt(d > 0.0 ? d : 1.0);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int l = lane + 32 * c;
                if (l >= j) {
                    col[c][j] *= rs;  // U[j][l]
                    rowbuf[l] = col[c][j];
                }
            }
            __syncwarp();
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int l = lane + 32 * c;
                const double ujl = col[c][j];
#pragma unroll
                for (int a = j + 1; a < RM; ++a)
                    if (a <= l) col[c][a] = fma(-rowbuf[a], ujl, col[c][a]);
            }
            __syncwarp();
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int l = lane + 32 * c;
        if (l < R) {
#pragma unroll
            for (int a = 0; a < RM; ++a)
                if (a < R) g[a * R + l] = a <= l ? col[c][a] : 0.0;
        }
    }
    return ok;
}

template <int RM, int NT>
__global__ void bench(int R, long long* out, double* sink) {
    __shared__ double g[64 * 64];
    __shared__ double rowbuf[64];
    auto fill = [&]() {
        for (int e = threadIdx.x; e < R * R; e += NT) {
            const int i = e / R, j = e % R;
            g[e] = (i == j) ? R + 1.0 : 1.0 / (1 + i + j);
        }
        __syncthreads();
    };
    fill();
    long long t0 = clock64();
    block_chol<NT, (RM * RM + NT - 1) / NT>(g, R, R);
    long long t1 = clock64();
    const double ref = g[R + 1];
    fill();
    long long t2 = clock64();
    if (threadIdx.x < 32) warp_chol_cols<RM>(g, R, rowbuf);
    __syncthreads();
    long long t3 = clock64();
    if (threadIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t3 - t2;
        sink[0] = g[R + 1] - ref;
    }
}

template <int RM, int NT>
void run(int R, long long* out, double* sink) {
    long long h[2];
    double diff;
    for (int rep = 0; rep < 3; ++rep) bench<RM, NT><<<1, NT>>>(R, out, sink);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(&diff, sink, 8, cudaMemcpyDeviceToHost);
    printf("R=%d NT=%d: block %lld  warp-cols %lld cycles  (U[1][1] diff %.2e) %s\n", R, NT, h[0],
           h[1], diff, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long* out;
    double* sink;
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 64);
    run<16, 512>(16, out, sink);
    run<32, 512>(20, out, sink);
    run<32, 512>(32, out, sink);
    run<64, 512>(64, out, sink);
    return 0;
}
