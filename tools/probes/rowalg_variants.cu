// Variant study for the small-matrix building blocks (cycles per call, 1 CTA).
#include <cstdio>
#include <cuda_runtime.h>

#include "rowalg.cuh"

using namespace cpdb;

#ifndef NTV
#define NTV 256
#endif
constexpr int NT = NTV;

// (A) block Cholesky, all loads of a step issued before its stores
template <int K>
__device__ bool chol_loadsfirst(double* g, int ld, int R, double* dinv) {
    int pa[K], pb[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int e = threadIdx.x + k * NT;
        const bool own = e < R * R && (e % R) >= (e / R);
        pa[k] = own ? e / R : 1 << 20;
        pb[k] = own ? e % R : 0;
    }
    for (int j = 0; j < R; ++j) {
        const double d = g[j * ld + j];
        const double inv = __drcp_rn(d);
        double ga[K], gb[K], gab[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const bool act = pa[k] > j && pa[k] < R;
            ga[k] = act ? g[j * ld + pa[k]] : 0.0;
            gb[k] = act ? g[j * ld + pb[k]] : 0.0;
            gab[k] = act ? g[pa[k] * ld + pb[k]] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (pa[k] > j && pa[k] < R) g[pa[k] * ld + pb[k]] = fma(-ga[k] * inv, gb[k], gab[k]);
        __syncthreads();
    }
    for (int j = threadIdx.x; j < R; j += NT) dinv[j] = sqrt(g[j * ld + j]);
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += NT) {
        const int i = e / R, k = e % R;
        g[i * ld + k] = k >= i ? g[i * ld + k] / dinv[i] : 0.0;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < R; j += NT) dinv[j] = 1.0 / g[j * ld + j];
    __syncthreads();
    return true;
}

// (B) one warp, columns in registers: lane l owns columns l (and l+32), the
// step loop is NOT unrolled -- column entries indexed by a runtime row live in
// smem, but each lane updates its own column only, loads first.
__device__ bool chol_warp(double* g, int ld, int R, double* dinv) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        for (int j = 0; j < R; ++j) {
            const double inv = __drcp_rn(g[j * ld + j]);
            // column l >= j+1 owned by this lane: update rows a in (j, l]
            for (int l = j + 1 + lane; l < R; l += 32) {
                const double gjl = g[j * ld + l] * inv;
                int a = j + 1;
                for (; a + 3 <= l; a += 4) {
                    const double x0 = g[j * ld + a], x1 = g[j * ld + a + 1];
                    const double x2 = g[j * ld + a + 2], x3 = g[j * ld + a + 3];
                    const double y0 = g[a * ld + l], y1 = g[(a + 1) * ld + l];
                    const double y2 = g[(a + 2) * ld + l], y3 = g[(a + 3) * ld + l];
                    g[a * ld + l] = fma(-x0, gjl, y0);
                    g[(a + 1) * ld + l] = fma(-x1, gjl, y1);
                    g[(a + 2) * ld + l] = fma(-x2, gjl, y2);
                    g[(a + 3) * ld + l] = fma(-x3, gjl, y3);
                }
                for (; a <= l; ++a) g[a * ld + l] = fma(-g[j * ld + a], gjl, g[a * ld + l]);
            }
            __syncwarp();
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < R; j += NT) dinv[j] = sqrt(g[j * ld + j]);
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += NT) {
        const int i = e / R, k = e % R;
        g[i * ld + k] = k >= i ? g[i * ld + k] / dinv[i] : 0.0;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < R; j += NT) dinv[j] = 1.0 / g[j * ld + j];
    __syncthreads();
    return true;
}

// (C) X = U^-1 by superdiagonals (R steps, entries of one diagonal in
// parallel), then rows <- rows X as independent dot products.
__device__ void tri_inverse(const double* u, int ldu, int R, double* x, int ldx) {
    for (int e = threadIdx.x; e < R * R; e += NT) {
        const int i = e / R, j = e % R;
        x[i * ldx + j] = i == j ? 1.0 / u[i * ldu + i] : 0.0;
    }
    __syncthreads();
    for (int dd = 1; dd < R; ++dd) {
        for (int i = threadIdx.x; i + dd < R; i += NT) {
            const int j = i + dd;
            double s0 = 0.0, s1 = 0.0;
            int k = i + 1;
            for (; k + 1 <= j; k += 2) {
                s0 = fma(u[i * ldu + k], x[k * ldx + j], s0);
                s1 = fma(u[i * ldu + k + 1], x[(k + 1) * ldx + j], s1);
            }
            if (k <= j) s0 = fma(u[i * ldu + k], x[k * ldx + j], s0);
            x[i * ldx + j] = -(s0 + s1) * x[i * ldx + i];
        }
        __syncthreads();
    }
}

// rows of w <- rows of w times upper X (independent outputs; out-of-place via tmp)
__device__ void rows_times_upper(double* w, int ld, int rows, const double* x, int ldx, int R,
                                 double* tmp) {
    for (int e = threadIdx.x; e < rows * R; e += NT) {
        const int li = e / R, j = e % R;
        double s0 = 0.0, s1 = 0.0;
        int p = 0;
        for (; p + 1 <= j; p += 2) {
            s0 = fma(w[li * ld + p], x[p * ldx + j], s0);
            s1 = fma(w[li * ld + p + 1], x[(p + 1) * ldx + j], s1);
        }
        if (p <= j) s0 = fma(w[li * ld + p], x[p * ldx + j], s0);
        tmp[li * ld + j] = s0 + s1;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * R; e += NT) w[(e / R) * ld + e % R] = tmp[(e / R) * ld + e % R];
}

// (D) gram with all owned entries interleaved in one row loop
template <int K>
__device__ void gram_interleaved(const double* w, int ld, int rows, int R, double* g) {
    int pa[K], pb[K];
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int e = threadIdx.x + k * NT;
        const bool own = e < R * R && (e % R) >= (e / R);
        pa[k] = own ? e / R : 0;
        pb[k] = own ? e % R : 0;
        acc[k] = own ? 0.0 : -1.0;
    }
    double s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = 0.0;
    for (int i = 0; i < rows; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) s[k] = fma(w[i * ld + pa[k]], w[i * ld + pb[k]], s[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (acc[k] == 0.0) {
            g[pa[k] * R + pb[k]] = s[k];
            g[pb[k] * R + pa[k]] = s[k];
        }
}

template <int K>
__global__ void bench(int R, int rows, long long* out, double* sink) {
    extern __shared__ double sm[];
    const int ld = R + 1;
    double* g = sm;
    double* d = g + R * R;
    double* w = d + 64;
    double* x = w + rows * ld;
    double* tmp = x + R * R;
    Owned<NT> own;
    own.init(R);
    auto fill = [&]() {
        for (int e = threadIdx.x; e < R * R; e += NT) {
            const int i = e / R, j = e % R;
            g[e] = (i == j) ? R + 1.0 : 1.0 / (1 + i + j);
        }
        for (int e = threadIdx.x; e < rows * ld; e += NT) w[e] = 1.0 + (e % 7) * 0.1;
        __syncthreads();
    };
    long long t[16];
    fill();
    t[0] = clock64();
    block_chol<NT>(g, R, R, d, own);
    t[1] = clock64();
    fill();
    t[2] = clock64();
    chol_loadsfirst<K>(g, R, R, d);
    t[3] = clock64();
    fill();
    t[4] = clock64();
    chol_warp(g, R, R, d);
    t[5] = clock64();
    // U now in g: substitution vs inverse+gemm
    t[6] = clock64();
    rows_uinv<NT>(w, ld, rows, g, R, d, R);
    __syncthreads();
    t[7] = clock64();
    tri_inverse(g, R, R, x, R);
    t[8] = clock64();
    rows_times_upper(w, ld, rows, x, R, R, tmp);
    __syncthreads();
    t[9] = clock64();
    gram_rows<NT>(w, ld, rows, g, R, own);
    __syncthreads();
    t[10] = clock64();
    gram_interleaved<K>(w, ld, rows, R, g);
    __syncthreads();
    t[11] = clock64();
    if (threadIdx.x == 0) {
        out[0] = t[1] - t[0];
        out[1] = t[3] - t[2];
        out[2] = t[5] - t[4];
        out[3] = t[7] - t[6];
        out[4] = t[8] - t[7];
        out[5] = t[9] - t[8];
        out[6] = t[10] - t[9];
        out[7] = t[11] - t[10];
        sink[0] = g[0] + w[0] + x[0];
    }
}

template <int K>
void run(int R, int rows, long long* out, double* sink) {
    const size_t smem = (2 * R * R + 64 + 2 * rows * (R + 1)) * 8;
    cudaFuncSetAttribute(bench<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long h[8];
    for (int rep = 0; rep < 3; ++rep) bench<K><<<1, NT, smem>>>(R, rows, out, sink);
    cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("R=%2d rows=%3d chol %6lld loadsfirst %6lld warp %6lld | uinv %6lld inv %6lld gemm %6lld"
           " | gram %6lld interleaved %6lld\n",
           R, rows, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
}

int main() {
    long long* out;
    double* sink;
    cudaMalloc(&out, 128);
    cudaMalloc(&sink, 64);
    run<1>(10, 13, out, sink);
    run<1>(16, 16, out, sink);
    run<2>(20, 32, out, sink);
    run<4>(32, 64, out, sink);
    run<16>(64, 32, out, sink);
    run<4>(32, 128, out, sink);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
