// Where do block_chol's ~500 cycles per pivot step go?  32 steps of
// (a) __syncthreads only, (b) + smem pivot read + rcp, (c) + the owned-entry
// loads / FMA / store of block_chol (KMAX = 2 / 4 at 512 / 256 threads).
#include <cstdio>
#include <cuda_runtime.h>

#include "device.cuh"

template <int NT, int MODE>
__global__ void __launch_bounds__(NT) k(long long* out, double* sink) {
    constexpr int R = 32, KMAX = (R * R + NT - 1) / NT;
    __shared__ double g[R * R];
    for (int e = threadIdx.x; e < R * R; e += NT) g[e] = (e % 33 == 0 ? 40.0 : 0.5);
    __syncthreads();
    int pa[KMAX], pb[KMAX];
    for (int kk = 0; kk < KMAX; ++kk) {
        const int e = threadIdx.x + kk * NT;
        const bool own = e < R * R && (e % R) >= (e / R);
        pa[kk] = own ? e / R : 1 << 20;
        pb[kk] = own ? e % R : 0;
    }
    double acc = 0.0;
    const long long t0 = clock64();
    for (int j = 0; j < R; ++j) {
        if (MODE >= 1) {
            const double d = g[j * R + j];
            double ga[KMAX], gb[KMAX], gab[KMAX];
            if (MODE >= 2) {
#pragma unroll
                for (int kk = 0; kk < KMAX; ++kk) {
                    const bool act = pa[kk] > j && pa[kk] < R;
                    ga[kk] = act ? g[j * R + pa[kk]] : 0.0;
                    gb[kk] = act ? g[j * R + pb[kk]] : 0.0;
                    gab[kk] = act ? g[pa[kk] * R + pb[kk]] : 0.0;
                }
            }
            const double inv = MODE == 3 ? __drcp_rn(d) : cpdb::rcp_nr(d);
            acc += inv;
            if (MODE >= 2) {
#pragma unroll
                for (int kk = 0; kk < KMAX; ++kk)
                    if (pa[kk] > j && pa[kk] < R)
                        g[pa[kk] * R + pb[kk]] = fma(-ga[kk] * inv, gb[kk], gab[kk]);
            }
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) *out = (t1 - t0) / R;
    sink[threadIdx.x] = acc + g[threadIdx.x % (R * R)];
}

int main() {
    long long* o;
    double* s;
    cudaMalloc(&o, 64);
    cudaMalloc(&s, 8192);
    long long h[7];
    k<512, 3><<<1, 512>>>(o + 6, s);
    k<512, 0><<<1, 512>>>(o + 0, s);
    k<512, 1><<<1, 512>>>(o + 1, s);
    k<512, 2><<<1, 512>>>(o + 2, s);
    k<256, 0><<<1, 256>>>(o + 3, s);
    k<256, 1><<<1, 256>>>(o + 4, s);
    k<256, 2><<<1, 256>>>(o + 5, s);
    cudaMemcpy(h, o, 56, cudaMemcpyDeviceToHost);
    printf("cycles/step  512 thr: sync %lld, +pivot/rcp %lld, +update %lld | 256 thr: %lld, %lld, %lld\n",
           h[0], h[1], h[2], h[3], h[4], h[5]);
    printf("512 thr, loads-first + __drcp_rn: %lld\n", h[6]);
    return 0;
}
