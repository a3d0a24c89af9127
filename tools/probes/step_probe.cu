// Latency of one Cholesky pivot step's critical chain (one warp):
// LDS pivot -> reciprocal -> FMA -> STS -> __syncwarp, 64 dependent steps.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_fast(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    // two Newton steps: r = r (2 - d r)
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

template <int MODE>
__global__ void k(double* out, long long* cyc) {
    __shared__ double s[64];
    const int l = threadIdx.x;
    s[l] = 1.0 + l * 1e-3;
    __syncwarp();
    long long t0 = clock64();
    double acc = 0.0;
    for (int j = 0; j < 62; ++j) {
        const double d = s[j];
        double inv;
        if (MODE == 0) inv = __drcp_rn(d);
        else if (MODE == 1) inv = 1.0 / d;
        else if (MODE == 2) inv = rcp_fast(d);
        else inv = d;  // no reciprocal
        const double v = fma(-inv, s[j + 1], 2.0);
        if (l == (j + 1) % 32) s[j + 1] = v;
        acc += v;
        __syncwarp();
    }
    long long t1 = clock64();
    if (l == 0) *cyc = (t1 - t0) / 62;
    out[l] = acc;
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 256);
    cudaMalloc(&c, 32);
    k<0><<<1, 32>>>(o, c);
    k<1><<<1, 32>>>(o, c + 1);
    k<2><<<1, 32>>>(o, c + 2);
    k<3><<<1, 32>>>(o, c + 3);
    long long h[4];
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles/step: drcp_rn %lld  div %lld  rcp.approx+2NR %lld  none %lld\n", h[0], h[1],
           h[2], h[3]);
    return 0;
}
