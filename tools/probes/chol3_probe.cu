// Cholesky latency inside one 512-thread CTA (the mode-update kernels' block
// size): block_chol (one block barrier per step) vs reg_chol (register team,
// named barrier) vs warp_chol (one warp, columns in registers, no block
// barriers).  clock64 cycles per factorisation (100 repetitions); all three
// must agree bit for bit.
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#include "rowalg.cuh"

using namespace cpdb;

// warp Cholesky (evaluated, not used by the library: see rowalg.cuh chol)
// Same factorisation and arithmetic as block_chol (bit-identical U) for
// R <= 32 in ONE warp with no block barriers: lane b keeps column b of the
// trailing matrix (G[a][b], a <= b) in registers.  Step j: the pivot comes
// from lane j by shuffle, every lane publishes w[b] = -G[j][b] / G[j][j]
// (as block_chol: (-G[j][b]) * rcp) to a 32-entry smem row (two rows,
// alternating, so one __syncwarp per step suffices), and each lane updates
// its column, G[a][b] += w[a] G[j][b], from broadcast reads -- row j+1
// first, so the next pivot's shuffle / reciprocal overlap the rest.
// Entries below the diagonal (a > b) are updated too and never read back
// (no predicates in the inner loop).  The other threads wait at the closing
// barrier.
template <int NT, int RM>
__device__ bool warp_chol(double* g, int ld, int R) {
    static_assert(RM <= 32, "warp_chol: one column per lane");
    __shared__ __align__(16) double w[2][32];  // double-buffered: one __syncwarp per step
    __shared__ int bad;
    // a warp index the compiler sees as warp-uniform (a plain threadIdx test
    // makes every shuffle / __syncwarp below take the divergent-path lowering)
    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
    if (warp == 0) {
        const int b = threadIdx.x & 31;
        double e[RM];
#pragma unroll
        for (int a = 0; a < RM; ++a) e[a] = (a <= b && b < R) ? g[a * ld + b] : 0.0;
        // software-pipelined: step j first finishes row j+1 (the next pivot
        // and multipliers) and publishes it, then updates the rest of the
        // column while the next step's chain is in flight
        double gb = e[0];
        double d = __shfl_sync(0xffffffffu, gb, 0);
        bool ok = d > 0.0;
        w[0][b] = -gb * rcp_nr(d);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < RM; ++j) {
            if (j < R) {
                double gbn = 0.0;
                if (j + 1 < RM && j + 1 < R) {
                    e[j + 1] = fma(w[j & 1][j + 1], gb, e[j + 1]);
                    gbn = e[j + 1];
                    const double dn = __shfl_sync(0xffffffffu, gbn, j + 1);
                    ok = ok && dn > 0.0;  // warp-uniform
                    w[(j + 1) & 1][b] = -gbn * rcp_nr(dn);
                }
#pragma unroll
                for (int a = j + 2; a < RM; ++a) e[a] = fma(w[j & 1][a], gb, e[a]);
                gb = gbn;
                __syncwarp();
            }
        }
        // U[a][b] = G^(a)[a][b] * rsqrt(G^(a)[a][a]) (block_chol's final
        // scaling): lane a computes its diagonal's rsqrt once and shares it
        double diag = 0.0;
#pragma unroll
        for (int a = 0; a < RM; ++a) diag = a == b ? e[a] : diag;
        w[RM & 1][b] = b < R ? rsqrt(diag) : 0.0;
        __syncwarp();
#pragma unroll
        for (int a = 0; a < RM; ++a)
            if (a < R && b < R) g[a * ld + b] = a <= b ? e[a] * w[RM & 1][a] : 0.0;
        if (b == 0) bad = ok ? 0 : 1;
    }
    __syncthreads();
    return bad == 0;
}


template <int RM, int MODE>
__global__ void __launch_bounds__(512) k(const double* g0, int R, long long* cyc, double* out) {
    __shared__ double g[RM * RM];
    long long t0 = 0;
    for (int rep = 0; rep < 101; ++rep) {
        if (rep == 1) t0 = clock64();
        for (int e = threadIdx.x; e < R * R; e += 512) g[e] = g0[e];
        __syncthreads();
        if (MODE == 0) block_chol<512, (RM * RM + 511) / 512>(g, R, R);
        else if (MODE == 1) reg_chol<512, RM>(g, R, R);
        else warp_chol<512, RM>(g, R, R);
        __syncthreads();
    }
    if (threadIdx.x == 0) *cyc = (clock64() - t0) / 100;
    for (int e = threadIdx.x; e < R * R; e += 512) out[e] = g[e];
}

template <int RM>
void run(int R) {
    double* h = new double[R * R];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) h[i * R + j] = (i == j ? R : 0.0) + 1.0 / (1 + i + j);
    double *g, *o[3];
    long long* c;
    cudaMalloc(&g, R * R * 8);
    for (auto& p : o) cudaMalloc(&p, R * R * 8);
    cudaMalloc(&c, 24);
    cudaMemcpy(g, h, R * R * 8, cudaMemcpyHostToDevice);
    k<RM, 0><<<1, 512>>>(g, R, c, o[0]);
    k<RM, 1><<<1, 512>>>(g, R, c + 1, o[1]);
    k<RM, 2><<<1, 512>>>(g, R, c + 2, o[2]);
    long long hc[3];
    static double a[3][4096];
    cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
    for (int v = 0; v < 3; ++v) cudaMemcpy(a[v], o[v], R * R * 8, cudaMemcpyDeviceToHost);
    printf("R=%2d block %6lld  reg %6lld  warp %6lld cycles  reg==block %d  warp==block %d  (%s)\n",
           R, hc[0], hc[1], hc[2], memcmp(a[0], a[1], R * R * 8) == 0,
           memcmp(a[0], a[2], R * R * 8) == 0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<8>(8);
    run<16>(10);
    run<16>(16);
    run<32>(20);
    run<32>(32);
    return 0;
}
