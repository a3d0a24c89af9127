// Wide ranks (R > 64): the mode-update tail in rank-generic kernels.
//
// The tuned kernels (zqr.cu, cluster.cu, smallmat.cu, finish.cu) keep a whole
// R x R triangle and R-wide rows in shared memory / registers and are
// instantiated for R <= 64 -- the BASELINE configs.  The reference accepts any
// rank up to the smallest extent (solvers.hpp:221-224), so beyond 64 the same
// launch interfaces (ZqrArgs / FinishArgs, kernels.hpp) are served by the
// kernels below, which follow the reference's own algorithm step by step:
//   Z = KhatriRao(R_k, k != n)                        tensor.hpp:343-368
//   Q0, R0 = thin_qr(Z)        Householder            linalg.hpp:39-99
//   A_hat  = V R0^-T           row-wise back substitution   linalg.hpp:192-216
//   lambda, A_n = normalize_columns(A_hat)            linalg.hpp:225-242
//   Q_n, R_n = thin_qr(A_n)                           factor_state.hpp:42-47
//   fitness_fast_qr                                   kruskal.hpp:109-128
// The Householder QR is a cooperative multi-CTA kernel: rows are split across
// the grid, each reflector costs one grid barrier in the factorisation and one
// in the accumulation of Q, every sum runs in a fixed order
// (deterministic), and the conventions are the reference's (alpha = -sign
// ||x||, zero columns skipped, nonnegative diag(R) by a final sign flip).
#include <cooperative_groups.h>

#include <algorithm>

#include "device.cuh"
#include "kernels.hpp"
#include "prims.hpp"
#include "rowalg.cuh"

namespace cg = cooperative_groups;

namespace cpdb {
namespace {

constexpr int kHT = 512;        // threads per CTA
constexpr int kHW = kHT / 32;   // warps = row groups
constexpr int kMaxWide = 1024;  // widest supported matrix (columns)

// Z rows in the natural order of the final Y: digits over the other modes in
// ascending mode order, the last fastest (ZqrArgs, kernels.hpp).
__global__ void kr_natural_kernel(ZqrArgs a, double* z) {
    const uint32_t R = a.R;
    const uint64_t n = a.zrows * R;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t rem = e / R;
        const uint32_t j = uint32_t(e % R);
        double p = 1.0;
        for (int k = int(a.nm) - 1; k >= 0; --k) {
            const uint64_t d = rem % R;
            rem /= R;
            p = __dmul_rn(p, a.rmats[k][d * R + j]);
        }
        z[e] = p;
    }
}

struct HhArgs {
    double* w;        // m x n, row-major; in: A, out: reflectors below the diagonal
    double* q;        // m x n out
    double* r;        // n x n out
    double* scratch;  // hh_scratch_doubles(n, grid)
    uint64_t m;
    uint32_t n;
};

__host__ __device__ inline size_t hh_scratch_doubles(uint32_t n, int grid) {
    return size_t(2) * grid * n + size_t(2) * n;
}

// sum of x over the CTA in a fixed order (warp tree, then warps in order)
__device__ double cta_sum(double x, double* red) {
    x = warp_sum(x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < kHW; ++w) t += red[w];
    return t;
}

// d[j] = sum over this CTA's rows i in [lo, hi) of vcoef(i) * mat[i][j], for
// j in [j0, n): warp g takes rows lo+g, lo+g+8, ... and lanes take 32
// consecutive columns; the warps' partials are added in warp order.
constexpr int kHU = 8;  // rows in flight per lane (the loads are L2 hits: latency-bound)

template <class V>
__device__ void cta_col_dots(const double* mat, uint32_t n, uint64_t lo, uint64_t hi, uint32_t j0,
                             V vcoef, double* part /*[kHW][n]*/, double* out /*[n]*/) {
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t jb = (j0 / 32) * 32; jb < n; jb += 32) {
        const uint32_t j = jb + lane;
        if (j >= n) continue;
        double d[kHU];
#pragma unroll
        for (int u = 0; u < kHU; ++u) d[u] = 0.0;
        for (uint64_t i = lo + g; i < hi; i += uint64_t(kHU) * kHW) {
            double v[kHU], x[kHU];
#pragma unroll
            for (int u = 0; u < kHU; ++u) {
                const uint64_t r = i + uint64_t(u) * kHW;
                v[u] = r < hi ? vcoef(r) : 0.0;
                x[u] = r < hi ? mat[r * n + j] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kHU; ++u) d[u] = fma(v[u], x[u], d[u]);
        }
        part[g * n + j] = ((d[0] + d[1]) + (d[2] + d[3])) + ((d[4] + d[5]) + (d[6] + d[7]));
    }
    __syncthreads();
    for (uint32_t j = j0 + threadIdx.x; j < n; j += kHT) {
        double t = 0.0;
        for (int w = 0; w < kHW; ++w) t += part[w * n + j];
        out[j] = t;
    }
}

// mat[i][j] -= dsh[j] * vcoef(i) for this CTA's rows i in [lo, hi) and the
// columns j >= j0: kHU rows per lane in flight.
template <class V>
__device__ void cta_rank1_update(double* mat, uint32_t n, uint64_t lo, uint64_t hi, uint32_t j0,
                                 V vcoef, const double* dsh) {
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint64_t i = lo + g; i < hi; i += uint64_t(kHU) * kHW) {
        double v[kHU];
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
            const uint64_t r = i + uint64_t(u) * kHW;
            v[u] = r < hi ? vcoef(r) : 0.0;
        }
        for (uint32_t j = (j0 / 32) * 32 + lane; j < n; j += 32) {
            if (j < j0) continue;
            double x[kHU];
#pragma unroll
            for (int u = 0; u < kHU; ++u) {
                const uint64_t r = i + uint64_t(u) * kHW;
                x[u] = r < hi ? mat[r * n + j] : 0.0;
            }
            const double dj = dsh[j];
#pragma unroll
            for (int u = 0; u < kHU; ++u) {
                const uint64_t r = i + uint64_t(u) * kHW;
                if (r < hi) mat[r * n + j] = fma(-dj, v[u], x[u]);
            }
        }
    }
}

// out[j] = sum over the grid's CTAs b of pd[b][j], j in [j0, n), in a fixed
// order: up to 8 threads per column take interleaved b with four loads in
// flight each (the partials come from L2), then the column's threads are
// added in order.  part: kHW x n shared scratch.
__device__ void grid_partials_sum(const double* pd, int G, uint32_t n, uint32_t j0, double* part,
                                  double* out) {
    const uint32_t nc = n - j0;
    uint32_t parts = kHT / nc;
    parts = parts < 1 ? 1 : parts > uint32_t(kHW) ? uint32_t(kHW) : parts;
    if (parts > uint32_t(G)) parts = uint32_t(G);
    for (uint32_t e = threadIdx.x; e < nc * parts; e += kHT) {
        const uint32_t j = j0 + e % nc, sub = e / nc;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int b = int(sub);
        const int st = int(parts);
        for (; b + 3 * st < G; b += 4 * st) {
            s0 += pd[size_t(b) * n + j];
            s1 += pd[size_t(b + st) * n + j];
            s2 += pd[size_t(b + 2 * st) * n + j];
            s3 += pd[size_t(b + 3 * st) * n + j];
        }
        for (; b < G; b += st) s0 += pd[size_t(b) * n + j];
        part[sub * n + j] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
    for (uint32_t j = j0 + threadIdx.x; j < n; j += kHT) {
        double t = 0.0;
        for (uint32_t sub = 0; sub < parts; ++sub) t += part[sub * n + j];
        out[j] = t;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kHT) hh_coop_kernel(HhArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    __shared__ double red[kHW];
    const uint32_t n = a.n;
    const uint64_t m = a.m;
    double* betas = sm;           // n
    double* vdiag = betas + n;    // n: v_k[0] = w_kk - alpha
    double* sgn = vdiag + n;      // n: -1 where R(k,k) < 0
    double* dsh = sgn + n;        // n
    double* part = dsh + n;       // kHW x n
    const int G = int(gridDim.x), c = int(blockIdx.x);
    const uint64_t chunk = (m + G - 1) / G;
    const uint64_t row0 = uint64_t(c) * chunk < m ? uint64_t(c) * chunk : m;
    const uint64_t row1 = row0 + chunk < m ? row0 + chunk : m;
    double* pd = a.scratch;  // [2][G][n]: per-CTA partial products, double-buffered
    double* prow = a.scratch + size_t(2) * G * n;  // [2][n]: row k as it was before its update
    double* w = a.w;

    // ---- factorisation: reflector k from column k, applied to columns > k.
    // One grid barrier per reflector: the products s_j = sum_{i > k} w_ik w_ij
    // (j >= k; s_k is the column's tail norm) need nothing from the
    // reflector's head, so each CTA publishes them for its rows first; after
    // the barrier every CTA knows ||x||, alpha, v_0 = w_kk - alpha, beta and
    // d_j = v_0 w_kj + s_j, and updates its own rows.
    for (uint32_t k = 0; k < n; ++k) {
        const uint64_t lo1 = row0 > k ? row0 : uint64_t(k) + 1;  // rows below the diagonal
        auto wk = [&](uint64_t i) { return w[i * n + k]; };
        double* pdk = pd + size_t(k & 1) * G * n;
        cta_col_dots(w, n, lo1, row1, k, wk, part, pdk + size_t(c) * n);
        // (its owner updates row k right after the barrier: the others read
        // this copy)
        double* prk = prow + size_t(k & 1) * n;
        if (k >= row0 && k < row1)
            for (uint32_t j = k + threadIdx.x; j < n; j += kHT) prk[j] = w[uint64_t(k) * n + j];
        grid.sync();
        grid_partials_sum(pdk, G, n, k, part, dsh);
        const double tail = dsh[k];
        const double wkk = prk[k];
        const double norm = sqrt(fma(wkk, wkk, tail));
        if (norm == 0.0) {  // zero column: R(k,k) stays 0 (uniform over the grid)
            if (threadIdx.x == 0) {
                betas[k] = 0.0;
                vdiag[k] = 0.0;
                sgn[k] = 1.0;
            }
            __syncthreads();
            continue;
        }
        const double alpha = wkk >= 0.0 ? -norm : norm;
        const double v0 = wkk - alpha;
        const double beta = 2.0 / fma(v0, v0, tail);
        if (threadIdx.x == 0) {
            betas[k] = beta;
            vdiag[k] = v0;
            sgn[k] = alpha < 0.0 ? -1.0 : 1.0;
        }
        // d_j = v_0 w_kj + s_j, scaled by beta (row k is final since the
        // previous reflector's update, before this barrier)
        __syncthreads();
        for (uint32_t j = k + 1 + threadIdx.x; j < n; j += kHT)
            dsh[j] = fma(v0, prk[j], dsh[j]) * beta;
        __syncthreads();
        // w_ij -= (beta d_j) v_i on this CTA's rows; column k keeps v below
        // the diagonal and alpha on it
        {
            const uint64_t lo = row0 > k ? row0 : uint64_t(k);
            auto vco = [&](uint64_t i) { return i == k ? v0 : w[i * n + k]; };
            cta_rank1_update(w, n, lo, row1, k + 1, vco, dsh);
        }
        __syncthreads();
        if (threadIdx.x == 0 && k >= row0 && k < row1) w[uint64_t(k) * n + k] = alpha;
        __syncthreads();
    }
    grid.sync();
    // ---- R (upper triangle, rows flipped to a nonnegative diagonal)
    for (uint64_t e = uint64_t(c) * kHT + threadIdx.x; e < uint64_t(n) * n; e += uint64_t(G) * kHT) {
        const uint32_t i = uint32_t(e / n), j = uint32_t(e % n);
        a.r[e] = j >= i ? w[e] * sgn[i] : 0.0;
    }
    // ---- Q = H_0 ... H_{n-1} [I; 0], reflectors applied in descending order
    double* q = a.q;
    for (uint64_t e = row0 * n + threadIdx.x; e < row1 * n; e += kHT)
        q[e] = (e / n == e % n) ? 1.0 : 0.0;
    __syncthreads();
    uint32_t it = 0;  // applied reflectors: parity of the partials buffer
    for (int k = int(n) - 1; k >= 0; --k) {
        const double beta = betas[k];
        if (beta == 0.0) continue;
        const double v0 = vdiag[k];
        const uint64_t lo = row0 > uint64_t(k) ? row0 : uint64_t(k);
        auto vco = [&](uint64_t i) { return i == uint64_t(k) ? v0 : w[i * n + k]; };
        double* pdk = pd + size_t(it++ & 1) * G * n;
        // (columns j < k of rows >= k are still zero)
        cta_col_dots(q, n, lo, row1, uint32_t(k), vco, part, pdk + size_t(c) * n);
        grid.sync();
        grid_partials_sum(pdk, G, n, uint32_t(k), part, dsh);
        for (uint32_t j = uint32_t(k) + threadIdx.x; j < n; j += kHT) dsh[j] *= beta;
        __syncthreads();
        cta_rank1_update(q, n, lo, row1, uint32_t(k), vco, dsh);
        __syncthreads();
    }
    for (uint64_t e = row0 * n + threadIdx.x; e < row1 * n; e += kHT)
        if (sgn[e % n] < 0.0) q[e] = -q[e];
}

int wide_sms() {
    static const int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 1;
    }();
    return n;
}

// one CTA per SM at most (cooperative launch: all CTAs co-resident)
cudaError_t hh_launch(const HhArgs& a, cudaStream_t s) {
    const int sms = wide_sms();
    if (a.n > uint32_t(kMaxWide)) return cudaErrorInvalidValue;
    const size_t smem = (size_t(4) + kHW) * a.n * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(hh_coop_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    // (at least 128 rows per CTA: a barrier costs more than a few rows)
    int grid = int(std::min<uint64_t>(uint64_t(sms), (a.m + 127) / 128));
    grid = std::max(grid, 1);
    HhArgs args = a;
    void* params[] = {&args};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(hh_coop_kernel), dim3(grid),
                                       dim3(kHT), params, smem, s);
}

// A_hat = V R0^-T (x R0^T = v per row): warp per row, the row in shared
// memory, back substitution with lane-split dot products.  status gets
// 1 | col << 8 for a ~0 diagonal entry (same test as the reference).
__global__ void __launch_bounds__(kHT)
solve_rows_wide_kernel(const double* v, const double* r0, uint32_t n, uint64_t rows, double* x,
                       int* status) {
    extern __shared__ double sm[];
    __shared__ int bad;
    if (threadIdx.x == 0) {
        double mx = 0.0;
        for (uint32_t i = 0; i < n; ++i) mx = fmax(mx, fabs(r0[size_t(i) * n + i]));
        bad = -1;
        for (uint32_t i = 0; i < n; ++i)
            if (fabs(r0[size_t(i) * n + i]) <= 1e-14 * mx) {
                bad = int(i);
                break;
            }
        if (bad >= 0 && blockIdx.x == 0) atomicOr(status, 1 | (bad << 8));
    }
    __syncthreads();
    if (bad >= 0) return;
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* xr = sm + size_t(g) * n;
    for (uint64_t row = uint64_t(blockIdx.x) * kHW + g; row < rows; row += uint64_t(gridDim.x) * kHW) {
        for (uint32_t j = lane; j < n; j += 32) xr[j] = v[row * n + j];
        __syncwarp();
        for (int c = int(n) - 1; c >= 0; --c) {
            double s = 0.0;
            for (uint32_t j = uint32_t(c) + 1 + lane; j < n; j += 32)
                s = fma(xr[j], r0[size_t(c) * n + j], s);
            s = warp_sum(s);
            if (lane == 0) xr[c] = (xr[c] - s) / r0[size_t(c) * n + c];
            __syncwarp();
        }
        for (uint32_t j = lane; j < n; j += 32) x[row * n + j] = xr[j];
        __syncwarp();
    }
}

// fitness_fast_qr (kruskal.hpp:109-128) across the grid: block b sums
// <V_fit, A_hat R0^T> over its rows (warp per row, lanes over the columns);
// the last kernel adds the blocks in order and forms ||K||^2 and the fitness.
constexpr int kFitBlocks = 148;

__global__ void __launch_bounds__(kHT)
fit_xk_kernel(const double* v, const double* ah, const double* r0, uint64_t rows, uint32_t r,
              double* partial) {
    __shared__ double red[kHW];
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double s = 0.0;
    for (uint64_t i = uint64_t(blockIdx.x) * kHW + g; i < rows; i += uint64_t(gridDim.x) * kHW)
        for (uint32_t j = lane; j < r; j += 32) {
            double m = 0.0;
            for (uint32_t p = j; p < r; ++p) m = fma(ah[i * r + p], r0[size_t(j) * r + p], m);
            s = fma(v[i * r + j], m, s);
        }
    s = cta_sum(s, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kHT)
fit_final_kernel(double nx2, const double* partial, int nb, const double* r0, const double* rn,
                 const double* lam, uint32_t r, double* fit_out) {
    __shared__ double red[kHW];
    double k = 0.0;
    for (uint32_t e = threadIdx.x; e < r * r; e += kHT) {
        const uint32_t i = e / r, j = e % r, top = i < j ? i : j;
        double g0 = 0.0, gn = 0.0;
        for (uint32_t p = 0; p <= top; ++p) {
            g0 = fma(r0[size_t(p) * r + i], r0[size_t(p) * r + j], g0);
            gn = fma(rn[size_t(p) * r + i], rn[size_t(p) * r + j], gn);
        }
        k += g0 * lam[i] * gn * lam[j];
    }
    k = cta_sum(k, red);
    if (threadIdx.x == 0) {
        double xk = 0.0;
        for (int b = 0; b < nb; ++b) xk += partial[b];
        const double raw = nx2 - 2.0 * xk + k;
        const double rad = raw < 0.0 ? 0.0 : raw;
        fit_out[0] = 1.0 - sqrt(rad) / sqrt(nx2);
        fit_out[1] = raw;
    }
}


// ---------------------------------------------------------------- solve_spd, n > 64
// linalg.hpp:132-185 with the factor in global memory: symmetry check,
// Cholesky G = U^T U (right-looking, one CTA), one ridge retry with delta =
// 1e-12 trace / n, then X = RHS U^-1 U^-T row by row.  u: n x n (U), ut: n x n
// (U^T, so both substitutions read contiguous rows).
__global__ void __launch_bounds__(512)
spd_factor_wide_kernel(const double* g, uint32_t n, double* u, double* ut, int* status, int* reg) {
    __shared__ double red[32];
    double mabs = 0.0, masym = 0.0;
    for (uint32_t e = threadIdx.x; e < n * n; e += 512) {
        const uint32_t i = e / n, j = e % n;
        mabs = fmax(mabs, fabs(g[e]));
        masym = fmax(masym, fabs(g[e] - g[j * n + i]));
    }
    mabs = block_max<512>(mabs, red);
    masym = block_max<512>(masym, red);
    if (masym > 1e-10 * mabs) {
        if (threadIdx.x == 0) *status = 5;
        return;
    }
    int used = 0;
    bool ok = false;
    for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
        double delta = 0.0;
        if (attempt == 1) {
            double tr = 0.0;
            for (uint32_t i = 0; i < n; ++i) tr += g[i * n + i];
            delta = 1e-12 * tr / double(n);
            used = 1;
        }
        for (uint32_t e = threadIdx.x; e < n * n; e += 512)
            u[e] = g[e] + ((e / n == e % n) ? delta : 0.0);
        __syncthreads();
        ok = true;
        for (uint32_t j = 0; j < n; ++j) {
            const double d = u[j * n + j];
            if (!(d > 0.0)) {  // uniform: every thread read the same d
                ok = false;
                break;
            }
            const double root = sqrt(d);
            __syncthreads();
            for (uint32_t b = j + threadIdx.x; b < n; b += 512)
                u[j * n + b] = b == j ? root : u[j * n + b] / root;
            __syncthreads();
            const uint32_t t = n - j - 1;  // trailing block (a, b > j, a <= b)
            for (uint32_t e = threadIdx.x; e < t * t; e += 512) {
                const uint32_t a = j + 1 + e / t, b = j + 1 + e % t;
                if (a <= b) u[a * n + b] = fma(-u[j * n + a], u[j * n + b], u[a * n + b]);
            }
            __syncthreads();
        }
        __syncthreads();
    }
    for (uint32_t e = threadIdx.x; e < n * n; e += 512) {
        const uint32_t i = e / n, j = e % n;
        const double v = j >= i ? u[e] : 0.0;
        ut[j * n + i] = v;
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < n * n; e += 512)
        if (e % n < e / n) u[e] = 0.0;
    if (threadIdx.x == 0) {
        *status = ok ? 0 : 4;
        *reg = used;
    }
}

__global__ void __launch_bounds__(kHT)
spd_rows_wide_kernel(const double* u, const double* ut, uint32_t n, double* x, uint64_t rows,
                     const int* status) {
    extern __shared__ double sm[];
    if (*status) return;
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* xr = sm + size_t(g) * n;
    for (uint64_t row = uint64_t(blockIdx.x) * kHW + g; row < rows; row += uint64_t(gridDim.x) * kHW) {
        for (uint32_t j = lane; j < n; j += 32) xr[j] = x[row * n + j];
        __syncwarp();
        // w U = rhs  (w L^T = rhs, L = U^T): forward, column c of U = row c of U^T
        for (uint32_t c = 0; c < n; ++c) {
            double s = 0.0;
            for (uint32_t j = lane; j < c; j += 32) s = fma(xr[j], ut[size_t(c) * n + j], s);
            s = warp_sum(s);
            if (lane == 0) xr[c] = (xr[c] - s) / ut[size_t(c) * n + c];
            __syncwarp();
        }
        // x U^T = w  (x L = w): backward, L[j][c] = U[c][j]
        for (int c = int(n) - 1; c >= 0; --c) {
            double s = 0.0;
            for (uint32_t j = uint32_t(c) + 1 + lane; j < n; j += 32)
                s = fma(xr[j], u[size_t(c) * n + j], s);
            s = warp_sum(s);
            if (lane == 0) xr[c] = (xr[c] - s) / u[size_t(c) * n + c];
            __syncwarp();
        }
        for (uint32_t j = lane; j < n; j += 32) x[row * n + j] = xr[j];
        __syncwarp();
    }
}

}  // namespace

bool wide_rank(uint32_t R) { return R > 64; }

size_t zqr_wide_work_doubles(uint32_t R) { return hh_scratch_doubles(R, wide_sms()) + 8; }

size_t finish_wide_scratch_doubles(uint64_t I, uint32_t R) {
    return 2 * I * R + hh_scratch_doubles(R, wide_sms()) + kFitBlocks + 16;
}

// Z into q1 (the kernel's working copy), Householder in place, Q0 / R0 out.
cudaError_t launch_zqr_wide(const ZqrArgs& a, cudaStream_t s) {
    const uint64_t n = a.zrows * a.R;
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 8192));
    kr_natural_kernel<<<grid, 256, 0, s>>>(a, a.q1);
    HhArgs h{a.q1, a.q0, a.r0, a.work, a.zrows, a.R};
    return hh_launch(h, s);
}

cudaError_t launch_finish_wide(const FinishArgs& a, cudaStream_t s) {
    const int sms = wide_sms();
    if (a.scratch == nullptr) return cudaErrorInvalidValue;
    const uint64_t I = a.I;
    const uint32_t R = a.R;
    double* ahat = a.scratch;           // I x R
    double* w = ahat + I * R;           // I x R: Householder working copy of A_n
    double* hs = w + I * R;             // hh scratch
    double* out4 = hs + hh_scratch_doubles(R, sms);
    if (!a.init) {
        if (a.nsplit != 1) return cudaErrorInvalidValue;
        const unsigned grid = unsigned(std::min<uint64_t>((I + kHW - 1) / kHW, 1024));
        const size_t smem = size_t(kHW) * R * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(solve_rows_wide_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
        solve_rows_wide_kernel<<<grid, kHT, smem, s>>>(a.vpart, a.r0, R, I, ahat, a.status);
        e = cudaMemcpyAsync(a.a_out, ahat, I * R * sizeof(double), cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return e;
        e = normalize_exact(a.a_out, I, R, a.lambda, s);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaMemcpyAsync(w, a.a_out, I * R * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    HhArgs h{w, a.q_out, a.r_out, hs, I, R};
    e = hh_launch(h, s);
    if (e != cudaSuccess) return e;
    e = pack_q(a.q_out, a.qp_out, uint32_t(I), R, s);
    if (e != cudaSuccess) return e;
    if (a.fitness && !a.init) {
        const double* vfit = a.dual ? a.vfitpart : a.vpart;
        const int nb = int(std::min<uint64_t>(kFitBlocks, (I + kHW - 1) / kHW));
        fit_xk_kernel<<<nb, kHT, 0, s>>>(vfit, ahat, a.r0, I, R, out4);
        fit_final_kernel<<<1, kHT, 0, s>>>(a.norm_x_sq, out4, nb, a.r0, a.r_out, a.lambda, R,
                                           a.fit_out);
    }
    return cudaGetLastError();
}

// thin_qr primitive on the cooperative kernel (a is copied into work first)
cudaError_t householder_qr_wide(const double* a, uint64_t m, uint32_t n, double* work, double* q,
                                double* r, cudaStream_t s) {
    cudaError_t e = cudaMemcpyAsync(work, a, m * n * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    HhArgs h{work, q, r, work + m * n, m, n};
    return hh_launch(h, s);
}

// u_work: 2 n^2 doubles (U and U^T)
cudaError_t launch_spd_solve_wide(const double* g, uint32_t n, double* u_work, double* x,
                                  uint64_t rows, int* status, int* reg, cudaStream_t s) {
    if (n > uint32_t(kMaxWide)) return cudaErrorInvalidValue;
    double* u = u_work;
    double* ut = u_work + size_t(n) * n;
    spd_factor_wide_kernel<<<1, 512, 0, s>>>(g, n, u, ut, status, reg);
    const size_t smem = size_t(kHW) * n * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(spd_rows_wide_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((rows + kHW - 1) / kHW, 1024)));
    spd_rows_wide_kernel<<<grid, kHT, smem, s>>>(u, ut, n, x, rows, status);
    return cudaGetLastError();
}

}  // namespace cpdb
