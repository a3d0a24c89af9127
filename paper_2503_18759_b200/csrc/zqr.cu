// K3: Q0, R0 of Z = KhatriRao(R_k, k != n) -- solvers.hpp:250-255
// (tensor.hpp:343-368 khatri_rao + linalg.hpp:39-99 thin_qr).
//
// Z is never materialised: a row of Z is the product of one row of each R_k.
// The QR is a structured CholeskyQR2:
//   G1 = Z^T Z = Hadamard_k (R_k^T R_k)            (exact identity, R x R)
//   U1 = chol(G1);  Q1 = Z U1^-1  (row-parallel)    G2 = Q1^T Q1 (DMMA partials)
//   U2 = chol(G2);  Q0 = Q1 U2^-1;  R0 = U2 U1
// diag(R0) > 0 matches the reference's sign convention (linalg.hpp:92-97), and
// Z's e1 first column makes Q0's first row/column e1 to rounding
// (linalg_test.cpp:88-109).  Z's rows are in the NATURAL order of the final Y
// (row-major over the other modes ascending, last fastest); the reference's
// Khatri-Rao order is its digit reversal (runtime.cpp natural_to_reference).
//
// Small Z (C1-C4) runs as one 8-CTA cluster kernel (cluster.cu); this file is
// the multi-kernel path for tall Z (C5: 262144 x 64).
#include <algorithm>

#include "kernels.hpp"
#include "rowalg.cuh"

namespace cpdb {
namespace {

constexpr int kNT = 512;
constexpr int kTile = 256;      // Z rows staged per tile (fewer when R is large)
constexpr int kMaxParts = 296;  // G2 partials (one per CTA)

// work layout (doubles): [U1 | G2 -> U2 | partials of G2 ...]
template <int RM>
__global__ void __launch_bounds__(kNT) zqr_prep_kernel(ZqrArgs a) {
    extern __shared__ double sm[];
    const int R = a.R, nm = a.nm;
    double* g = sm;
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) {
        const int p = e / R, q = e % R;
        const int lo = p < q ? p : q, hi = p < q ? q : p;
        double h = 1.0;
        for (int t = nm - 1; t >= 0; --t) {
            const double* m = a.rmats[t];
            double s = 0.0;
            for (int k = 0; k <= lo; ++k) s = fma(m[k * R + lo], m[k * R + hi], s);
            h = (t == nm - 1) ? s : h * s;
        }
        g[e] = h;
    }
    __syncthreads();
    if (!chol<kNT, RM>(g, R, R) && threadIdx.x == 0) *a.status = 2;
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) a.work[e] = g[e];
}

// Q1 = Z U1^-1 tile by tile; per-CTA partial G2 = Q1^T Q1 on DMMA.
template <int RM>
__global__ void __launch_bounds__(kNT) zqr_rows_kernel(ZqrArgs a, int tile_rows) {
    using Row = LaneRow<RM>;
    constexpr int T = Row::T, G = kNT / T;
    extern __shared__ double sm[];
    const int R = a.R, nm = a.nm, ld = R + 1;
    double* mats = sm;                 // nm x R x R
    double* u = mats + nm * R * R;     // RM x RM
    double* dinv = u + RM * RM;        // RM
    double* part = dinv + RM;          // R x R  (this CTA's G2 partial)
    double* tile = part + R * R;       // kTile x (R+1)
    for (int t = 0; t < nm; ++t)
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) mats[t * R * R + e] = a.rmats[t][e];
    stage_tri<RM>(a.work, R, R, u, dinv, kNT);
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) part[e] = 0.0;
    const int grp = threadIdx.x / T, q = threadIdx.x % T;
    const uint64_t ntiles = (a.zrows + tile_rows - 1) / tile_rows;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t row0 = t * tile_rows;
        const int rows = int(min(uint64_t(tile_rows), a.zrows - row0));
        __syncthreads();
        for (int li = grp; li < tile_rows + (G - tile_rows % G) % G; li += G) {
            const bool act = li < rows;
            Row x;
            // Z row = product over the other modes (descending, like the
            // reference Khatri-Rao fold), digits peeled in the same order
            // (32-bit: zrows < 2^32 on this path); rolled over the modes
            {
                uint32_t rem = uint32_t(row0) + uint32_t(act ? li : 0);
#pragma unroll 1
                for (int k = nm - 1; k >= 0; --k) {
                    const uint32_t qt = rem / uint32_t(R);
                    const double* m = mats + (k * R + int(rem - qt * uint32_t(R))) * R;
                    rem = qt;
#pragma unroll
                    for (int s = 0; s < Row::S; ++s) {
                        const int c = s * T + q;
                        const double v = m[c < R ? c : 0];
                        x.t[s] = (k == nm - 1) ? v : x.t[s] * v;
                    }
                }
#pragma unroll
                for (int s = 0; s < Row::S; ++s)
                    if (!(act && s * T + q < R)) x.t[s] = 0.0;
            }
            x.uinv(u, dinv, R, q);
            if (act) {
                x.store(tile + li * ld, R, q);
                x.store(a.q1 + (row0 + li) * R, R, q);
            }
        }
        __syncthreads();
        gram_dmma<kNT>(tile, ld, rows, R, part, R, true);
    }
    __syncthreads();
    double* out = a.work + 2 * R * R + size_t(blockIdx.x) * R * R;
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) out[e] = part[e];
}

__global__ void __launch_bounds__(kNT) zqr_reduce_kernel(ZqrArgs a, int nparts) {
    const int R2 = a.R * a.R;
    for (int e = blockIdx.x * kNT + threadIdx.x; e < R2; e += gridDim.x * kNT) {
        const double* p = a.work + 2 * R2 + e;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int b = 0;
        for (; b + 3 < nparts; b += 4) {
            s0 += p[size_t(b) * R2];
            s1 += p[size_t(b + 1) * R2];
            s2 += p[size_t(b + 2) * R2];
            s3 += p[size_t(b + 3) * R2];
        }
        for (; b < nparts; ++b) s0 += p[size_t(b) * R2];
        a.work[R2 + e] = (s0 + s1) + (s2 + s3);
    }
}

template <int RM>
__global__ void __launch_bounds__(kNT) zqr_fin_kernel(ZqrArgs a) {
    extern __shared__ double sm[];
    const int R = a.R;
    double* g = sm;
    double* u1 = g + R * R;
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) {
        g[e] = a.work[R * R + e];
        u1[e] = a.work[e];
    }
    __syncthreads();
    // G2 = Q1^T Q1 = I + O(kappa^2 eps): series factorisation (rowalg.cuh)
    __shared__ double red[32];
    const bool ok = near_identity_chol<kNT>(g, R, g + 2 * R * R, g + 3 * R * R, red) > 0 ||
                    chol<kNT, RM>(g, R, R);
    if (!ok && threadIdx.x == 0) *a.status = 2;
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) {
        const int i = e / R, j = e % R;
        double s = 0.0;
        for (int p = i; p <= j; ++p) s = fma(g[i * R + p], u1[p * R + j], s);
        a.r0[e] = i <= j ? s : 0.0;
        a.work[R * R + e] = g[e];  // U2
    }
}

// Q0 = Q1 U2^-1, one lane group per row
template <int RM>
__global__ void __launch_bounds__(kNT) zqr_apply_kernel(ZqrArgs a) {
    using Row = LaneRow<RM>;
    constexpr int T = Row::T, G = kNT / T;
    __shared__ double u[RM * RM];
    __shared__ double dinv[RM];
    const int R = a.R;
    stage_tri<RM>(a.work + R * R, R, R, u, dinv, kNT);
    __syncthreads();
    const int grp = threadIdx.x / T, q = threadIdx.x % T;
    const uint64_t stride = uint64_t(gridDim.x) * G;
    const uint64_t total = ((a.zrows + stride - 1) / stride) * stride;
    for (uint64_t r = blockIdx.x * uint64_t(G) + grp; r < total; r += stride) {
        const bool act = r < a.zrows;
        Row x;
        x.load(a.q1 + (act ? r : 0) * R, act ? R : 0, q);
        x.uinv(u, dinv, R, q);
        if (act) x.store(a.q0 + r * R, R, q);
    }
}

template <int RM>
cudaError_t run_multi(const ZqrArgs& a, cudaStream_t s, int sms) {
    const int R = a.R;
    if (a.zrows >= (1ull << 32)) return cudaErrorInvalidValue;  // 32-bit row digits
    const size_t fixed = size_t(a.nm) * R * R + RM * RM + RM + size_t(R) * R;
    constexpr size_t kBudget = 220 * 1024 / sizeof(double);
    if (fixed + 32 * size_t(R + 1) > kBudget) return cudaErrorInvalidValue;
    // rows per staged tile: as many as fit (multiple of 32), at most kTile
    const int tile = int(std::min<size_t>(kTile, ((kBudget - fixed) / (R + 1)) / 32 * 32));
    const size_t rows_smem = (fixed + size_t(tile) * (R + 1)) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(zqr_rows_kernel<RM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return e;
    zqr_prep_kernel<RM><<<1, kNT, size_t(R) * R * sizeof(double), s>>>(a);
    const uint64_t ntiles = (a.zrows + tile - 1) / tile;
    const int grid = int(std::min<uint64_t>(ntiles, uint64_t(std::min(2 * sms, kMaxParts))));
    zqr_rows_kernel<RM><<<grid, kNT, rows_smem, s>>>(a, tile);
    zqr_reduce_kernel<<<(R * R + kNT - 1) / kNT, kNT, 0, s>>>(a, grid);
    e = cudaFuncSetAttribute(zqr_fin_kernel<RM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(4 * RM * RM * sizeof(double)));
    if (e != cudaSuccess) return e;
    zqr_fin_kernel<RM><<<1, kNT, 4 * size_t(R) * R * sizeof(double), s>>>(a);
    const uint64_t groups = (a.zrows + (kNT / LaneRow<RM>::T) - 1) / (kNT / LaneRow<RM>::T);
    const int agrid = int(std::min<uint64_t>(groups, uint64_t(4 * sms)));
    zqr_apply_kernel<RM><<<agrid, kNT, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

size_t zqr_work_doubles(uint32_t R) { return size_t(2 + kMaxParts) * R * R; }

cudaError_t launch_zqr(const ZqrArgs& a, cudaStream_t s, int sms) {
    if (zqr_cluster_fits(a.zrows, a.R, a.nm)) return launch_zqr_cluster(a, s);
    return launch_zqr_multi(a, s, sms);
}

cudaError_t launch_zqr_multi(const ZqrArgs& a, cudaStream_t s, int sms) {
    if (a.R <= 8) return run_multi<8>(a, s, sms);
    if (a.R <= 16) return run_multi<16>(a, s, sms);
    if (a.R <= 32) return run_multi<32>(a, s, sms);
    if (a.R <= 64) return run_multi<64>(a, s, sms);
    return cudaErrorInvalidValue;
}

}  // namespace cpdb
