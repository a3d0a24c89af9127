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
#include <cstdlib>

#include "kernels.hpp"
#include "rowalg.cuh"

namespace cpdb {
namespace {

constexpr int kNT = 512;
constexpr int kTile = 256;      // Z rows staged per tile (fewer when R is large)
constexpr int kMaxParts = 296;  // G2 partials (one per CTA)

// work layout (doubles): [U1 | G2 -> U2 | W1 = U1^-1 | W2 = U2^-1 | partials of G2 ...]
constexpr int kPartOff = 4;  // partials start at kPartOff * R * R
// W = U^-1 for upper-triangular U (R x R, stride R, R <= 64, in shared
// memory): rows of W from the last up, W[i][j] = -(sum_{k=i+1..j} U[i][k]
// W[k][j]) / U[i][i], the columns j of a row in parallel, NT/64 threads per
// column summing fixed strided subsets combined by a fixed shuffle butterfly
// (deterministic); w: R x R shared scratch, dinv: R shared.  The result is
// written to `out` (global, stride R).
template <int NT>
__device__ void upper_inverse(const double* u, int R, double* w, double* dinv, double* out) {
    constexpr int TPC = NT / 64;
    for (int e = threadIdx.x; e < R * R; e += NT) w[e] = 0.0;
    for (int i = threadIdx.x; i < R; i += NT) dinv[i] = 1.0 / u[i * R + i];
    __syncthreads();
    const int j = threadIdx.x / TPC, sub = threadIdx.x % TPC;
#pragma unroll 1
    for (int i = R - 1; i >= 0; --i) {
        double acc = 0.0;
        if (j < R && j > i)
#pragma unroll 1
            for (int k = i + 1 + sub; k <= j; k += TPC) acc = fma(u[i * R + k], w[k * R + j], acc);
#pragma unroll
        for (int o = TPC / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (sub == 0 && j < R && j >= i) w[i * R + j] = j == i ? dinv[i] : -acc * dinv[i];
        __syncthreads();
    }
    for (int e = threadIdx.x; e < R * R; e += NT) out[e] = w[e];
}

template <int RM>
__global__ void __launch_bounds__(kNT) zqr_prep_kernel(ZqrArgs a) {
    extern __shared__ double sm[];
    const int R = a.R, nm = a.nm;
    double* g = sm;
    // G1 = Hadamard_k R_k^T R_k: each R_k staged (behind g's R x R, the
    // inverse's scratch later) and its Gram on DMMA (gram_dmma), the last
    // mode's first
    double* stage = g + R * R;
    double* gk = stage + R * R;
#pragma unroll 1
    for (int t = nm - 1; t >= 0; --t) {
        __syncthreads();
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) stage[e] = a.rmats[t][e];
        __syncthreads();
        gram_dmma<kNT>(stage, R, R, R, gk, R);
        __syncthreads();
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) g[e] = t == nm - 1 ? gk[e] : g[e] * gk[e];
    }
    __syncthreads();
    // (the staging area behind g is free: scratch of the shifted retry)
    const int fp = chol_first_pass<kNT, RM>(g, R, a.zrows, g + R * R);
    if (fp < 0 && threadIdx.x == 0) *a.status = 2;
    if (fp == 1 && threadIdx.x == 0) atomicOr(a.status, kStatusShifted);
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) a.work[e] = g[e];
    __syncthreads();
    // W1 = U1^-1 (the GEMM form of Q1 = Z U1^-1)
    upper_inverse<kNT>(g, R, g + R * R, g + 2 * R * R, a.work + 2 * R * R);
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
    double* out = a.work + kPartOff * R * R + size_t(blockIdx.x) * R * R;
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) out[e] = part[e];
}

// Q1 = Z W1 on the FP64 tensor cores (W1 = U1^-1 from zqr_prep), tile by
// tile of kGT rows: the tile of Z is built in shared memory from the rows of
// the R_k (the fastest digit's R_k staged, the slower ones read through L2),
// multiplied by the staged W1 (DMMA m8n8k4, warp w owns rows 8w..8w+7), Q1
// stored, and the tile's Gram added to this CTA's G2 partial (DMMA, fixed
// order).  Replaces the row-by-row register substitution (zqr_rows_kernel,
// CPDB_ZQR_GEMM=0; C5: 0.62 ms per update).
constexpr int kGT = 128;  // rows per tile (16 warps x 8)
template <int RM>
struct ZgSmem {
    static constexpr int LD = RM + 4;  // padded rows: conflict-free fragments
    static constexpr size_t doubles(int R) {
        return size_t(RM) * LD + size_t(kGT) * LD + size_t(R) * LD + size_t(R) * R +
               size_t(kGT / R + 2) * R;
    }
};

// Warp tiling of a kGT x RM tile product over the 16 warps: WR x WC blocks
// (16 x 32 at RM = 64: per 4-k step 2 A + 4 B fragment loads feed 8 DMMAs,
// against 1 + 8 with one 8-row strip per warp)
template <int RM>
struct WarpTile {
    static constexpr int WC = RM / 2 >= 8 ? RM / 2 : 8;  // columns per warp
    static constexpr int CG = RM / WC;                   // column groups
    static constexpr int RG = (kNT / 32) / CG;           // row groups
    static constexpr int WR = kGT / RG;                  // rows per warp
    static constexpr int RBW = WR / 8, CBW = WC / 8;
};

template <int RM>
__global__ void __launch_bounds__(kNT) zqr_rows_gemm_kernel(ZqrArgs a) {
    constexpr int LD = ZgSmem<RM>::LD;
    extern __shared__ double sm[];
    const int R = a.R, nm = a.nm;
    double* w1 = sm;                // RM x LD
    double* zt = w1 + RM * LD;      // kGT x LD: Z tile, then Q1 tile
    double* fast = zt + kGT * LD;   // R x LD: the fastest digit's R_k (padded rows)
    double* part = fast + R * LD;   // R x R: this CTA's G2 partial
    double* slow = part + R * R;    // (kGT / R + 2) x R: products of the slower digits' rows
    const double* wsrc = a.work + 2 * R * R;
#pragma unroll 1
    for (int e = threadIdx.x; e < RM * RM; e += kNT) {
        const int i = e / RM, j = e % RM;
        w1[i * LD + j] = (i < R && j < R) ? wsrc[i * R + j] : 0.0;
    }
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) {
        fast[(e / R) * LD + e % R] = a.rmats[nm - 1][e];
        part[e] = 0.0;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = lane >> 2, kq = lane & 3;
    // G2 partial in registers for the whole CTA: the (nt(nt+1)/2) upper 8x8
    // blocks dealt round-robin to the warps (up to kGP each), every block one
    // DMMA chain over the tile rows -- no shared-memory read-modify-write per
    // tile, independent chains per warp
    constexpr int NT8 = RM / 8, NPAIR = NT8 * (NT8 + 1) / 2;
    constexpr int kGP = (NPAIR + kNT / 32 - 1) / (kNT / 32);
    int gpa[kGP], gpb[kGP];
    double gacc[kGP][2];
#pragma unroll
    for (int j = 0; j < kGP; ++j) {
        const int pidx = warp + j * (kNT / 32);
        int ti = 0, rem = pidx;
        while (ti < NT8 && rem >= NT8 - ti) {
            rem -= NT8 - ti;
            ++ti;
        }
        const bool live = pidx < NPAIR;
        gpa[j] = live ? ti : -1;
        gpb[j] = live ? ti + rem : -1;
        gacc[j][0] = gacc[j][1] = 0.0;
    }
    const uint64_t ntiles = (a.zrows + kGT - 1) / kGT;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t row0 = t * kGT;
        const int rows = int(min(uint64_t(kGT), a.zrows - row0));
        __syncthreads();  // the previous tile's Gram is done with zt / slow
        // Z row t = R_{nm-1}[t % R] * P[t / R], P[q] = the product of the
        // slower digits' rows of q (the next slower first): one product per
        // group of R consecutive rows, then one multiply per element
        const uint32_t g0 = uint32_t(row0) / uint32_t(R);
        const int ng = int((uint32_t(row0) + uint32_t(rows) - 1) / uint32_t(R) - g0) + 1;
#pragma unroll 1
        for (int e = threadIdx.x; e < ng * R; e += kNT) {
            const int gi = e / R, c = e % R;
            uint32_t rem = g0 + uint32_t(gi);
            double v = 1.0;
#pragma unroll 1
            for (int k = nm - 2; k >= 0; --k) {
                const uint32_t qt = rem / uint32_t(R);
                const double m = a.rmats[k][int(rem - qt * uint32_t(R)) * R + c];
                v = (k == nm - 2) ? m : v * m;
                rem = qt;
            }
            slow[e] = v;
        }
        __syncthreads();
        // A fragments straight from the staged rows (no Z tile):
        // Z[t][k] = R_fast[t % R][k] * P[t / R][k]
        using WT = WarpTile<RM>;
        const int rw0 = (warp % WT::RG) * WT::WR, cw0 = (warp / WT::RG) * WT::WC;
        double acc[WT::RBW][WT::CBW][2];
#pragma unroll
        for (int x = 0; x < WT::RBW; ++x)
#pragma unroll
            for (int y = 0; y < WT::CBW; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
        {
            const double* fr[WT::RBW];
            const double* sr[WT::RBW];
            bool rowok[WT::RBW];
#pragma unroll
            for (int x = 0; x < WT::RBW; ++x) {
                const int rr = rw0 + x * 8 + m;
                rowok[x] = rr < rows;
                const uint32_t t = uint32_t(row0) + uint32_t(rowok[x] ? rr : 0);
                const uint32_t q = t / uint32_t(R);
                fr[x] = fast + int(t - q * uint32_t(R)) * LD;
                sr[x] = slow + int(q - g0) * R;
            }
#pragma unroll
            for (int k4 = 0; k4 < RM / 4; ++k4) {
                const int k = 4 * k4 + kq;
                double af[WT::RBW];
#pragma unroll
                for (int x = 0; x < WT::RBW; ++x)
                    af[x] = (rowok[x] && k < R) ? fr[x][k] * sr[x][k] : 0.0;
#pragma unroll
                for (int y = 0; y < WT::CBW; ++y) {
                    const double bv = w1[(4 * k4 + kq) * LD + cw0 + y * 8 + m];
#pragma unroll
                    for (int x = 0; x < WT::RBW; ++x)
                        dmma(acc[x][y][0], acc[x][y][1], af[x], bv);
                }
            }
        }
#pragma unroll
        for (int x = 0; x < WT::RBW; ++x) {
            const int r = rw0 + x * 8 + m;
#pragma unroll
            for (int y = 0; y < WT::CBW; ++y) {
                const int c = cw0 + y * 8 + 2 * kq;
                zt[r * LD + c] = acc[x][y][0];
                zt[r * LD + c + 1] = acc[x][y][1];
                if (r < rows) {
                    double* q = a.q1 + (row0 + r) * R;
                    if (c < R) q[c] = acc[x][y][0];
                    if (c + 1 < R) q[c + 1] = acc[x][y][1];
                }
            }
        }
        __syncthreads();
        // Gram of the Q1 tile (rows past `rows` are zero in zt)
#pragma unroll 4
        for (int k0 = 0; k0 < kGT; k0 += 4) {
            const double* zr = zt + (k0 + kq) * LD;
#pragma unroll
            for (int j = 0; j < kGP; ++j) {
                if (gpa[j] < 0) continue;
                dmma(gacc[j][0], gacc[j][1], zr[gpa[j] * 8 + m], zr[gpb[j] * 8 + m]);
            }
        }
    }
    // C[m][2kq + {0,1}] of each block; the mirrored copy of an off-diagonal
    // block is written by the same lane (one writer per entry)
    double* out = a.work + kPartOff * R * R + size_t(blockIdx.x) * R * R;
#pragma unroll
    for (int j = 0; j < kGP; ++j) {
        if (gpa[j] < 0) continue;
        const int r = gpa[j] * 8 + m, cc = gpb[j] * 8 + 2 * kq;
        if (r < R) {
            if (cc < R) {
                out[r * R + cc] = gacc[j][0];
                if (gpa[j] != gpb[j]) out[cc * R + r] = gacc[j][0];
            }
            if (cc + 1 < R) {
                out[r * R + cc + 1] = gacc[j][1];
                if (gpa[j] != gpb[j]) out[(cc + 1) * R + r] = gacc[j][1];
            }
        }
    }
    (void)part;
}

// Q0 = Q1 W2 (W2 = U2^-1, near the identity) on DMMA, kGT rows per tile.
template <int RM>
__global__ void __launch_bounds__(kNT, 2) zqr_apply_gemm_kernel(ZqrArgs a) {
    constexpr int LD = ZgSmem<RM>::LD;
    extern __shared__ double sm[];
    const int R = a.R;
    double* w2 = sm;            // RM x LD
    double* qt = w2 + RM * LD;  // kGT x LD
    const double* wsrc = a.work + 3 * R * R;
#pragma unroll 1
    for (int e = threadIdx.x; e < RM * RM; e += kNT) {
        const int i = e / RM, j = e % RM;
        w2[i * LD + j] = (i < R && j < R) ? wsrc[i * R + j] : 0.0;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = lane >> 2, kq = lane & 3;
    const uint64_t ntiles = (a.zrows + kGT - 1) / kGT;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t row0 = t * kGT;
        const int rows = int(min(uint64_t(kGT), a.zrows - row0));
        __syncthreads();
#pragma unroll
        for (int e = threadIdx.x; e < kGT * RM; e += kNT) {
            const int r = e / RM, c = e % RM;
            qt[r * LD + c] = (r < rows && c < R) ? __ldcs(a.q1 + (row0 + r) * R + c) : 0.0;
        }
        __syncthreads();
        using WT = WarpTile<RM>;
        const int rw0 = (warp % WT::RG) * WT::WR, cw0 = (warp / WT::RG) * WT::WC;
        double acc[WT::RBW][WT::CBW][2];
#pragma unroll
        for (int x = 0; x < WT::RBW; ++x)
#pragma unroll
            for (int y = 0; y < WT::CBW; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
#pragma unroll
        for (int k4 = 0; k4 < RM / 4; ++k4) {
            double af[WT::RBW];
#pragma unroll
            for (int x = 0; x < WT::RBW; ++x) af[x] = qt[(rw0 + x * 8 + m) * LD + 4 * k4 + kq];
#pragma unroll
            for (int y = 0; y < WT::CBW; ++y) {
                const double bv = w2[(4 * k4 + kq) * LD + cw0 + y * 8 + m];
#pragma unroll
                for (int x = 0; x < WT::RBW; ++x) dmma(acc[x][y][0], acc[x][y][1], af[x], bv);
            }
        }
#pragma unroll
        for (int x = 0; x < WT::RBW; ++x) {
            const int r = rw0 + x * 8 + m;
            if (r >= rows) continue;
            double* q = a.q0 + (row0 + r) * R;
#pragma unroll
            for (int y = 0; y < WT::CBW; ++y) {
                const int c = cw0 + y * 8 + 2 * kq;
                if (c < R) q[c] = acc[x][y][0];
                if (c + 1 < R) q[c + 1] = acc[x][y][1];
            }
        }
    }
}

__global__ void __launch_bounds__(kNT) zqr_reduce_kernel(ZqrArgs a, int nparts) {
    const int R2 = a.R * a.R;
    for (int e = blockIdx.x * kNT + threadIdx.x; e < R2; e += gridDim.x * kNT) {
        const double* p = a.work + kPartOff * R2 + e;
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
    __syncthreads();
    // W2 = U2^-1 (the GEMM apply); g + 2R^2 .. is the series' scratch, free now
    upper_inverse<kNT>(g, R, g + 2 * R * R, g + 3 * R * R, a.work + 3 * R * R);
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
    static const bool gemm = [] {
        const char* v = std::getenv("CPDB_ZQR_GEMM");
        return !(v && v[0] == '0');
    }();
    const size_t psm = (3 * size_t(R) * R + R) * sizeof(double);
    e = cudaFuncSetAttribute(zqr_prep_kernel<RM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int((3 * size_t(RM) * RM + RM) * sizeof(double)));
    if (e != cudaSuccess) return e;
    zqr_prep_kernel<RM><<<1, kNT, psm, s>>>(a);
    int grid;
    if (gemm) {
        const size_t gsm = ZgSmem<RM>::doubles(R) * sizeof(double);
        e = cudaFuncSetAttribute(zqr_rows_gemm_kernel<RM>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(gsm));
        if (e != cudaSuccess) return e;
        const uint64_t ntiles = (a.zrows + kGT - 1) / kGT;
        grid = int(std::min<uint64_t>(ntiles, uint64_t(std::min(sms, kMaxParts))));
        zqr_rows_gemm_kernel<RM><<<grid, kNT, gsm, s>>>(a);
    } else {
        const uint64_t ntiles = (a.zrows + tile - 1) / tile;
        grid = int(std::min<uint64_t>(ntiles, uint64_t(std::min(2 * sms, kMaxParts))));
        zqr_rows_kernel<RM><<<grid, kNT, rows_smem, s>>>(a, tile);
    }
    zqr_reduce_kernel<<<(R * R + kNT - 1) / kNT, kNT, 0, s>>>(a, grid);
    e = cudaFuncSetAttribute(zqr_fin_kernel<RM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(4 * RM * RM * sizeof(double)));
    if (e != cudaSuccess) return e;
    zqr_fin_kernel<RM><<<1, kNT, 4 * size_t(R) * R * sizeof(double), s>>>(a);
    if (gemm) {
        const size_t asm_ = size_t(RM + kGT) * ZgSmem<RM>::LD * sizeof(double);
        e = cudaFuncSetAttribute(zqr_apply_gemm_kernel<RM>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(asm_));
        if (e != cudaSuccess) return e;
        const uint64_t ntiles = (a.zrows + kGT - 1) / kGT;
        const int agrid = int(std::min<uint64_t>(ntiles, uint64_t(2 * sms)));  // 2 per SM
        zqr_apply_gemm_kernel<RM><<<agrid, kNT, asm_, s>>>(a);
    } else {
        const uint64_t groups = (a.zrows + (kNT / LaneRow<RM>::T) - 1) / (kNT / LaneRow<RM>::T);
        const int agrid = int(std::min<uint64_t>(groups, uint64_t(4 * sms)));
        zqr_apply_kernel<RM><<<agrid, kNT, 0, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace

size_t zqr_work_doubles(uint32_t R) {
    return std::max(zqr_wide_work_doubles(R), wide_rank(R) ? size_t(0)
                                                           : size_t(kPartOff + kMaxParts) * R * R);
}

cudaError_t launch_zqr(const ZqrArgs& a, cudaStream_t s, int sms) {
    if (wide_rank(a.R) || a.householder) return launch_zqr_wide(a, s);
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
