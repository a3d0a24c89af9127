// Small dense building blocks for the mode-update kernels (R <= 64).
//
// The matrices are tiny (I <= a few hundred rows, R <= 64), so latency, not
// FLOPs, bounds them.  Measured on B200 (tools/probes/, profiles/):
// dependent LDS ~55 cycles, DFMA 8.6, __syncthreads ~29, shuffle ~25,
// DDIV ~400 (!), rcp/rsqrt ~70.  Hence:
//  * a row's triangular solve runs "right-looking" in REGISTERS, spread over
//    T = RM/8 lanes (lane q owns columns k = 8*i + ... with k % T == q): once
//    x_j is final its owner broadcasts it with one shuffle and every lane
//    updates its own partial sums -- the critical path is R x (mul + shfl +
//    fma) and every lane holds exactly 8 columns;
//  * Grams W^T W run on the FP64 tensor cores (mma.m8n8k4 -> DMMA);
//  * no IEEE division inside loops (reciprocals are precomputed).
#pragma once

#include "device.cuh"

namespace cpdb {

template <int NT>
__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (warp == 0) {
        s = lane < NT / 32 ? red[lane] : 0.0;
        s = warp_sum(s);
    }
    return s;  // valid in warp 0
}

// max over the block, returned to every thread
template <int NT>
__device__ double block_max(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double m = red[0];
    for (int w = 1; w < NT / 32; ++w) m = fmax(m, red[w]);
    return m;
}

// ---------------------------------------------------------------- lane rows
// A row of length <= RM distributed over T = RM/8 lanes: lane q holds
// x[8*i... ] as t[s] = x[s*T + q], s < 8.
// SL = slots per lane: 8 by default; fewer slots (more lanes per row) when a
// CTA has fewer rows than lane groups, which shortens every solve step.
template <int RM, int SL = 8>
struct LaneRow {
    static constexpr int T = RM / SL > 0 ? RM / SL : 1;  // lanes per row (<= 32)
    static constexpr int S = RM / T;                    // slots per lane
    static_assert(T <= 32, "LaneRow: at most one warp per row");
    double t[S];

    __device__ __forceinline__ void load(const double* src, int R, int q) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int k = s * T + q;
            t[s] = k < R ? src[k] : 0.0;
        }
    }
    // sum of n row copies src[p * stride + k], p = 0..n-1 in order (the
    // V-GEMM's split-K partials: fixed order -> deterministic)
    __device__ __forceinline__ void load_sum(const double* src, uint64_t stride, uint32_t n,
                                             int R, int q) {
#pragma unroll
        for (int s = 0; s < S; ++s) t[s] = 0.0;
        // four partials' loads in flight per step, summed in order
        uint32_t p = 0;
#pragma unroll 1
        for (; p + 4 <= n; p += 4) {
            const double* row = src + p * stride + q;
            double v[4][S];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int s = 0; s < S; ++s)
                    v[u][s] = s * T + q < R ? row[u * stride + s * T] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int s = 0; s < S; ++s) t[s] += v[u][s];
        }
#pragma unroll 1
        for (; p < n; ++p) {
            const double* row = src + p * stride + q;
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (s * T + q < R) t[s] += row[s * T];
        }
    }
    __device__ __forceinline__ void store(double* dst, int R, int q) const {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int k = s * T + q;
            if (k < R) dst[k] = t[s];
        }
    }
    // The solves below run j (the pivot column) as an UNROLLED loop over the
    // owner's slot js and a ROLLED loop over the owner lane o (j = js*T + o),
    // so every register index stays static while the code is S x (S FMAs)
    // instead of RM x S.  Measured (ncu source counters, C2): the fully
    // unrolled form made the mode-update kernels instruction-fetch bound
    // (~12k SASS instructions executed once per launch, "no instruction"
    // the top stall of their serial phases).  Same operations in the same
    // order as the unrolled form -> bit-identical results.

    // x <- x U^-1, U upper with stride RM (zero padded, unit diagonal beyond
    // R), dinv[j] = 1/U[j][j]: right-looking forward substitution.
    __device__ __forceinline__ void uinv(const double* U, const double* dinv, int R, int q) {
#pragma unroll
        for (int js = 0; js < S; ++js) {
#pragma unroll 1
            for (int o = 0; o < T; ++o) {
                const int j = js * T + o;
                if (j >= R) break;  // uniform
                double xj = t[js] * dinv[j];
                xj = __shfl_sync(0xffffffffu, xj, o, T);
                const double* Uj = U + j * RM + q;
                if (q == o) t[js] = xj;
                else if (q > o) t[js] = fma(-xj, Uj[js * T], t[js]);
#pragma unroll
                for (int s2 = js + 1; s2 < S; ++s2) t[s2] = fma(-xj, Uj[s2 * T], t[s2]);
            }
        }
    }
    // x <- x U^-T (solve x U^T = v; lower L = U^T), right-looking backward:
    // x_c = t_c / U[c][c], then t_k -= x_c U[k][c] for k < c -- the
    // row-wise triangular solve of linalg.hpp:192-216 with L = R0^T.
    // Ut is U TRANSPOSED (stride RM), so a lane group reads consecutive words.
    __device__ __forceinline__ void utinv(const double* Ut, const double* dinv, int R, int q) {
#pragma unroll
        for (int cs = S - 1; cs >= 0; --cs) {
#pragma unroll 1
            for (int o = T - 1; o >= 0; --o) {
                const int c = cs * T + o;
                if (c >= R) continue;  // uniform
                double xc = t[cs] * dinv[c];
                xc = __shfl_sync(0xffffffffu, xc, o, T);
                const double* Uc = Ut + c * RM + q;
                if (q == o) t[cs] = xc;
                else if (q < o) t[cs] = fma(-xc, Uc[cs * T], t[cs]);
#pragma unroll
                for (int s2 = 0; s2 < cs; ++s2) t[s2] = fma(-xc, Uc[s2 * T], t[s2]);
            }
        }
    }
    // this <- v U for upper U (stride RM): t[k] = sum_{j<=k} v[j] U[j][k]
    __device__ __forceinline__ void set_times_upper(const LaneRow& v, const double* U, int R,
                                                    int q) {
#pragma unroll
        for (int s = 0; s < S; ++s) t[s] = 0.0;
#pragma unroll
        for (int js = 0; js < S; ++js) {
#pragma unroll 1
            for (int o = 0; o < T; ++o) {
                const int j = js * T + o;
                if (j >= R) break;  // uniform
                const double vj = __shfl_sync(0xffffffffu, v.t[js], o, T);
                const double* Uj = U + j * RM + q;
                if (q >= o) t[js] = fma(vj, Uj[js * T], t[js]);
#pragma unroll
                for (int s2 = js + 1; s2 < S; ++s2) t[s2] = fma(vj, Uj[s2 * T], t[s2]);
            }
        }
    }
    // sum over lanes of the group
    __device__ __forceinline__ static double group_sum(double v) {
#pragma unroll
        for (int o = 1; o < T; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    }
};

// Triangular factor staged in smem with the compile-time stride RM:
// entries beyond R are 0 off the diagonal and 1 on it.
template <int RM>
__device__ void stage_tri(const double* src, int ld_src, int R, double* dst, double* dinv,
                          int nthreads) {
#pragma unroll 1
    for (int e = threadIdx.x; e < RM * RM; e += nthreads) {
        const int i = e / RM, j = e % RM;
        dst[e] = (i < R && j < R) ? src[i * ld_src + j] : (i == j ? 1.0 : 0.0);
    }
#pragma unroll 1
    for (int j = threadIdx.x; j < RM; j += nthreads)
        dinv[j] = j < R ? __drcp_rn(src[j * ld_src + j]) : 1.0;
}

// Same, transposed: dst[j][i] = src[i][j] (for LaneRow::utinv).
template <int RM>
__device__ void stage_tri_t(const double* src, int ld_src, int R, double* dst, double* dinv,
                            int nthreads) {
#pragma unroll 1
    for (int e = threadIdx.x; e < RM * RM; e += nthreads) {
        const int i = e / RM, j = e % RM;
        dst[j * RM + i] = (i < R && j < R) ? src[i * ld_src + j] : (i == j ? 1.0 : 0.0);
    }
#pragma unroll 1
    for (int j = threadIdx.x; j < RM; j += nthreads)
        dinv[j] = j < R ? __drcp_rn(src[j * ld_src + j]) : 1.0;
}

// ---------------------------------------------------------------- Gram on DMMA
// G[p][q] (full R x R, stride ldg) = sum_i W[i][p] W[i][q] over `rows` rows
// of W (stride ld), FP64 tensor cores: one warp per 8x8 output tile, k = 4
// rows per DMMA; fixed order -> deterministic.
template <int NT>
__device__ void gram_dmma(const double* w, int ld, int rows, int R, double* g, int ldg,
                          bool accumulate = false) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nt = (R + 7) / 8;
    const int m = lane >> 2, kq = lane & 3;
    for (int tix = warp; tix < nt * nt; tix += NT / 32) {
        const int ti = tix / nt, tj = tix % nt;
        if (tj < ti) continue;
        const int pa = ti * 8 + m, pb = tj * 8 + m;
        double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
        int k0 = 0;
        for (; k0 + 4 < rows; k0 += 8) {
            const int i0 = k0 + kq, i1 = k0 + 4 + kq;
            const double a0 = (pa < R) ? w[i0 * ld + pa] : 0.0;
            const double b0 = (pb < R) ? w[i0 * ld + pb] : 0.0;
            const double a1 = (pa < R && i1 < rows) ? w[i1 * ld + pa] : 0.0;
            const double b1 = (pb < R && i1 < rows) ? w[i1 * ld + pb] : 0.0;
            dmma(c0, c1, a0, b0);
            dmma(d0, d1, a1, b1);
        }
        for (; k0 < rows; k0 += 4) {
            const int i0 = k0 + kq;
            const double a0 = (pa < R && i0 < rows) ? w[i0 * ld + pa] : 0.0;
            const double b0 = (pb < R && i0 < rows) ? w[i0 * ld + pb] : 0.0;
            dmma(c0, c1, a0, b0);
        }
        c0 += d0;
        c1 += d1;
        // C[m][2*kq + {0,1}] of the tile; the mirrored copy of a diagonal
        // tile is written by the lane that owns it, so each entry has one writer
        const int r = ti * 8 + m, cc = tj * 8 + 2 * kq;
        if (r < R) {
            if (cc < R) {
                const double v = accumulate ? g[r * ldg + cc] + c0 : c0;
                g[r * ldg + cc] = v;
                if (ti != tj) g[cc * ldg + r] = v;
            }
            if (cc + 1 < R) {
                const double v = accumulate ? g[r * ldg + cc + 1] + c1 : c1;
                g[r * ldg + cc + 1] = v;
                if (ti != tj) g[(cc + 1) * ldg + r] = v;
            }
        }
    }
}

// ---------------------------------------------------------------- Cholesky
// Right-looking Cholesky of the symmetric R x R matrix g (stride ld) by the
// whole block, one barrier per step: G[a][b] -= G[j][a] G[j][b] / G[j][j]
// for j < a <= b (row j is final once step j starts); then
// U[j][i] = G[j][i] / sqrt(G[j][j]).  In place (strict lower zeroed).
// Each thread owns fixed entries (precomputed, no per-step index math) and
// issues all loads of a step before its stores.  Returns false
// (block-uniform) on a non-positive pivot.
template <int NT, int KMAX>
__device__ bool block_chol(double* g, int ld, int R) {
    int pa[KMAX], pb[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        const int e = threadIdx.x + k * NT;
        const bool own = e < R * R && (e % R) >= (e / R);
        pa[k] = own ? e / R : 1 << 20;
        pb[k] = own ? e % R : 0;
    }
    bool ok = true;
    for (int j = 0; j < R; ++j) {
        // every load of the step first (they only depend on the barrier),
        // then the branch-free reciprocal of the pivot
        const double d = g[j * ld + j];
        double ga[KMAX], gb[KMAX], gab[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const bool act = pa[k] > j && pa[k] < R;
            ga[k] = act ? g[j * ld + pa[k]] : 0.0;
            gb[k] = act ? g[j * ld + pb[k]] : 0.0;
            gab[k] = act ? g[pa[k] * ld + pb[k]] : 0.0;
        }
        if (!(d > 0.0)) {
            ok = false;  // uniform: every thread read the same d
            break;
        }
        const double inv = rcp_nr(d);
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (pa[k] > j && pa[k] < R) g[pa[k] * ld + pb[k]] = fma(-ga[k] * inv, gb[k], gab[k]);
        __syncthreads();
    }
    if (!ok) {
        __syncthreads();
        return false;
    }
    __shared__ double rs[64];
#pragma unroll 1
    for (int j = threadIdx.x; j < R; j += NT) rs[j] = rsqrt(g[j * ld + j]);
    __syncthreads();
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += NT) {
        const int i = e / R, k = e % R;
        g[i * ld + k] = k >= i ? g[i * ld + k] * rs[i] : 0.0;
    }
    __syncthreads();
    return true;
}

// ---------------------------------------------------------------- register Cholesky
// Same factorisation and arithmetic as block_chol (bit-identical U), but the
// trailing matrix lives in REGISTERS of a small team (NTC = 2*RM threads,
// RM in {8,16,32,64}): thread t owns column b = t/2, rows a == t%2 (mod 2),
// a <= b.  Step j reads the published pivot row j from smem (2 distinct
// addresses per warp -> broadcasts), updates its entries, publishes row j+1
// and meets the team at a named barrier -- ~150 cycles per step instead of a
// full-block barrier and three smem round trips per entry.  Rows j are
// published exactly when final, so afterwards g holds G^(j)[j][b] and is
// scaled to U in place.  Called by all NT threads; block-uniform result.
template <int NT, int RM>
__device__ bool reg_chol(double* g, int ld, int R) {
    constexpr int NTC = 2 * RM < 32 ? 32 : 2 * RM;
    constexpr int E = (RM + 1) / 2;  // entries per thread
    static_assert(NTC <= NT, "reg_chol: team larger than the block");
    __shared__ int bad;
    const int t = threadIdx.x;
    if (t == 0) bad = 0;
    __syncthreads();
    if (t < NTC) {
        const int b = t >> 1, par = t & 1;
        double e[E];
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const int a = 2 * i + par;
            e[i] = (a <= b && b < R) ? g[a * ld + b] : 0.0;
        }
        for (int j = 0; j < R; ++j) {
            const double d = g[j * ld + j];
            if (!(d > 0.0)) {  // team-uniform (every thread read the same d)
                if (t == 0) bad = 1;
                break;
            }
            const double gb = b < R ? g[j * ld + b] : 0.0;  // G[j][b]
            const double inv = rcp_nr(d);
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const int a = 2 * i + par;
                if (a > j && a <= b && b < R) e[i] = fma(-g[j * ld + a] * inv, gb, e[i]);
            }
            // publish row j+1 (final after this step) for the next pivot
#pragma unroll
            for (int i = 0; i < E; ++i)
                if (2 * i + par == j + 1 && j + 1 <= b && b < R) g[(j + 1) * ld + b] = e[i];
            asm volatile("bar.sync 1, %0;" ::"r"(NTC) : "memory");
        }
    }
    __syncthreads();
    if (bad) return false;
    __shared__ double rs[64];
#pragma unroll 1
    for (int j = threadIdx.x; j < R; j += NT) rs[j] = rsqrt(g[j * ld + j]);
    __syncthreads();
#pragma unroll 1
    for (int x = threadIdx.x; x < R * R; x += NT) {
        const int i = x / R, k = x % R;
        g[i * ld + k] = k >= i ? g[i * ld + k] * rs[i] : 0.0;
    }
    __syncthreads();
    return true;
}

// Measured (tools/probes/chol2_probe.cu, one 256-thread CTA): block_chol is
// faster up to R = 32 (17.3k vs 23.4k cycles), reg_chol at R = 64 (76k vs 121k).
// A one-warp register Cholesky (tools/probes/chol3_probe.cu: warp_chol) is
// faster alone at R = 32 (14.5k vs 19.5k cycles) but 1.5-3.5x slower inside
// the solver while TTM kernels run concurrently on the other SMs
// (CPDB_PHASE_TRACE, C2: 5.2 us alone, 18.5 us beside the root TTM; block
// form 7.0 / 10.2 us), so the block-wide form stays.
template <int NT, int RM>
__device__ bool chol(double* g, int ld, int R) {
    if constexpr (RM >= 64) {
        return reg_chol<NT, RM>(g, ld, R);
    } else {
        return block_chol<NT, (RM * RM + NT - 1) / NT>(g, ld, R);
    }
}

// ---------------------------------------------------------------- first CholeskyQR pass
// Cholesky of the first pass's Gram G (R x R, stride R) of an m x R matrix
// with a shifted retry (shifted CholeskyQR, Fukaya-Kannan-Nakatsukasa-
// Yamamoto-Yanagisawa 2020): when G is numerically indefinite (kappa of the
// matrix beyond ~1e8, where the reference's Householder QR still works), G +
// s I with s = 11 (m R + R (R + 1)) u tr(G) is factored instead.  The
// second pass (near_identity_chol, or the pivoted chol when G2 is not close
// to I) then restores the orthogonality, so the run continues where
// CholeskyQR2 would stop.  copy: R x R scratch.  Block-uniform result: 0
// plain, 1 shifted, -1 breakdown even with the shift.
// status-word bit: a first pass needed the shifted retry (not an error)
constexpr int kStatusShifted = 1 << 16;

template <int NT, int RM>
__device__ int chol_first_pass(double* g, int R, uint64_t m, double* copy) {
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += NT) copy[e] = g[e];
    __syncthreads();
    if (chol<NT, RM>(g, R, R)) return 0;
    double tr = 0.0;
    for (int i = 0; i < R; ++i) tr += copy[i * R + i];
    const double sh =
        11.0 * (double(m) * R + double(R) * (R + 1)) * 1.1102230246251565e-16 * tr;
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += NT)
        g[e] = copy[e] + ((e / R == e % R) ? sh : 0.0);
    __syncthreads();
    return chol<NT, RM>(g, R, R) ? 1 : -1;
}

// ---------------------------------------------------------------- near-identity Cholesky
// The second CholeskyQR pass factors G = Q1^T Q1 = I + E with |E| ~ kappa^2
// eps (Q1 is already orthonormal to working accuracy).  Its Cholesky factor
// is U = I + X, X upper, with X + X^T + X^T X = E, i.e. the fixed point
//     X = up(E - X^T X),   up(S) = strict upper part of S + diag(S) / 2.
// From X_1 = up(E) every step multiplies the error by ~rho = 2 R max|E|, so
// the whole factorisation is a few R x R products (all entries in parallel)
// instead of an R-step pivot chain (block_chol: ~8 us at R = 32).  The step
// count is a deterministic function of max|E| (error <= 1e-18 absolute, far
// below the rounding of U's unit diagonal).  g (stride R) holds G on entry
// and U on exit (strict lower zeroed); xa, xb are R x R scratch.  Returns
// the number of products + 1, or 0 (block-uniform) when |E| is too large for
// the series: the caller then runs chol() on the untouched g.
template <int NT>
__device__ int near_identity_chol(double* g, int R, double* xa, double* xb, double* red) {
    double m = 0.0;
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += NT) {
        const int i = e / R, j = e % R;
        m = fmax(m, fabs(g[e] - (i == j ? 1.0 : 0.0)));
    }
    m = block_max<NT>(m, red);
    const double rho = 2.0 * double(R) * m;
    if (!(rho < 0.05)) return 0;  // (NaN lands here too)
    int steps = 1;
    for (double err = m * rho; err > 1e-18 && steps < 8; err *= rho) ++steps;
    if (steps >= 8) return 0;
    // X_1 = up(E)
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += NT) {
        const int i = e / R, j = e % R;
        xa[e] = i < j ? g[e] : (i == j ? 0.5 * (g[e] - 1.0) : 0.0);
    }
    __syncthreads();
    double* x = xa;
    double* xn = xb;
    for (int it = 1; it < steps; ++it) {
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += NT) {
            const int i = e / R, j = e % R;
            double v = 0.0;
            if (i <= j) {
                // (X^T X)_ij = sum_{p <= i} X[p][i] X[p][j]
                double s0 = 0.0, s1 = 0.0;
                int p = 0;
                for (; p + 1 <= i; p += 2) {
                    s0 = fma(x[p * R + i], x[p * R + j], s0);
                    s1 = fma(x[(p + 1) * R + i], x[(p + 1) * R + j], s1);
                }
                if (p <= i) s0 = fma(x[p * R + i], x[p * R + j], s0);
                const double s = g[e] - (i == j ? 1.0 : 0.0) - (s0 + s1);
                v = i < j ? s : 0.5 * s;
            }
            xn[e] = v;
        }
        __syncthreads();
        double* t = x;
        x = xn;
        xn = t;
    }
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += NT) {
        const int i = e / R, j = e % R;
        g[e] = i < j ? x[e] : (i == j ? 1.0 + x[e] : 0.0);
    }
    __syncthreads();
    return steps;
}

}  // namespace cpdb
