// Per-mode tail of a CP-ALS-QR update, single-CTA variant (used when the
// 8-CTA cluster kernel's shared-memory plan does not fit, e.g. very tall
// factors; the working matrix then lives in global memory / L2).  Same
// algorithm and building blocks as finish_cluster_kernel (cluster.cu):
//   A_hat = V R0^-T          row-wise triangular solve   (linalg.hpp:192-216)
//   lambda, A_n = A_hat / lambda                          (linalg.hpp:225-242)
//   Q_n, R_n = QR(A_n)       CholeskyQR2                  (factor_state.hpp:42-47)
//   packed Q_n, and on the last mode the fast-QR fitness  (kruskal.hpp:109-128)
#include <cmath>

#include "kernels.hpp"
#include "rowalg.cuh"

namespace cpdb {
namespace {

constexpr int kNT = 512;

template <int RM>
__global__ void __launch_bounds__(kNT) finish_single_kernel(FinishArgs a, int w_in_smem) {
    using Row = LaneRow<RM>;
    constexpr int T = Row::T, G = kNT / T;
    extern __shared__ double sm[];
    __shared__ double red[32];
    const int R = a.R, ld = R + 1;
    const int I = int(a.I);
    double* u = sm;            // RM x RM
    double* ut = u + RM * RM;  // RM x RM (transpose, for utinv)
    double* dinv = ut + RM * RM;
    double* vec = dinv + RM;
    double* g = vec + RM;      // R x R
    double* g1 = g + R * R;    // R x R (U1 kept for R_n)
    double* w = w_in_smem ? g1 + R * R : a.scratch;
    const int grp = threadIdx.x / T, q = threadIdx.x % T;
    const int Ipad = I + (G - I % G) % G;

    if (!a.init) {
        double mx = 0.0;
        for (int i = 0; i < R; ++i) mx = fmax(mx, fabs(a.r0[i * R + i]));
        for (int i = 0; i < R; ++i)
            if (fabs(a.r0[i * R + i]) <= 1e-14 * mx) {
                if (threadIdx.x == 0) *a.status = 1 | (i << 8);
                return;
            }
    }
    double xk_part = 0.0;
    if (!a.init) {
        stage_tri<RM>(a.r0, R, R, u, dinv, kNT);
        stage_tri_t<RM>(a.r0, R, R, ut, dinv, kNT);
        __syncthreads();
        for (int i = grp; i < Ipad; i += G) {
            const bool act = i < I;
            Row x;
            x.load(a.vpart + (act ? i : 0) * R, act ? R : 0, q);
            x.utinv(ut, dinv, R, q);
            if (a.fitness) {  // uniform: lane groups shuffle inside
                Row vf, wr;
                vf.load((a.dual ? a.vfitpart : a.vpart) + (act ? i : 0) * R, act ? R : 0, q);
                wr.set_times_upper(vf, u, R, q);
#pragma unroll
                for (int s = 0; s < Row::S; ++s) xk_part = fma(x.t[s], wr.t[s], xk_part);
            }
            if (act) x.store(w + i * ld, R, q);
        }
    } else {
#pragma unroll 1
        for (int e = threadIdx.x; e < I * R; e += kNT) w[(e / R) * ld + e % R] = a.a_out[e];
    }
    __syncthreads();
    gram_dmma<kNT>(w, ld, I, R, g, R);
    __syncthreads();
    if (!a.init) {
#pragma unroll 1
        for (int c = threadIdx.x; c < RM; c += kNT) {
            const double l = c < R ? sqrt(g[c * R + c]) : 0.0;
            vec[c] = l < 1e-300 ? 0.0 : __drcp_rn(l);
            if (c < R) a.lambda[c] = l < 1e-300 ? 0.0 : l;
        }
        __syncthreads();
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) {
            const double li = vec[e / R], lj = vec[e % R];
            g[e] = (li == 0.0 || lj == 0.0) ? (e / R == e % R ? 1.0 : 0.0) : g[e] * li * lj;
        }
        __syncthreads();
    }
    const int fp = chol_first_pass<kNT, RM>(g, R, I, g1);
    if (fp < 0) {
        if (threadIdx.x == 0) *a.status = 2;
        return;
    }
    if (fp == 1 && threadIdx.x == 0) atomicOr(a.status, kStatusShifted);
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) g1[e] = g[e];
    stage_tri<RM>(g, R, R, u, dinv, kNT);
    __syncthreads();
    for (int i = grp; i < Ipad; i += G) {
        const bool act = i < I;
        Row x;
        x.load(w + (act ? i : 0) * ld, act ? R : 0, q);
        if (!a.init) {
#pragma unroll
            for (int s = 0; s < Row::S; ++s) {
                const int k = s * T + q;
                if (k < R) {
                    const double il = vec[k];
                    x.t[s] = il == 0.0 ? (i == 0 ? 1.0 : 0.0) : x.t[s] * il;
                }
            }
            if (act) x.store(a.a_out + i * R, R, q);
        }
        x.uinv(u, dinv, R, q);
        if (act) x.store(w + i * ld, R, q);
    }
    __syncthreads();
    gram_dmma<kNT>(w, ld, I, R, g, R);
    __syncthreads();
    if (!chol<kNT, RM>(g, R, R)) {
        if (threadIdx.x == 0) *a.status = 2;
        return;
    }
    stage_tri<RM>(g, R, R, u, dinv, kNT);
    __syncthreads();
    const uint32_t Rp = ttm_rpad_dev(R);
    for (int i = grp; i < Ipad; i += G) {
        const bool act = i < I;
        Row x;
        x.load(w + (act ? i : 0) * ld, act ? R : 0, q);
        x.uinv(u, dinv, R, q);
        if (act) {
            x.store(a.q_out + uint64_t(i) * R, R, q);
            double* qp = a.qp_out + ((uint64_t(i) >> 2) * Rp) * 4 + (i & 3);
#pragma unroll
            for (int s = 0; s < Row::S; ++s) {
                const int k = s * T + q;
                if (k < int(Rp)) qp[k * 4] = k < R ? x.t[s] : 0.0;
            }
        }
    }
    const uint64_t Kpad = ((uint64_t(I) + 31) / 32) * 32;
    for (uint64_t e = uint64_t(I) * Rp + threadIdx.x; e < Kpad * Rp; e += kNT) {
        const uint64_t k = e / Rp, r = e % Rp;
        a.qp_out[((k >> 2) * Rp + r) * 4 + (k & 3)] = 0.0;
    }
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) {
        const int i = e / R, j = e % R;
        double s = 0.0;
        for (int p = i; p <= j; ++p) s = fma(g[i * R + p], g1[p * R + j], s);
        a.r_out[e] = i <= j ? s : 0.0;
    }
    __syncthreads();
    if (a.fitness && !a.init) {
        double s = 0.0;
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) {
            const int i = e / R, j = e % R;
            double p0 = 0.0, pn = 0.0;
            const int top = i < j ? i : j;
            for (int p = 0; p <= top; ++p) {
                p0 = fma(a.r0[p * R + i], a.r0[p * R + j], p0);
                pn = fma(a.r_out[p * R + i], a.r_out[p * R + j], pn);
            }
            s += p0 * a.lambda[i] * pn * a.lambda[j];
        }
        const double kk = block_sum<kNT>(s, red);
        const double xk = block_sum<kNT>(xk_part, red);
        if (threadIdx.x == 0) {
            const double raw = a.norm_x_sq - 2.0 * xk + kk;
            const double rad = raw < 0.0 ? 0.0 : raw;
            a.fit_out[0] = 1.0 - sqrt(rad) / sqrt(a.norm_x_sq);
            a.fit_out[1] = raw;
        }
    }
}

template <int RM>
cudaError_t run_single(const FinishArgs& a, cudaStream_t s) {
    const size_t base = (2 * size_t(RM) * RM + 2 * RM + 2 * size_t(a.R) * a.R) * sizeof(double);
    const size_t wbytes = a.I * (a.R + 1) * sizeof(double);
    const bool in_smem = base + wbytes <= 210 * 1024;
    if (!in_smem && a.scratch == nullptr) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(finish_single_kernel<RM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 215 * 1024);
    if (e != cudaSuccess) return e;
    finish_single_kernel<RM><<<1, kNT, base + (in_smem ? wbytes : 0), s>>>(a, in_smem ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace

bool finish_sums_splits(uint64_t I, uint32_t R) {
    return !wide_rank(R) && finish_cluster_smem(I, R) <= 220 * 1024;
}

cudaError_t launch_finish(const FinishArgs& a, cudaStream_t s) {
    if (wide_rank(a.R) || a.householder) return launch_finish_wide(a, s);
    // the 8-CTA cluster kernel (cluster.cu) whenever its smem plan fits
    if (finish_cluster_smem(a.I, a.R) <= 220 * 1024) return launch_finish_cluster(a, s);
    return launch_finish_single(a, s);
}

cudaError_t launch_finish_single(const FinishArgs& a, cudaStream_t s) {
    if (a.R <= 8) return run_single<8>(a, s);
    if (a.R <= 16) return run_single<16>(a, s);
    if (a.R <= 32) return run_single<32>(a, s);
    if (a.R <= 64) return run_single<64>(a, s);
    return cudaErrorInvalidValue;
}

}  // namespace cpdb
