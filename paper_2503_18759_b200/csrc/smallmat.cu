// K3-K6: the small-matrix side of a CP-ALS-QR mode update, plus reductions.
//
//   launch_zqr     Khatri-Rao(R_k) + QR  (tensor.hpp:343-368 + linalg.hpp:39-99
//                  at solvers.hpp:250-255), structured CholeskyQR2
//   launch_vgemm   V = unfold(Y,n) * Q0_hat, extrapolation fused into the
//                  operand load (solvers.hpp:260-271, 277-284)
//   launch_finish  A_hat = V R0^-T, normalise, factor QR, pack, fitness
//                  (solvers.hpp:272-275, factor_state.hpp:42-47,
//                   kruskal.hpp:109-128)
//   norm_sq        inner(x, x) (tensor.hpp:394-399)
// All reductions use fixed partitions and fixed trees: repeated runs are
// bit-identical (solver_test.cpp:272-282 requires it).
#include <algorithm>
#include <cmath>

#include "device.cuh"
#include "kernels.hpp"

namespace cpdb {
namespace {

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

// ------------------------------------------------------------------ norms
constexpr int kNormThreads = 256;

__global__ void __launch_bounds__(kNormThreads)
sumprod_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, uint64_t n,
                       double* __restrict__ partials) {
    __shared__ double red[32];
    double s0 = 0.0, s1 = 0.0;
    const uint64_t pairs = n / 2;
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* b2 = reinterpret_cast<const double2*>(b);
    const uint64_t stride = uint64_t(kNormBlocks) * kNormThreads;
    for (uint64_t i = uint64_t(blockIdx.x) * kNormThreads + threadIdx.x; i < pairs; i += stride) {
        const double2 u = a2[i], v = b2[i];
        s0 = fma(u.x, v.x, s0);
        s1 = fma(u.y, v.y, s1);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) s0 = fma(a[n - 1], b[n - 1], s0);
    const double s = block_sum<kNormThreads>(s0 + s1, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) sum_final_kernel(const double* __restrict__ partials,
                                                         int n, double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 1024) s += partials[i];
    s = block_sum<1024>(s, red);
    if (threadIdx.x == 0) *out = s;
}

// ------------------------------------------------------------------ dense helpers
// Right-looking Cholesky of the symmetric R x R matrix in g (row-major,
// leading dim ld), in place: the upper triangle becomes U with U^T U = G.
// The strict lower triangle is zeroed.  Returns false on a non-positive pivot.
template <int NT>
__device__ bool chol_upper(double* g, int R, int ld, int* flag) {
    for (int j = 0; j < R; ++j) {
        if (threadIdx.x == 0) {
            const double d = g[j * ld + j];
            if (!(d > 0.0)) *flag = 1;
            g[j * ld + j] = sqrt(d > 0.0 ? d : 0.0);
        }
        __syncthreads();
        if (*flag) return false;
        const double piv = g[j * ld + j];
        for (int i = j + 1 + threadIdx.x; i < R; i += NT) g[j * ld + i] /= piv;
        __syncthreads();
        const int m = R - j - 1;
        for (int e = threadIdx.x; e < m * m; e += NT) {
            const int a = j + 1 + e / m, b = j + 1 + e % m;
            if (a <= b) g[a * ld + b] -= g[j * ld + a] * g[j * ld + b];
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < R * R; e += NT)
        if (e / R > e % R) g[(e / R) * ld + e % R] = 0.0;
    __syncthreads();
    return true;
}

// Inverse of an upper-triangular R x R matrix u (ld) into x (ld), one column
// per thread, back substitution with the column kept in x.
template <int NT>
__device__ void inv_upper(const double* u, double* x, int R, int ld) {
    for (int c = threadIdx.x; c < R; c += NT) {
        for (int i = 0; i < R; ++i) x[i * ld + c] = 0.0;
        x[c * ld + c] = 1.0 / u[c * ld + c];
        for (int i = c - 1; i >= 0; --i) {
            double s0 = 0.0, s1 = 0.0;
            int p = i + 1;
            for (; p + 1 <= c; p += 2) {
                s0 = fma(u[i * ld + p], x[p * ld + c], s0);
                s1 = fma(u[i * ld + p + 1], x[(p + 1) * ld + c], s1);
            }
            if (p <= c) s0 = fma(u[i * ld + p], x[p * ld + c], s0);
            x[i * ld + c] = -(s0 + s1) / u[i * ld + i];
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ Z-QR
constexpr int kZThreads = 256;
constexpr int kZTile = 64;  // rows per tile in the row kernels

size_t zqr_smem_mats(uint32_t nm, uint32_t R) { return size_t(nm) * R * R; }

// work layout (doubles): [R1 | R1inv | R2inv | partial G2 x grid]
__global__ void __launch_bounds__(kZThreads)
zqr_prep_kernel(ZqrArgs a) {
    extern __shared__ double sm[];
    const int R = a.R, nm = a.nm;
    double* g = sm;            // R x R
    double* x = g + R * R;     // R x R
    __shared__ int flag;
    if (threadIdx.x == 0) flag = 0;
    // G1 = hadamard_t (R_t^T R_t)
    for (int e = threadIdx.x; e < R * R; e += kZThreads) {
        const int p = e / R, q = e % R;
        double h = 1.0;
        if (p <= q) {
            for (int t = nm - 1; t >= 0; --t) {
                const double* m = a.rmats[t];
                double s = 0.0;
                for (int k = 0; k <= p; ++k) s = fma(m[k * R + p], m[k * R + q], s);  // upper
                h *= s;
            }
            g[p * R + q] = h;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += kZThreads) {
        const int p = e / R, q = e % R;
        if (p > q) g[p * R + q] = g[q * R + p];
    }
    __syncthreads();
    if (!chol_upper<kZThreads>(g, R, R, &flag)) {
        if (threadIdx.x == 0) *a.status = 2;
        return;
    }
    inv_upper<kZThreads>(g, x, R, R);
    for (int e = threadIdx.x; e < R * R; e += kZThreads) {
        a.work[e] = g[e];              // R1
        a.work[R * R + e] = x[e];      // R1inv
    }
}

// Q1 = Z R1inv with Z rows generated on the fly; per-block partial G2 = Q1^T Q1.
template <int RM>
__global__ void __launch_bounds__(kZThreads)
zqr_rows_kernel(ZqrArgs a) {
    extern __shared__ double sm[];
    const int R = a.R, nm = a.nm;
    double* mats = sm;                            // nm x R x R
    double* rinv = mats + nm * R * R;             // R x R
    double* zt = rinv + R * R;                    // kZTile x (R+1)
    const int ld = R + 1;
    for (int e = threadIdx.x; e < nm * R * R; e += kZThreads)
        mats[e] = a.rmats[e / (R * R)][e % (R * R)];
    for (int e = threadIdx.x; e < R * R; e += kZThreads) rinv[e] = a.work[R * R + e];
    constexpr int PER = (RM * RM + kZThreads - 1) / kZThreads;
    double g2[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) g2[u] = 0.0;
    __syncthreads();
    const uint64_t ntiles = (a.zrows + kZTile - 1) / kZTile;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t row0 = tile * kZTile;
        // Z tile (natural order; product over modes descending like the
        // reference Khatri-Rao fold)
        for (int e = threadIdx.x; e < kZTile * R; e += kZThreads) {
            const int rr = e / R, c = e % R;
            const uint64_t row = row0 + rr;
            double z = 0.0;
            if (row < a.zrows) {
                uint64_t rem = row;
                double prod = 1.0;
                // digit of mats[t]: t = nm-1 is the fastest
                uint64_t digits[8];
                for (int t = nm - 1; t >= 0; --t) {
                    digits[t] = rem % R;
                    rem /= R;
                }
                for (int t = nm - 1; t >= 0; --t) {
                    const double v = mats[(t * R + digits[t]) * R + c];
                    prod = (t == nm - 1) ? v : prod * v;
                }
                z = prod;
            }
            zt[rr * ld + c] = z;
        }
        __syncthreads();
        // Q1 tile = Z tile * R1inv (upper): q[rr][c] = sum_{p<=c} z[rr][p] rinv[p][c]
        double qv[(kZTile * RM + kZThreads - 1) / kZThreads];
        int nq = 0;
        for (int e = threadIdx.x; e < kZTile * R; e += kZThreads, ++nq) {
            const int rr = e / R, c = e % R;
            double s = 0.0;
            for (int p = 0; p <= c; ++p) s = fma(zt[rr * ld + p], rinv[p * R + c], s);
            qv[nq] = s;
        }
        __syncthreads();
        nq = 0;
        for (int e = threadIdx.x; e < kZTile * R; e += kZThreads, ++nq) {
            const int rr = e / R, c = e % R;
            zt[rr * ld + c] = qv[nq];
            const uint64_t row = row0 + rr;
            if (row < a.zrows) a.q1[row * R + c] = qv[nq];
        }
        __syncthreads();
        const int rows = (a.zrows - row0 < uint64_t(kZTile)) ? int(a.zrows - row0) : kZTile;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int e = threadIdx.x + u * kZThreads;
            if (e < R * R) {
                const int p = e / R, q = e % R;
                double s = g2[u];
                for (int rr = 0; rr < rows; ++rr) s = fma(zt[rr * ld + p], zt[rr * ld + q], s);
                g2[u] = s;
            }
        }
        __syncthreads();
    }
    double* part = a.work + 3 * R * R + size_t(blockIdx.x) * R * R;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int e = threadIdx.x + u * kZThreads;
        if (e < R * R) part[e] = g2[u];
    }
}

__global__ void __launch_bounds__(kZThreads)
zqr_fin_kernel(ZqrArgs a, int nparts) {
    extern __shared__ double sm[];
    const int R = a.R;
    double* g = sm;          // G2 -> R2
    double* x = g + R * R;   // R2inv
    double* r1 = x + R * R;  // R1
    __shared__ int flag;
    if (threadIdx.x == 0) flag = 0;
    for (int e = threadIdx.x; e < R * R; e += kZThreads) {
        double s = 0.0;
        for (int b = 0; b < nparts; ++b) s += a.work[3 * R * R + size_t(b) * R * R + e];
        g[e] = s;
        r1[e] = a.work[e];
    }
    __syncthreads();
    if (!chol_upper<kZThreads>(g, R, R, &flag)) {
        if (threadIdx.x == 0) *a.status = 2;
        return;
    }
    inv_upper<kZThreads>(g, x, R, R);
    for (int e = threadIdx.x; e < R * R; e += kZThreads) {
        const int i = e / R, j = e % R;
        double s = 0.0;
        for (int p = i; p <= j; ++p) s = fma(g[i * R + p], r1[p * R + j], s);
        a.r0[e] = (i <= j) ? s : 0.0;
        a.work[2 * R * R + e] = x[e];  // R2inv
    }
}

// Q0 = Q1 * R2inv
__global__ void __launch_bounds__(kZThreads)
zqr_apply_kernel(ZqrArgs a) {
    extern __shared__ double sm[];
    const int R = a.R, ld = R + 1;
    double* x = sm;              // R2inv
    double* t = x + R * R;       // kZTile x (R+1)
    for (int e = threadIdx.x; e < R * R; e += kZThreads) x[e] = a.work[2 * R * R + e];
    const uint64_t ntiles = (a.zrows + kZTile - 1) / kZTile;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t row0 = tile * kZTile;
        __syncthreads();
        for (int e = threadIdx.x; e < kZTile * R; e += kZThreads) {
            const uint64_t row = row0 + e / R;
            t[(e / R) * ld + e % R] = row < a.zrows ? a.q1[row * R + e % R] : 0.0;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kZTile * R; e += kZThreads) {
            const int rr = e / R, c = e % R;
            const uint64_t row = row0 + rr;
            if (row >= a.zrows) continue;
            double s = 0.0;
            for (int p = 0; p <= c; ++p) s = fma(t[rr * ld + p], x[p * R + c], s);
            a.q0[row * R + c] = s;
        }
    }
}

// ------------------------------------------------------------------ V-GEMM
constexpr int kVThreads = 256;
constexpr int kVBI = 64;  // rows of V per block
constexpr int kVBK = 16;  // k per smem tile

template <int RM, bool DUAL>
__global__ void __launch_bounds__(kVThreads)
vgemm_kernel(VgemmArgs a, uint64_t kchunk) {
    __shared__ double yt[kVBI][kVBK + 1];
    __shared__ double pt[kVBK][RM];
    __shared__ double ft[DUAL ? kVBK : 1][RM];
    const int R = a.R;
    const uint64_t I = a.I, J = a.J, K = a.O * a.J;
    const uint64_t i0 = uint64_t(blockIdx.x) * kVBI;
    const uint64_t kb = uint64_t(blockIdx.y) * kchunk;
    const uint64_t ke = min(K, kb + kchunk);
    const int ii = threadIdx.x % kVBI, rg = threadIdx.x / kVBI;  // rg in [0,4)
    constexpr int RPT = RM / 4;                                    // r per thread
    double acc[RPT], accf[DUAL ? RPT : 1];
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc[u] = 0.0;
#pragma unroll
    for (int u = 0; u < (DUAL ? RPT : 1); ++u) accf[u] = 0.0;
    const bool jfast = J >= kVBK;
    for (uint64_t k0 = kb; k0 < ke; k0 += kVBK) {
        for (int e = threadIdx.x; e < kVBI * kVBK; e += kVThreads) {
            int r_, c_;
            if (jfast) {
                r_ = e / kVBK;
                c_ = e % kVBK;
            } else {
                r_ = e % kVBI;
                c_ = e / kVBI;
            }
            const uint64_t k = k0 + c_, i = i0 + r_;
            double v = 0.0;
            if (k < ke && i < I) {
                const uint64_t o = k / J, j = k % J;
                v = a.y[(o * I + i) * J + j];
            }
            yt[r_][c_] = v;
        }
        for (int e = threadIdx.x; e < kVBK * RM; e += kVThreads) {
            const int kk = e / RM, r = e % RM;
            const uint64_t k = k0 + kk;
            double q = 0.0, p = 0.0;
            if (k < ke && r < R) {
                q = a.q0[k * R + r];
                p = q;
                if (a.extrap) p = q + a.beta * (q - a.alpha * a.hist[k * R + r]);
            }
            pt[kk][r] = p;
            if (DUAL) ft[kk][r] = q;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < kVBK; ++kk) {
            const double yv = yt[ii][kk];
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                acc[u] = fma(yv, pt[kk][rg + 4 * u], acc[u]);
                if (DUAL) accf[u] = fma(yv, ft[kk][rg + 4 * u], accf[u]);
            }
        }
        __syncthreads();
    }
    const uint64_t i = i0 + ii;
    if (i < I) {
        double* vp = a.vpart + (uint64_t(blockIdx.y) * I + i) * R;
        double* fp = DUAL ? a.vfitpart + (uint64_t(blockIdx.y) * I + i) * R : nullptr;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int r = rg + 4 * u;
            if (r < R) {
                vp[r] = acc[u];
                if (DUAL) fp[r] = accf[u];
            }
        }
    }
}

// ------------------------------------------------------------------ finisher
constexpr int kFThreads = 512;

template <int NT>
__device__ void gram_upper(const double* w, int ld, uint64_t I, int R, double* g) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int E = R * (R + 1) / 2;
    for (int e = warp; e < E; e += NT / 32) {
        // map e -> (p, q), p <= q
        int p = 0, rem = e;
        while (rem >= R - p) {
            rem -= R - p;
            ++p;
        }
        const int q = p + rem;
        double s = 0.0;
        for (uint64_t i = lane; i < I; i += 32) s = fma(w[i * ld + p], w[i * ld + q], s);
        s = warp_sum(s);
        if (lane == 0) {
            g[p * R + q] = s;
            g[q * R + p] = s;
        }
    }
    __syncthreads();
}

// rows of w <- rows of w * U^-1 (forward substitution, U upper), in place
template <int NT>
__device__ void rows_times_uinv(double* w, int ld, uint64_t I, int R, const double* u) {
    for (uint64_t i = threadIdx.x; i < I; i += NT) {
        double* row = w + i * ld;
        for (int j = 0; j < R; ++j) {
            double s0 = row[j], s1 = 0.0;
            int p = 0;
            for (; p + 1 < j; p += 2) {
                s0 = fma(-row[p], u[p * R + j], s0);
                s1 = fma(-row[p + 1], u[(p + 1) * R + j], s1);
            }
            if (p < j) s0 = fma(-row[p], u[p * R + j], s0);
            row[j] = (s0 + s1) / u[j * R + j];
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kFThreads)
finish_kernel(FinishArgs a, int w_in_smem) {
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ int flag;
    const int R = a.R, ld = R + 1;
    const uint64_t I = a.I;
    double* r0 = sm;              // R x R
    double* g1 = r0 + R * R;      // R x R  (gram -> R1)
    double* g2 = g1 + R * R;      // R x R  (gram -> R2)
    double* rowpart = g2 + R * R; // I
    double* w = w_in_smem ? rowpart + I : a.scratch;
    if (threadIdx.x == 0) flag = 0;

    double xk = 0.0;
    if (!a.init) {
        for (int e = threadIdx.x; e < R * R; e += kFThreads) r0[e] = a.r0[e];
        const uint64_t n = I * R;
        for (uint64_t e = threadIdx.x; e < n; e += kFThreads) {
            double s = 0.0, f = 0.0;
            for (uint32_t p = 0; p < a.nsplit; ++p) {
                s += a.vpart[p * n + e];
                if (a.dual) f += a.vfitpart[p * n + e];
            }
            w[(e / R) * ld + e % R] = s;
            a.v_out[e] = a.dual ? f : s;
        }
        __syncthreads();
        // singular check (linalg.hpp:199-203)
        if (threadIdx.x == 0) {
            double mx = 0.0;
            for (int i = 0; i < R; ++i) mx = fmax(mx, fabs(r0[i * R + i]));
            const double tau = 1e-14 * mx;
            for (int i = 0; i < R; ++i)
                if (fabs(r0[i * R + i]) <= tau) {
                    *a.status = 1 | (i << 8);
                    flag = 1;
                    break;
                }
        }
        __syncthreads();
        if (flag) return;
        // A_hat rows: x R0^T = v  (L = R0^T, L[j][c] = R0[c][j]); back substitution
        for (uint64_t i = threadIdx.x; i < I; i += kFThreads) {
            double* row = w + i * ld;
            for (int c = R - 1; c >= 0; --c) {
                double s = row[c];
                for (int j = c + 1; j < R; ++j) s = fma(-row[j], r0[c * R + j], s);
                row[c] = s / r0[c * R + c];
            }
            if (a.fitness) {
                // <V, A_hat R0^T> restricted to row i
                const double* v = a.v_out + i * R;
                double t = 0.0;
                for (int j = 0; j < R; ++j) {
                    double m = 0.0;
                    for (int p = j; p < R; ++p) m = fma(row[p], r0[j * R + p], m);
                    t = fma(v[j], m, t);
                }
                rowpart[i] = t;
            }
        }
        __syncthreads();
        if (a.fitness) {
            double s = 0.0;
            for (uint64_t i = threadIdx.x; i < I; i += kFThreads) s += rowpart[i];
            xk = block_sum<kFThreads>(s, red);  // valid in warp 0
        }
        // column norms -> lambda (linalg.hpp:225-242)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int c = warp; c < R; c += kFThreads / 32) {
            double s = 0.0;
            for (uint64_t i = lane; i < I; i += 32) s = fma(w[i * ld + c], w[i * ld + c], s);
            s = warp_sum(s);
            if (lane == 0) g1[c] = sqrt(s);
        }
        __syncthreads();
        for (uint64_t e = threadIdx.x; e < I * R; e += kFThreads) {
            const uint64_t i = e / R;
            const int c = int(e % R);
            const double nrm = g1[c];
            double v;
            if (nrm < 1e-300) v = (i == 0) ? 1.0 : 0.0;
            else v = w[i * ld + c] / nrm;
            w[i * ld + c] = v;
            a.a_out[e] = v;
        }
        for (int c = threadIdx.x; c < R; c += kFThreads) a.lambda[c] = g1[c] < 1e-300 ? 0.0 : g1[c];
        __syncthreads();
    } else {
        for (uint64_t e = threadIdx.x; e < I * R; e += kFThreads) w[(e / R) * ld + e % R] = a.a_out[e];
        __syncthreads();
    }

    // CholQR2 of the factor (factor_state.hpp:42-47 re-QR)
    gram_upper<kFThreads>(w, ld, I, R, g1);
    if (!chol_upper<kFThreads>(g1, R, R, &flag)) {
        if (threadIdx.x == 0) *a.status = 2;
        return;
    }
    rows_times_uinv<kFThreads>(w, ld, I, R, g1);
    gram_upper<kFThreads>(w, ld, I, R, g2);
    if (!chol_upper<kFThreads>(g2, R, R, &flag)) {
        if (threadIdx.x == 0) *a.status = 2;
        return;
    }
    rows_times_uinv<kFThreads>(w, ld, I, R, g2);
    // R_n = R2 R1 (kept in rowpart-free smem: reuse g1 after product)
    double rn_local[(64 * 64 + kFThreads - 1) / kFThreads];
    int nr = 0;
    for (int e = threadIdx.x; e < R * R; e += kFThreads, ++nr) {
        const int i = e / R, j = e % R;
        double s = 0.0;
        for (int p = i; p <= j; ++p) s = fma(g2[i * R + p], g1[p * R + j], s);
        rn_local[nr] = i <= j ? s : 0.0;
    }
    __syncthreads();
    nr = 0;
    for (int e = threadIdx.x; e < R * R; e += kFThreads, ++nr) {
        g1[e] = rn_local[nr];
        a.r_out[e] = rn_local[nr];
    }
    // Q_n and its packed copy ([Kpad/4][Rp][4], zero padded)
    const uint32_t Rp = ttm_rpad_dev(R);
    const uint64_t Kpad = ((I + 31) / 32) * 32;
    for (uint64_t e = threadIdx.x; e < I * R; e += kFThreads) a.q_out[e] = w[(e / R) * ld + e % R];
    for (uint64_t idx = threadIdx.x; idx < Kpad * Rp; idx += kFThreads) {
        const uint64_t kq = idx % 4, r = (idx / 4) % Rp, kg = idx / (4 * Rp);
        const uint64_t k = kg * 4 + kq;
        a.qp_out[idx] = (k < I && r < uint64_t(R)) ? w[k * ld + r] : 0.0;
    }
    __syncthreads();

    if (a.fitness && !a.init) {
        // ||K||^2 = sum_ij (R0^T R0)_ij l_i (Rn^T Rn)_ij l_j   (kruskal.hpp:457-462)
        double s = 0.0;
        for (int e = threadIdx.x; e < R * R; e += kFThreads) {
            const int i = e / R, j = e % R;
            double p0 = 0.0, pn = 0.0;
            const int top = min(i, j);
            for (int p = 0; p <= top; ++p) {
                p0 = fma(r0[p * R + i], r0[p * R + j], p0);
                pn = fma(g1[p * R + i], g1[p * R + j], pn);
            }
            s += p0 * a.lambda[i] * pn * a.lambda[j];
        }
        const double kk = block_sum<kFThreads>(s, red);
        if (threadIdx.x == 0) {
            const double raw = a.norm_x_sq - 2.0 * xk + kk;
            const double rad = raw < 0.0 ? 0.0 : raw;
            a.fit_out[0] = 1.0 - sqrt(rad) / sqrt(a.norm_x_sq);
            a.fit_out[1] = raw;
        }
    }
}

// ------------------------------------------------------------------ misc kernels
__global__ void normalize_exact_kernel(double* a, uint64_t m, uint32_t n, double* weights) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double s = 0.0;
    for (uint64_t i = 0; i < m; ++i) s = __dadd_rn(s, __dmul_rn(a[i * n + c], a[i * n + c]));
    const double nrm = __dsqrt_rn(s);
    if (nrm < 1e-300) {
        for (uint64_t i = 0; i < m; ++i) a[i * n + c] = i == 0 ? 1.0 : 0.0;
        if (weights) weights[c] = 0.0;
    } else {
        for (uint64_t i = 0; i < m; ++i) a[i * n + c] = __ddiv_rn(a[i * n + c], nrm);
        if (weights) weights[c] = nrm;
    }
}

// Householder thin QR with the reference's conventions (alpha = -sign ||x||,
// backward Q accumulation, nonnegative diag(R)); one CTA, work = m*n + m*n + n.
__global__ void __launch_bounds__(256)
householder_kernel(const double* a, uint64_t m, uint32_t n, double* work, double* q, double* r) {
    __shared__ double red[32];
    __shared__ double sh_alpha, sh_beta;
    __shared__ int sh_skip;
    double* w = work;              // m x n
    double* v = work + m * n;      // reflectors, column-major by k: v_k at v + k*m
    double* betas = v + m * n;     // n
    for (uint64_t e = threadIdx.x; e < m * n; e += 256) w[e] = a[e];
    __syncthreads();
    for (uint32_t k = 0; k < n; ++k) {
        double s = 0.0;
        for (uint64_t i = k + threadIdx.x; i < m; i += 256) s = fma(w[i * n + k], w[i * n + k], s);
        s = block_sum<256>(s, red);
        if (threadIdx.x == 0) {
            const double nrm = sqrt(s);
            sh_skip = nrm == 0.0;
            sh_alpha = w[k * n + k] >= 0.0 ? -nrm : nrm;
        }
        __syncthreads();
        if (sh_skip) {
            if (threadIdx.x == 0) betas[k] = 0.0;
            __syncthreads();
            continue;
        }
        double* vk = v + uint64_t(k) * m;
        for (uint64_t i = k + threadIdx.x; i < m; i += 256)
            vk[i - k] = (i == k) ? w[k * n + k] - sh_alpha : w[i * n + k];
        __syncthreads();
        double vs = 0.0;
        for (uint64_t i = threadIdx.x; i < m - k; i += 256) vs = fma(vk[i], vk[i], vs);
        vs = block_sum<256>(vs, red);
        if (threadIdx.x == 0) sh_beta = 2.0 / vs;
        __syncthreads();
        const double beta = sh_beta;
        for (uint32_t j = k; j < n; ++j) {
            double d = 0.0;
            for (uint64_t i = k + threadIdx.x; i < m; i += 256) d = fma(vk[i - k], w[i * n + j], d);
            d = block_sum<256>(d, red);
            if (threadIdx.x == 0) red[31] = d * beta;
            __syncthreads();
            const double sc = red[31];
            for (uint64_t i = k + threadIdx.x; i < m; i += 256) w[i * n + j] -= sc * vk[i - k];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            w[k * n + k] = sh_alpha;
            betas[k] = beta;
        }
        __syncthreads();
    }
    for (uint64_t e = threadIdx.x; e < uint64_t(n) * n; e += 256) {
        const uint64_t i = e / n, j = e % n;
        r[e] = j >= i ? w[i * n + j] : 0.0;
    }
    for (uint64_t e = threadIdx.x; e < m * n; e += 256) q[e] = (e / n == e % n) ? 1.0 : 0.0;
    __syncthreads();
    for (int k = int(n) - 1; k >= 0; --k) {
        const double beta = betas[k];
        if (beta == 0.0) continue;
        const double* vk = v + uint64_t(k) * m;
        for (uint32_t j = 0; j < n; ++j) {
            double d = 0.0;
            for (uint64_t i = k + threadIdx.x; i < m; i += 256) d = fma(vk[i - k], q[i * n + j], d);
            d = block_sum<256>(d, red);
            if (threadIdx.x == 0) red[31] = d * beta;
            __syncthreads();
            const double sc = red[31];
            for (uint64_t i = k + threadIdx.x; i < m; i += 256) q[i * n + j] -= sc * vk[i - k];
            __syncthreads();
        }
    }
    __syncthreads();
    for (uint32_t k = 0; k < n; ++k) {
        const bool neg = r[uint64_t(k) * n + k] < 0.0;
        __syncthreads();
        if (neg) {
            for (uint32_t j = k + threadIdx.x; j < n; j += 256) r[uint64_t(k) * n + j] = -r[uint64_t(k) * n + j];
            for (uint64_t i = threadIdx.x; i < m; i += 256) q[i * n + k] = -q[i * n + k];
        }
        __syncthreads();
    }
}

__global__ void reduce_splits_kernel(const double* part, uint32_t nsplit, uint64_t n,
                                     double* out) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (uint32_t p = 0; p < nsplit; ++p) s += part[p * n + e];
        out[e] = s;
    }
}

__global__ void permute_rows_kernel(const double* in, double* out, const uint64_t* perm,
                                    uint64_t rows, uint32_t w) {
    const uint64_t n = rows * w;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x)
        out[e] = in[perm[e / w] * w + e % w];
}

template <int RM>
cudaError_t zqr_run(const ZqrArgs& a, cudaStream_t s, int sms) {
    const int R = a.R;
    const size_t prep = 2 * size_t(R) * R * sizeof(double);
    zqr_prep_kernel<<<1, kZThreads, prep, s>>>(a);
    const size_t rows_smem = (size_t(a.nm) * R * R + R * R + kZTile * (R + 1)) * sizeof(double);
    auto rk = zqr_rows_kernel<RM>;
    static bool cfg = false;
    if (!cfg) {
        cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(zqr_fin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(zqr_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(zqr_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cfg = true;
    }
    const uint64_t ntiles = (a.zrows + kZTile - 1) / kZTile;
    const int grid = int(std::min<uint64_t>(ntiles, uint64_t(2 * sms)));
    rk<<<grid, kZThreads, rows_smem, s>>>(a);
    zqr_fin_kernel<<<1, kZThreads, 3 * size_t(R) * R * sizeof(double), s>>>(a, grid);
    const size_t ap = (size_t(R) * R + kZTile * (R + 1)) * sizeof(double);
    zqr_apply_kernel<<<grid, kZThreads, ap, s>>>(a);
    return cudaGetLastError();
}

template <int RM, bool DUAL>
cudaError_t vgemm_run(VgemmArgs& a, cudaStream_t s, int sms) {
    const uint64_t K = a.O * a.J;
    const uint64_t iblocks = (a.I + kVBI - 1) / kVBI;
    const uint64_t ktiles = (K + kVBK - 1) / kVBK;
    uint64_t nsplit = std::max<uint64_t>(1, (2 * uint64_t(sms)) / iblocks);
    nsplit = std::min<uint64_t>({nsplit, ktiles, uint64_t(vgemm_max_split())});
    const uint64_t kchunk = ((ktiles + nsplit - 1) / nsplit) * kVBK;
    nsplit = (K + kchunk - 1) / kchunk;
    a.nsplit = uint32_t(nsplit);
    const dim3 grid{unsigned(iblocks), unsigned(nsplit), 1u};
    vgemm_kernel<RM, DUAL><<<grid, kVThreads, 0, s>>>(a, kchunk);
    return cudaGetLastError();
}

}  // namespace

cudaError_t norm_sq(const double* x, uint64_t n, double* partials, double* out, cudaStream_t s) {
    return dot_dev(x, x, n, partials, out, s);
}

cudaError_t dot_dev(const double* a, const double* b, uint64_t n, double* partials, double* out,
                    cudaStream_t s) {
    sumprod_partial_kernel<<<kNormBlocks, kNormThreads, 0, s>>>(a, b, n, partials);
    sum_final_kernel<<<1, 1024, 0, s>>>(partials, kNormBlocks, out);
    return cudaGetLastError();
}

size_t zqr_work_doubles(uint32_t R) { return size_t(3 + 2 * 148 * 2) * R * R; }

cudaError_t launch_zqr(const ZqrArgs& a, cudaStream_t s, int sms) {
    if (a.R <= 8) return zqr_run<8>(a, s, sms);
    if (a.R <= 16) return zqr_run<16>(a, s, sms);
    if (a.R <= 32) return zqr_run<32>(a, s, sms);
    if (a.R <= 64) return zqr_run<64>(a, s, sms);
    return cudaErrorInvalidValue;
}

uint32_t vgemm_max_split() { return 1024; }

cudaError_t launch_vgemm(VgemmArgs& a, cudaStream_t s, int sms) {
    const bool d = a.dual != 0;
    if (a.R <= 8) return d ? vgemm_run<8, true>(a, s, sms) : vgemm_run<8, false>(a, s, sms);
    if (a.R <= 16) return d ? vgemm_run<16, true>(a, s, sms) : vgemm_run<16, false>(a, s, sms);
    if (a.R <= 32) return d ? vgemm_run<32, true>(a, s, sms) : vgemm_run<32, false>(a, s, sms);
    if (a.R <= 64) return d ? vgemm_run<64, true>(a, s, sms) : vgemm_run<64, false>(a, s, sms);
    return cudaErrorInvalidValue;
}

cudaError_t launch_finish(const FinishArgs& a, cudaStream_t s) {
    const size_t base = (3 * size_t(a.R) * a.R + a.I) * sizeof(double);
    const size_t wbytes = a.I * (a.R + 1) * sizeof(double);
    const bool in_smem = base + wbytes <= 200 * 1024;
    static bool cfg = false;
    if (!cfg) {
        cudaFuncSetAttribute(finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cfg = true;
    }
    if (!in_smem && a.scratch == nullptr) return cudaErrorInvalidValue;
    if (base > 200 * 1024) return cudaErrorInvalidValue;
    finish_kernel<<<1, kFThreads, base + (in_smem ? wbytes : 0), s>>>(a, in_smem ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t reduce_splits(const double* part, uint32_t nsplit, uint64_t n, double* out,
                          cudaStream_t s) {
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 1024));
    reduce_splits_kernel<<<std::max(grid, 1u), 256, 0, s>>>(part, nsplit, n, out);
    return cudaGetLastError();
}

cudaError_t normalize_exact(double* a, uint64_t m, uint32_t n, double* weights, cudaStream_t s) {
    normalize_exact_kernel<<<(n + 63) / 64, 64, 0, s>>>(a, m, n, weights);
    return cudaGetLastError();
}

cudaError_t householder_qr(const double* a, uint64_t m, uint32_t n, double* work, double* q,
                           double* r, cudaStream_t s) {
    householder_kernel<<<1, 256, 0, s>>>(a, m, n, work, q, r);
    return cudaGetLastError();
}

cudaError_t permute_rows(const double* in, double* out, const uint64_t* perm, uint64_t rows,
                         uint32_t w, cudaStream_t s) {
    const uint64_t n = rows * w;
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 4096));
    permute_rows_kernel<<<std::max(grid, 1u), 256, 0, s>>>(in, out, perm, rows, w);
    return cudaGetLastError();
}

}  // namespace cpdb
