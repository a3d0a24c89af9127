// CP-ALS through the normal equations (the paper's
// comparison solver, /root/reference/proj/include/cpd/solvers.hpp:149-208).
//
// MTTKRP (tensor.hpp:453-488) M = X_(n) KR(A_k, k != n) runs as
//   T = X x_c A_c^T        one root-sized TTM on the TMA/DMMA kernel of the QR
//                          path (A_c packed like a Q), c = N-1 (c = 0 when n
//                          is the last mode) -- 2|X|R flops, the whole cost;
//   M = KR-contraction of T over the modes other than n and c with the
//                          Khatri-Rao table W of their factors (krc_* below):
//                          one pass over T, HBM-bound, deterministic.
// The host side is als_solver.cpp.  The SPD solve, normalisation, Gram and
// fitness of a mode update run in one 8-CTA cluster kernel (cluster.cu,
// als_finish_cluster_kernel).  This file also holds the single-call
// primitives behind the drop-in headers
// (solve_spd linalg.hpp:132-187, fitness_fast_als kruskal.hpp:88-104).
#include <algorithm>

#include "device.cuh"
#include "kernels.hpp"
#include "rowalg.cuh"

namespace cpdb {
namespace {

constexpr int kKT = 256;  // threads of the KR-contraction kernels
constexpr int kTN = 4;    // M rows per CTA (r-fastest layout)

// W[pq][r] = prod over the modes in `km` (ascending, the last fastest) of
// A_k[i_k][r] -- the Khatri-Rao table of the contracted-away modes in T's
// natural row order (tensor.hpp:343-368 with ascending mode order).
__global__ void kr_table_kernel(KrcArgs a, double* w) {
    const uint64_t n = a.rows_w * a.R;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = e / a.R;
        const uint32_t r = uint32_t(e % a.R);
        uint64_t rem = row;
        double p = 1.0;
        for (int t = int(a.nkm) - 1; t >= 0; --t) {
            const uint32_t k = a.km[t];
            const uint64_t i = rem % a.dims[k];
            rem /= a.dims[k];
            p = (t == int(a.nkm) - 1) ? a.fac[k][i * a.R + r] : a.fac[k][i * a.R + r] * p;
        }
        w[e] = p;
    }
}

// T = [P, In, Q, R] (c = N-1): CTA = kTN rows of M x one split of the (p, q)
// range; thread = (group g, column r), groups interleave over (p, q).
template <int RP>
__global__ void __launch_bounds__(kKT) krc_rfast_kernel(KrcArgs a, const double* __restrict__ w,
                                                        double* __restrict__ out) {
    constexpr int G = kKT / RP;
    __shared__ double red[G][kTN][RP];
    const int rl = threadIdx.x % RP, g = threadIdx.x / RP;
    const int r = int(blockIdx.z) * RP + rl;  // column block (ranks wider than RP)
    const uint32_t R = a.R;
    const uint64_t In = a.In, Q = a.Q, PQ = a.P * a.Q;
    const uint64_t i0 = uint64_t(blockIdx.x) * kTN;
    const uint64_t chunk = (PQ + gridDim.y - 1) / gridDim.y;
    const uint64_t lo = min(PQ, uint64_t(blockIdx.y) * chunk), hi = min(PQ, lo + chunk);
    double acc[kTN];
#pragma unroll
    for (int t = 0; t < kTN; ++t) acc[t] = 0.0;
    if (r < int(R)) {
        uint64_t pq = lo + g;
        uint64_t p = pq / Q, q = pq % Q;
        const uint64_t pstep = G / Q, qstep = G % Q;
        for (; pq < hi; pq += G) {
            const double wt = w[pq * R + r];
            const double* src = a.t + ((p * In + i0) * Q + q) * R + r;
#pragma unroll
            for (int t = 0; t < kTN; ++t)
                if (i0 + t < In) acc[t] = fma(src[uint64_t(t) * Q * R], wt, acc[t]);
            q += qstep;
            p += pstep;
            if (q >= Q) {
                q -= Q;
                ++p;
            }
        }
    }
#pragma unroll
    for (int t = 0; t < kTN; ++t) red[g][t][rl] = acc[t];
    __syncthreads();
    for (int e = threadIdx.x; e < kTN * RP; e += kKT) {
        const int t = e / RP, rr = e % RP, rc = int(blockIdx.z) * RP + rr;
        double s = 0.0;
        for (int gg = 0; gg < G; ++gg) s += red[gg][t][rr];
        if (rc < int(R) && i0 + t < In) out[(uint64_t(blockIdx.y) * In + i0 + t) * R + rc] = s;
    }
}

// T = [R, Q, In] (c = 0, n = N-1): CTA = one r x TI columns of M x one split
// of q; thread = (group g, column i).
template <int TI>
__global__ void __launch_bounds__(kKT) krc_router_kernel(KrcArgs a, const double* __restrict__ w,
                                                         double* __restrict__ out) {
    constexpr int G = kKT / TI;
    __shared__ double red[G][TI];
    const int ti = threadIdx.x % TI, g = threadIdx.x / TI;
    const uint32_t R = a.R;
    const uint64_t In = a.In, Q = a.Q;
    const uint32_t r = blockIdx.x % R;
    const uint64_t i = uint64_t(blockIdx.x / R) * TI + ti;
    const uint64_t chunk = (Q + gridDim.y - 1) / gridDim.y;
    const uint64_t lo = min(Q, uint64_t(blockIdx.y) * chunk), hi = min(Q, lo + chunk);
    double s0 = 0.0, s1 = 0.0;
    if (i < In) {
        const double* src = a.t + uint64_t(r) * Q * In + i;
        uint64_t q = lo + g;
        for (; q + G < hi; q += 2 * G) {
            s0 = fma(src[q * In], w[q * R + r], s0);
            s1 = fma(src[(q + G) * In], w[(q + G) * R + r], s1);
        }
        if (q < hi) s0 = fma(src[q * In], w[q * R + r], s0);
    }
    red[g][ti] = s0 + s1;
    __syncthreads();
    if (g == 0 && i < In) {
        double s = 0.0;
        for (int gg = 0; gg < G; ++gg) s += red[gg][ti];
        out[(uint64_t(blockIdx.y) * In + i) * R + r] = s;
    }
}

int pow2_at_least(uint64_t v, int lo, int hi) {
    int p = lo;
    while (p < hi && uint64_t(p) < v) p *= 2;
    return p;
}

// ---------------------------------------------------------------- solve_spd
// linalg.hpp:132-165: symmetric check, Cholesky, one ridge retry with
// delta = 1e-12 trace / n, else singular.  One CTA; U (= L^T) to u_out.
// status: 0 ok, 4 singular after the ridge, 5 not symmetric; *reg = ridge used.
template <int RM>
__global__ void __launch_bounds__(512) spd_factor_kernel(const double* g, uint32_t n, double* u_out,
                                                         int* status, int* reg) {
    __shared__ double s[RM * RM];
    __shared__ double red[32];
    double mabs = 0.0, masym = 0.0;
    for (uint32_t e = threadIdx.x; e < n * n; e += 512) {
        const uint32_t i = e / n, j = e % n;
        mabs = fmax(mabs, fabs(g[e]));
        masym = fmax(masym, fabs(g[e] - g[j * n + i]));
        s[e] = g[e];
    }
    mabs = block_max<512>(mabs, red);
    masym = block_max<512>(masym, red);
    __syncthreads();
    if (masym > 1e-10 * mabs) {
        if (threadIdx.x == 0) *status = 5;
        return;
    }
    bool ok = chol<512, RM>(s, int(n), int(n));
    int used = 0;
    if (!ok) {
        double tr = 0.0;
        for (uint32_t i = 0; i < n; ++i) tr += g[i * n + i];
        const double delta = 1e-12 * tr / double(n);
        for (uint32_t e = threadIdx.x; e < n * n; e += 512)
            s[e] = g[e] + ((e / n == e % n) ? delta : 0.0);
        __syncthreads();
        ok = chol<512, RM>(s, int(n), int(n));
        used = 1;
    }
    for (uint32_t e = threadIdx.x; e < n * n; e += 512) u_out[e] = s[e];
    if (threadIdx.x == 0) {
        *status = ok ? 0 : 4;
        *reg = used;
    }
}

// x = rhs U^-1 U^-T row by row (linalg.hpp:167-185: w L^T = rhs, x L = w).
template <int RM>
__global__ void __launch_bounds__(512) spd_rows_kernel(const double* u, uint32_t n, double* x,
                                                       uint64_t rows, const int* status) {
    using Row = LaneRow<RM>;
    constexpr int T = Row::T, G = 512 / T;
    extern __shared__ double sm[];  // U, U^T (RM x RM each), 1/diag
    double* su = sm;
    double* sut = su + RM * RM;
    double* dinv = sut + RM * RM;
    if (*status) return;
    stage_tri<RM>(u, int(n), int(n), su, dinv, 512);
    stage_tri_t<RM>(u, int(n), int(n), sut, dinv, 512);
    __syncthreads();
    const int grp = threadIdx.x / T, q = threadIdx.x % T;
    const uint64_t stride = uint64_t(gridDim.x) * G;
    const uint64_t total = ((rows + stride - 1) / stride) * stride;
    for (uint64_t row = uint64_t(blockIdx.x) * G + grp; row < total; row += stride) {
        const bool act = row < rows;
        Row v;
        v.load(x + (act ? row : 0) * n, act ? int(n) : 0, q);
        v.uinv(su, dinv, int(n), q);
        v.utinv(sut, dinv, int(n), q);
        if (act) v.store(x + row * n, int(n), q);
    }
}

// fitness_fast_als (kruskal.hpp:88-104): out = {fitness, raw}.  One CTA.
__global__ void __launch_bounds__(512) fitness_als_kernel(double nx2, const double* m,
                                                          const double* ah, uint64_t n_mr,
                                                          const double* gamma, const double* lam,
                                                          const double* s_last, uint32_t r,
                                                          double* out) {
    __shared__ double red[32];
    double xk = 0.0;
    for (uint64_t e = threadIdx.x; e < n_mr; e += 512) xk = fma(m[e], ah[e], xk);
    xk = block_sum<512>(xk, red);
    double kk = 0.0;
    for (uint32_t e = threadIdx.x; e < r * r; e += 512) {
        const uint32_t i = e / r, j = e % r;
        kk += gamma[e] * lam[i] * s_last[e] * lam[j];
    }
    kk = block_sum<512>(kk, red);
    if (threadIdx.x == 0) {
        const double raw = nx2 - 2.0 * xk + kk;
        const double rad = raw < 0.0 ? 0.0 : raw;
        out[0] = 1.0 - sqrt(rad) / sqrt(nx2);
        out[1] = raw;
    }
}

// G = A^T A (R x R), one thread per entry, rows summed in order.
__global__ void gram_kernel(const double* a, uint64_t m, uint32_t n, double* g) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * n) return;
    const uint32_t p = e / n, q = e % n;
    double s = 0.0;
    for (uint64_t i = 0; i < m; ++i) s = fma(a[i * n + p], a[i * n + q], s);
    g[e] = s;
}

// Gamma = Hadamard of the given R x R matrices, from a ones matrix
__global__ void hadamard_kernel(GramList l, uint32_t r, double* out) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= r * r) return;
    double h = 1.0;
    for (uint32_t t = 0; t < l.n; ++t) h = h * l.g[t][e];
    out[e] = h;
}

__global__ void or_flag_kernel(const int* src, int* dst) {
    if (*src) *dst = 1;
}

}  // namespace

cudaError_t launch_or_flag(const int* src, int* dst, cudaStream_t s) {
    or_flag_kernel<<<1, 1, 0, s>>>(src, dst);
    return cudaGetLastError();
}

cudaError_t gram_dev(const double* a, uint64_t m, uint32_t n, double* g, cudaStream_t s) {
    gram_kernel<<<(n * n + 127) / 128, 128, 0, s>>>(a, m, n, g);
    return cudaGetLastError();
}

cudaError_t hadamard_dev(const GramList& l, uint32_t r, double* out, cudaStream_t s) {
    hadamard_kernel<<<(r * r + 127) / 128, 128, 0, s>>>(l, r, out);
    return cudaGetLastError();
}

uint64_t krc_split(const KrcArgs& a, int sms) {
    if (a.router) {
        const uint64_t ctas = uint64_t(a.R) * ((a.In + 255) / 256);
        return std::max<uint64_t>(1, std::min<uint64_t>((2 * uint64_t(sms) + ctas - 1) / ctas,
                                                        std::max<uint64_t>(1, a.Q / 64)));
    }
    const uint64_t ctas = (a.In + kTN - 1) / kTN;
    return std::max<uint64_t>(1, std::min<uint64_t>((2 * uint64_t(sms) + ctas - 1) / ctas,
                                                    std::max<uint64_t>(1, a.P * a.Q / 64)));
}

cudaError_t launch_kr_table(const KrcArgs& a, double* w, cudaStream_t s) {
    const uint64_t n = a.rows_w * a.R;
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 4096)));
    kr_table_kernel<<<grid, 256, 0, s>>>(a, w);
    return cudaGetLastError();
}

cudaError_t launch_krc(const KrcArgs& a, const double* w, double* out, uint64_t split,
                       cudaStream_t s) {
    if (a.router) {
        const int ti = pow2_at_least(a.In, 32, 256);
        const dim3 grid(unsigned(uint64_t(a.R) * ((a.In + ti - 1) / ti)), unsigned(split));
        switch (ti) {
            case 32: krc_router_kernel<32><<<grid, kKT, 0, s>>>(a, w, out); break;
            case 64: krc_router_kernel<64><<<grid, kKT, 0, s>>>(a, w, out); break;
            case 128: krc_router_kernel<128><<<grid, kKT, 0, s>>>(a, w, out); break;
            default: krc_router_kernel<256><<<grid, kKT, 0, s>>>(a, w, out); break;
        }
        return cudaGetLastError();
    }
    const int rp = pow2_at_least(a.R, 8, 64);
    const dim3 grid(unsigned((a.In + kTN - 1) / kTN), unsigned(split), unsigned((a.R + rp - 1) / rp));
    switch (rp) {
        case 8: krc_rfast_kernel<8><<<grid, kKT, 0, s>>>(a, w, out); break;
        case 16: krc_rfast_kernel<16><<<grid, kKT, 0, s>>>(a, w, out); break;
        case 32: krc_rfast_kernel<32><<<grid, kKT, 0, s>>>(a, w, out); break;
        default: krc_rfast_kernel<64><<<grid, kKT, 0, s>>>(a, w, out); break;
    }
    return cudaGetLastError();
}

size_t spd_work_doubles(uint32_t n) { return (n > 64 ? 2 : 1) * size_t(n) * n; }

cudaError_t launch_spd_solve(const double* g, uint32_t n, double* u_work, double* x, uint64_t rows,
                             int* status, int* reg, cudaStream_t s, int sms) {
    const uint32_t rm = n <= 8 ? 8 : n <= 16 ? 16 : n <= 32 ? 32 : 64;
    if (n > 64) return launch_spd_solve_wide(g, n, u_work, x, rows, status, reg, s);
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(rows / 16 + 1,
                                                                            uint64_t(2 * sms))));
#define CPDB_SPD(RM_)                                                                    \
    {                                                                                  \
        const size_t smem = (2 * RM_ * RM_ + RM_) * sizeof(double);                    \
        cudaError_t e = cudaFuncSetAttribute(spd_rows_kernel<RM_>,                     \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             int(smem));                               \
        if (e != cudaSuccess) return e;                                                \
        spd_factor_kernel<RM_><<<1, 512, 0, s>>>(g, n, u_work, status, reg);           \
        spd_rows_kernel<RM_><<<grid, 512, smem, s>>>(u_work, n, x, rows, status);      \
    }
    switch (rm) {
        case 8: CPDB_SPD(8) break;
        case 16: CPDB_SPD(16) break;
        case 32: CPDB_SPD(32) break;
        default: CPDB_SPD(64) break;
    }
#undef CPDB_SPD
    return cudaGetLastError();
}

cudaError_t launch_fitness_als(double nx2, const double* m, const double* ah, uint64_t n_mr,
                               const double* gamma, const double* lam, const double* s_last,
                               uint32_t r, double* out, cudaStream_t s) {
    fitness_als_kernel<<<1, 512, 0, s>>>(nx2, m, ah, n_mr, gamma, lam, s_last, r, out);
    return cudaGetLastError();
}

}  // namespace cpdb
