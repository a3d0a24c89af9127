// Mode-update kernels as 8-CTA thread-block clusters (sm_100a DSMEM).
//
// The per-mode small-matrix work of CP-ALS-QR is a chain of row-parallel
// triangular solves separated by R x R reductions (two Grams per
// CholeskyQR2).  One CTA is FP64-throughput bound and a grid-wide barrier
// costs microseconds; a cluster gives 8 SMs and barrier.cluster in a few
// hundred cycles, with the Gram partials reduced through distributed shared
// memory (rank 0 reads the other ranks' smem in a fixed order ->
// deterministic).  Row solves are register-resident and lane-parallel, Grams
// run on DMMA (rowalg.cuh).
//
//   finish_cluster_kernel   A_hat = V R0^-T, lambda, A_n, CholQR2(A_n) -> Q_n,
//                           R_n, packed Q_n, fitness   (solvers.hpp:272-292,
//                           linalg.hpp:192-242, factor_state.hpp:42-47,
//                           kruskal.hpp:109-128)
//   zqr_cluster_kernel      Q0, R0 of Khatri-Rao(R_k, k != n) when R^(N-1)
//                           rows fit the cluster's smem  (solvers.hpp:250-255)
#include <cooperative_groups.h>

#include <cmath>

#include "kernels.hpp"
#include "launch.hpp"
#include "rowalg.cuh"

namespace cg = cooperative_groups;

// phase timestamps for profiling (FinishArgs::ts, rank 0 thread 0)
#define CPDB_TS(k) \
    do { if (a.ts && rank == 0 && threadIdx.x == 0) a.ts[k] = globaltimer(); } while (0)

namespace cpdb {
namespace {

constexpr int kCS = 8;    // cluster size (portable maximum)
constexpr int kNT = 512;  // threads per CTA

// Split cluster barrier: every CTA arrives once its remote reads of rank 0's
// shared memory are done; only rank 0 waits, right before it exits (its
// shared memory must outlive those reads), the others exit freely.
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// rank 0: G = sum_r P_r over the cluster, fixed rank order
__device__ void cluster_reduce(cg::cluster_group& cl, const double* P, int n, double* G) {
#pragma unroll 1
    for (int e = threadIdx.x; e < n; e += kNT) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < kCS; ++r) s += cl.map_shared_rank(P, r)[e];
        G[e] = s;
    }
}

// shared-memory plan (doubles)
template <int RM>
struct Smem {
    double *u, *ut, *dinv, *vec, *p, *g, *misc, *w;
    __device__ Smem(double* sm, int R) {
        u = sm;               // RM x RM   triangular factor of the row solves
        ut = u + RM * RM;     // RM x RM   its transpose (LaneRow::utinv)
        dinv = ut + RM * RM;  // RM
        vec = dinv + RM;      // RM        1/lambda (or lambda on rank 0)
        p = vec + RM;         // R x R     Gram partial (read through DSMEM)
        g = p + R * R;        // R x R     rank 0: reduced Gram -> Cholesky
        misc = g + R * R;     // 16
        w = misc + 16;        // per x (R+1), then R x R scratch
    }
    static size_t doubles(int R, uint64_t per) {
        return 2 * size_t(RM) * RM + 2 * RM + 2 * size_t(R) * R + 16 + per * (R + 1) +
               size_t(R) * R;
    }
};

template <int RM, int SL>
__global__ void __launch_bounds__(kNT) finish_cluster_kernel(FinishArgs a) {
    using Row = LaneRow<RM, SL>;
    constexpr int T = Row::T, G = kNT / T;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = int(cl.block_rank());
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ int flag;
    const int R = a.R, ld = R + 1;
    const uint64_t I = a.I;
    const int per = int((I + kCS - 1) / kCS);
    const uint64_t r0 = uint64_t(per) * rank;
    const int rows = int(r0 < I ? (I - r0 < uint64_t(per) ? I - r0 : uint64_t(per)) : 0);
    Smem<RM> S(sm, R);
    double* scratch = S.w + per * ld;
    const int grp = threadIdx.x / T, q = threadIdx.x % T;
    pdl_entry();
    CPDB_TS(0);

    double xk_part = 0.0;
    if (!a.init) {
        stage_tri<RM>(a.r0, R, R, S.u, S.dinv, kNT);
        stage_tri_t<RM>(a.r0, R, R, S.ut, S.dinv, kNT);
        __syncthreads();
        CPDB_TS(16);
        // R0 singular check (linalg.hpp:199-203), warp-parallel on the staged
        // copy; every CTA decides identically
        {
            const int lane = threadIdx.x & 31;
            double mx = 0.0;
            for (int i = lane; i < R; i += 32) mx = fmax(mx, fabs(S.u[i * RM + i]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            int bad = R;
            for (int i = lane; i < R; i += 32)
                if (fabs(S.u[i * RM + i]) <= 1e-14 * mx) bad = min(bad, i);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
            if (bad < R) {
                if (rank == 0 && threadIdx.x == 0) *a.status = 1 | (bad << 8);
                return;  // uniform across the cluster
            }
        }
        CPDB_TS(17);
        // phase A: A_hat = V R0^-T (+ this row's share of <V_fit, A_hat R0^T>)
        for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
            const bool act = li < rows;
            // V row = sum of the V-GEMM's split-K partials (nsplit x I x R)
            const uint64_t roff = (act ? (r0 + li) : r0) * R;
            Row v;
            v.load_sum(a.vpart + roff, I * R, a.nsplit, act ? R : 0, q);
            Row x = v;
            x.utinv(S.ut, S.dinv, R, q);
            if (a.fitness) {  // uniform branch: the lane groups shuffle inside
                // <vf, a_hat R0^T> = sum_k a_hat[k] * (vf R0)[k]
                Row vf = v, w;
                if (a.dual) vf.load_sum(a.vfitpart + roff, I * R, a.nsplit, act ? R : 0, q);
                w.set_times_upper(vf, S.u, R, q);
#pragma unroll
                for (int s = 0; s < Row::S; ++s) xk_part = fma(x.t[s], w.t[s], xk_part);
            }
            if (act) x.store(S.w + li * ld, R, q);
        }
    } else {
#pragma unroll 1
        for (int e = threadIdx.x; e < rows * R; e += kNT)
            S.w[(e / R) * ld + e % R] = a.a_out[(r0 + e / R) * R + e % R];
    }
    __syncthreads();
    CPDB_TS(1);
    gram_dmma<kNT>(S.w, ld, rows, R, S.p, R);
    if (!a.init && a.fitness) {
        const double x = block_sum<kNT>(xk_part, red);
        if (threadIdx.x == 0) S.misc[0] = x;
    }
    CPDB_TS(2);
    cl.sync();  // ---- 1: Gram partials of A_hat ready
    CPDB_TS(3);

    if (rank == 0) {
        cluster_reduce(cl, S.p, R * R, S.g);
        if (!a.init && a.fitness && threadIdx.x == 0) {
            double s = 0.0;
            for (int r = 0; r < kCS; ++r) s += cl.map_shared_rank(S.misc, r)[0];
            S.misc[1] = s;  // <V_fit, A_hat R0^T>
        }
        __syncthreads();
        CPDB_TS(4);
        if (!a.init) {
            // lambda = column norms of A_hat = sqrt(diag G); G1 = D G D
#pragma unroll 1
            for (int c = threadIdx.x; c < R; c += kNT) {
                const double l = sqrt(S.g[c * R + c]);
                scratch[c] = l;                             // lambda (published)
                S.vec[c] = l < 1e-300 ? 0.0 : __drcp_rn(l);  // 1/lambda
            }
            __syncthreads();
#pragma unroll 1
            for (int e = threadIdx.x; e < R * R; e += kNT) {
                const double li = S.vec[e / R], lj = S.vec[e % R];
                S.g[e] = (li == 0.0 || lj == 0.0) ? (e / R == e % R ? 1.0 : 0.0)
                                                   : S.g[e] * li * lj;
            }
            __syncthreads();
        }
        // (rank 0's own Gram partial S.p is free after the reduction)
        const int fp = chol_first_pass<kNT, RM>(S.g, R, I, S.p);
        const bool ok = fp >= 0;
        if (threadIdx.x == 0) S.misc[2] = ok ? 0.0 : 1.0;
        if (fp == 1 && threadIdx.x == 0) atomicOr(a.status, kStatusShifted);
        CPDB_TS(5);
    }
    cl.sync();  // ---- 2: lambda (rank 0's scratch), U1 (rank 0's g) published
    CPDB_TS(6);
    {
        const double* g0 = cl.map_shared_rank(S.g, 0);
        stage_tri<RM>(g0, R, R, S.u, S.dinv, kNT);
        if (!a.init) {
            const double* l0 = cl.map_shared_rank(scratch, 0);
#pragma unroll 1
            for (int c = threadIdx.x; c < RM; c += kNT) {
                const double l = c < R ? l0[c] : 0.0;
                S.vec[c] = l < 1e-300 ? 0.0 : __drcp_rn(l);
                if (rank == 0 && c < R) a.lambda[c] = l < 1e-300 ? 0.0 : l;
            }
        }
        if (threadIdx.x == 0) flag = cl.map_shared_rank(S.misc, 0)[2] != 0.0;
    }
    // (rank 0 next writes its g / scratch after barrier 3, which every rank
    // reaches only after these copies: no cluster barrier needed here)
    __syncthreads();
    CPDB_TS(7);
    if (flag) {
        if (rank == 0 && threadIdx.x == 0) *a.status = 2;
        return;  // uniform: every rank read the same flag
    }
    // phase B: A_n = A_hat / lambda (vanishing column -> e1), A1 = A_n U1^-1
    for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
        const bool act = li < rows;
        Row x;
        x.load(S.w + (act ? li : 0) * ld, act ? R : 0, q);
        if (!a.init) {
#pragma unroll
            for (int s = 0; s < Row::S; ++s) {
                const int k = s * T + q;
                if (k < R) {
                    const double il = S.vec[k];
                    x.t[s] = il == 0.0 ? ((r0 + li) == 0 ? 1.0 : 0.0) : x.t[s] * il;
                }
            }
            if (act) x.store(a.a_out + (r0 + li) * R, R, q);
        }
        x.uinv(S.u, S.dinv, R, q);
        if (act) x.store(S.w + li * ld, R, q);
    }
    __syncthreads();
    CPDB_TS(8);
    gram_dmma<kNT>(S.w, ld, rows, R, S.p, R);
    CPDB_TS(9);
    cl.sync();  // ---- 3: Gram partials of A1 ready
    CPDB_TS(10);

    if (rank == 0) {
        cluster_reduce(cl, S.p, R * R, S.g);
        __syncthreads();
        CPDB_TS(19);
        // A1 is orthonormal to working accuracy: its Gram is I + O(kappa^2 eps)
        // (rank 0's own partial S.p and the lambda scratch are free again)
        const int steps = near_identity_chol<kNT>(S.g, R, S.p, scratch, red);
        if (a.ts && threadIdx.x == 0) a.ts[20] = a.ts[0] + 1000ull * steps;
        const bool ok = steps > 0 || chol<kNT, RM>(S.g, R, R);
        if (threadIdx.x == 0) S.misc[2] = ok ? 0.0 : 1.0;
        CPDB_TS(11);
        if (ok) {
            // R_n = U2 U1 (U1 in S.u, stride RM)
#pragma unroll 1
            for (int e = threadIdx.x; e < R * R; e += kNT) {
                const int i = e / R, j = e % R;
                double s = 0.0;
                for (int p = i; p <= j; ++p) s = fma(S.g[i * R + p], S.u[p * RM + j], s);
                scratch[e] = i <= j ? s : 0.0;
                a.r_out[e] = scratch[e];
            }
            __syncthreads();
            if (!a.init && a.fitness) {
                // R0 into rank 0's free Gram partial (conflict-free reads below)
#pragma unroll 1
                for (int e = threadIdx.x; e < R * R; e += kNT) S.p[e] = a.r0[e];
                __syncthreads();
                // ||K||^2 = sum_ij (R0^T R0)_ij l_i (Rn^T Rn)_ij l_j  (kruskal.hpp:457-462)
                double s = 0.0;
#pragma unroll 1
                for (int e = threadIdx.x; e < R * R; e += kNT) {
                    const int i = e / R, j = e % R;
                    const double li = a.lambda[i], lj = a.lambda[j];
                    double p0 = 0.0, pn = 0.0, p1 = 0.0, pm = 0.0;
                    const int top = i < j ? i : j;
                    int p = 0;
                    for (; p + 1 <= top; p += 2) {
                        p0 = fma(S.p[p * R + i], S.p[p * R + j], p0);
                        pn = fma(scratch[p * R + i], scratch[p * R + j], pn);
                        p1 = fma(S.p[(p + 1) * R + i], S.p[(p + 1) * R + j], p1);
                        pm = fma(scratch[(p + 1) * R + i], scratch[(p + 1) * R + j], pm);
                    }
                    if (p <= top) {
                        p0 = fma(S.p[p * R + i], S.p[p * R + j], p0);
                        pn = fma(scratch[p * R + i], scratch[p * R + j], pn);
                    }
                    s += (p0 + p1) * li * (pn + pm) * lj;
                }
                const double kk = block_sum<kNT>(s, red);
                if (threadIdx.x == 0) {
                    const double raw = a.norm_x_sq - 2.0 * S.misc[1] + kk;
                    const double rad = raw < 0.0 ? 0.0 : raw;
                    a.fit_out[0] = 1.0 - sqrt(rad) / sqrt(a.norm_x_sq);
                    a.fit_out[1] = raw;
                }
            }
            // zero padding rows of the packed Q (k >= I)
            const uint32_t Rp = ttm_rpad_dev(R);
            const uint64_t Kpad = ((I + 31) / 32) * 32;
#pragma unroll 1
            for (uint64_t e = I * Rp + threadIdx.x; e < Kpad * Rp; e += kNT) {
                const uint64_t k = e / Rp, r = e % Rp;
                a.qp_out[((k >> 2) * Rp + r) * 4 + (k & 3)] = 0.0;
            }
        }
        CPDB_TS(12);
    }
    cl.sync();  // ---- 4: U2 (rank 0's g) published
    CPDB_TS(13);
    {
        const double* g0 = cl.map_shared_rank(S.g, 0);
        stage_tri<RM>(g0, R, R, S.u, S.dinv, kNT);
        if (threadIdx.x == 0) flag = cl.map_shared_rank(S.misc, 0)[2] != 0.0;
    }
    __syncthreads();
    cluster_arrive();  // this CTA's reads of rank 0's smem are done
    if (!flag) {
        // phase C: Q = A1 U2^-1 (+ packed copy [Kpad/4][Rp][4])
        const uint32_t Rp = ttm_rpad_dev(R);
        for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
            const bool act = li < rows;
            Row x;
            x.load(S.w + (act ? li : 0) * ld, act ? R : 0, q);
            x.uinv(S.u, S.dinv, R, q);
            if (act) {
                const uint64_t i = r0 + li;
                x.store(a.q_out + i * R, R, q);
                double* qp = a.qp_out + ((i >> 2) * Rp) * 4 + (i & 3);
#pragma unroll
                for (int s = 0; s < Row::S; ++s) {
                    const int k = s * T + q;
                    if (k < int(Rp)) qp[k * 4] = k < R ? x.t[s] : 0.0;
                }
            }
        }
    } else if (rank == 0 && threadIdx.x == 0) {
        *a.status = 2;
    }
    CPDB_TS(14);
    if (rank == 0) cluster_wait();  // rank 0's smem outlives the others' DSMEM reads
    CPDB_TS(15);
}

// ---------------------------------------------------------------- Z-QR (small Z)
template <int RM, int SL>
__global__ void __launch_bounds__(kNT) zqr_cluster_kernel(ZqrArgs a) {
    using Row = LaneRow<RM, SL>;
    constexpr int T = Row::T, G = kNT / T;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = int(cl.block_rank());
    extern __shared__ double sm[];
    const int R = a.R, nm = a.nm, ld = R + 1;
    const int per = int((a.zrows + kCS - 1) / kCS);
    const uint64_t r0 = uint64_t(per) * rank;
    const int rows = int(r0 < a.zrows ? (a.zrows - r0 < uint64_t(per) ? a.zrows - r0
                                                                      : uint64_t(per))
                                      : 0);
    __shared__ double red[32];
    Smem<RM> S(sm, R);
    pdl_entry();
    CPDB_TS(0);
    double* mats = S.w + per * ld;  // nm x R x R (after the R x R scratch)
    mats += R * R;
    const int grp = threadIdx.x / T, q = threadIdx.x % T;

    for (int t = 0; t < nm; ++t)
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) mats[t * R * R + e] = a.rmats[t][e];
    __syncthreads();
    // G1 = Hadamard_t (R_t^T R_t), computed redundantly by every rank (tiny);
    // four independent accumulators break the FMA dependency chain
#pragma unroll 1
    for (int e = threadIdx.x; e < R * R; e += kNT) {
        const int i = e / R, j = e % R;
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        double h = 1.0;
        for (int t = nm - 1; t >= 0; --t) {
            const double* m = mats + t * R * R;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int k = 0;
            for (; k + 3 <= lo; k += 4) {
                s0 = fma(m[k * R + lo], m[k * R + hi], s0);
                s1 = fma(m[(k + 1) * R + lo], m[(k + 1) * R + hi], s1);
                s2 = fma(m[(k + 2) * R + lo], m[(k + 2) * R + hi], s2);
                s3 = fma(m[(k + 3) * R + lo], m[(k + 3) * R + hi], s3);
            }
            for (; k <= lo; ++k) s0 = fma(m[k * R + lo], m[k * R + hi], s0);
            const double sum = (s0 + s1) + (s2 + s3);
            h = (t == nm - 1) ? sum : h * sum;
        }
        S.g[e] = h;
    }
    __syncthreads();
    CPDB_TS(1);
    // (S.p, this rank's G2 partial later, is free here)
    const int fp1 = chol_first_pass<kNT, RM>(S.g, R, a.zrows, S.p);
    const bool ok1 = fp1 >= 0;
    if (!ok1 && rank == 0 && threadIdx.x == 0) *a.status = 2;
    if (fp1 == 1 && rank == 0 && threadIdx.x == 0) atomicOr(a.status, kStatusShifted);
    stage_tri<RM>(S.g, R, R, S.u, S.dinv, kNT);  // U1 (kept in S.g too)
    __syncthreads();
    CPDB_TS(2);
    // Q1 = Z U1^-1 on this rank's rows; Z rows are generated in registers
    // (product in descending mode order like the reference Khatri-Rao fold)
    for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
        const bool act = li < rows;
        Row x;
        // Z row = product over the other modes (descending, like the
        // reference Khatri-Rao fold) of one row of each R_k; the row index's
        // digits are peeled in the same order (32-bit: the cluster path has
        // R^(N-1) rows in shared memory).  Rolled over the modes: compact code.
        {
            uint32_t rem = uint32_t(r0) + uint32_t(act ? li : 0);
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
        x.uinv(S.u, S.dinv, R, q);
        if (act) x.store(S.w + li * ld, R, q);
    }
    __syncthreads();
    CPDB_TS(3);
    gram_dmma<kNT>(S.w, ld, rows, R, S.p, R);
    CPDB_TS(4);
    cl.sync();
    CPDB_TS(5);
    if (rank == 0) {
        double* u1 = S.w + per * ld;  // keep U1 (stride R) for R0 = U2 U1
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) u1[e] = S.g[e];
        __syncthreads();
        cluster_reduce(cl, S.p, R * R, S.g);
        __syncthreads();
        CPDB_TS(11);
        // Q1 = Z U1^-1 is orthonormal to working accuracy (S.p and the
        // Khatri-Rao inputs are free again)
        const int steps = near_identity_chol<kNT>(S.g, R, S.p, mats, red);
        if (a.ts && threadIdx.x == 0) a.ts[12] = a.ts[0] + 1000ull * steps;
        const bool ok2 = steps > 0 || chol<kNT, RM>(S.g, R, R);
        if (!ok2 && threadIdx.x == 0) *a.status = 2;
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) {  // R0 = U2 U1
            const int i = e / R, j = e % R;
            double s0 = 0.0, s1 = 0.0;
            int k = i;
            for (; k + 1 <= j; k += 2) {
                s0 = fma(S.g[i * R + k], u1[k * R + j], s0);
                s1 = fma(S.g[i * R + k + 1], u1[(k + 1) * R + j], s1);
            }
            if (k <= j) s0 = fma(S.g[i * R + k], u1[k * R + j], s0);
            a.r0[e] = i <= j ? s0 + s1 : 0.0;
        }
        CPDB_TS(6);
    }
    cl.sync();
    CPDB_TS(7);
    stage_tri<RM>(cl.map_shared_rank(S.g, 0), R, R, S.u, S.dinv, kNT);
    __syncthreads();
    cluster_arrive();  // this CTA's reads of rank 0's smem are done
    CPDB_TS(8);
    for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
        const bool act = li < rows;
        Row x;
        x.load(S.w + (act ? li : 0) * ld, act ? R : 0, q);
        x.uinv(S.u, S.dinv, R, q);
        if (act) x.store(a.q0 + (r0 + li) * R, R, q);
    }
    CPDB_TS(9);
    if (rank == 0) cluster_wait();  // rank 0's smem outlives the others' reads
    CPDB_TS(10);
}

// ---------------------------------------------------------------- CP-ALS mode tail
// solvers.hpp:177-197 for mode n: Gamma = Hadamard_k G_k (k != n, ascending,
// from a ones matrix), A_hat = solve_spd(Gamma, M) (linalg.hpp:132-187),
// (A_n, lambda) = normalize_columns(A_hat) (linalg.hpp:225-242), G_n =
// gram(A_n), and on the last mode fitness_fast_als (kruskal.hpp:88-104).
// Rank 0 factors Gamma (U^T U = Gamma, i.e. U = L^T); every rank solves its
// rows, x = m U^-1 U^-T, and the two Grams are reduced over DSMEM.
template <int RM, int SL>
__global__ void __launch_bounds__(kNT) als_finish_cluster_kernel(AlsFinishArgs a) {
    using Row = LaneRow<RM, SL>;
    constexpr int T = Row::T, G = kNT / T;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = int(cl.block_rank());
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ int flag;
    const int R = a.R, ld = R + 1;
    const uint64_t I = a.I;
    const int per = int((I + kCS - 1) / kCS);
    const uint64_t r0 = uint64_t(per) * rank;
    const int rows = int(r0 < I ? (I - r0 < uint64_t(per) ? I - r0 : uint64_t(per)) : 0);
    Smem<RM> S(sm, R);
    double* gam = S.w + per * ld;  // R x R: Gamma (rank 0)
    const int grp = threadIdx.x / T, q = threadIdx.x % T;
    pdl_entry();
    CPDB_TS(0);

    if (rank == 0) {
        double mabs = 0.0, masym = 0.0;
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) {
            double h = 1.0;
            for (uint32_t t = 0; t < a.ng; ++t) h = h * a.grams[t][e];
            gam[e] = h;
            S.g[e] = h;
        }
        __syncthreads();
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) {
            const int i = e / R, j = e % R;
            mabs = fmax(mabs, fabs(gam[e]));
            masym = fmax(masym, fabs(gam[e] - gam[j * R + i]));
        }
        mabs = block_max<kNT>(mabs, red);
        masym = block_max<kNT>(masym, red);
        int code = 0, used = 0;
        if (masym > 1e-10 * mabs) {
            code = 5;
        } else {
            bool ok = chol<kNT, RM>(S.g, R, R);
            if (!ok) {  // ridge retry, delta = 1e-12 trace / n (linalg.hpp:147-154)
                double tr = 0.0;
                for (int i = 0; i < R; ++i) tr += gam[i * R + i];
                const double delta = 1e-12 * tr / double(R);
#pragma unroll 1
                for (int e = threadIdx.x; e < R * R; e += kNT)
                    S.g[e] = gam[e] + ((e / R == e % R) ? delta : 0.0);
                __syncthreads();
                ok = chol<kNT, RM>(S.g, R, R);
                used = 1;
            }
            code = ok ? 0 : 4;
        }
        if (threadIdx.x == 0) {
            S.misc[2] = double(code);
            if (used) *a.regularized = 1;
        }
        CPDB_TS(1);
    }
    cl.sync();  // ---- 1: U (rank 0's g) published
    {
        const double* g0 = cl.map_shared_rank(S.g, 0);
        stage_tri<RM>(g0, R, R, S.u, S.dinv, kNT);
        stage_tri_t<RM>(g0, R, R, S.ut, S.dinv, kNT);
        if (threadIdx.x == 0) flag = int(cl.map_shared_rank(S.misc, 0)[2]);
    }
    cl.sync();  // rank 0 may reuse g only after every rank copied U
    if (flag) {
        if (rank == 0 && threadIdx.x == 0) *a.status = flag;
        return;  // uniform across the cluster
    }
    // rows: A_hat = M U^-1 U^-T (+ this rank's share of <M, A_hat>)
    double xk_part = 0.0;
    for (int li = grp; li < rows + (G - rows % G) % G; li += G) {
        const bool act = li < rows;
        Row x;
        x.load(a.m + (act ? (r0 + li) : r0) * R, act ? R : 0, q);
        Row m = x;
        x.uinv(S.u, S.dinv, R, q);
        x.utinv(S.ut, S.dinv, R, q);
        if (a.fitness) {
#pragma unroll
            for (int s = 0; s < Row::S; ++s) xk_part = fma(m.t[s], x.t[s], xk_part);
        }
        if (act) x.store(S.w + li * ld, R, q);
    }
    __syncthreads();
    CPDB_TS(2);
    gram_dmma<kNT>(S.w, ld, rows, R, S.p, R);
    if (a.fitness) {
        const double x = block_sum<kNT>(xk_part, red);
        if (threadIdx.x == 0) S.misc[0] = x;
    }
    cl.sync();  // ---- 2: Gram partials of A_hat
    if (rank == 0) {
        cluster_reduce(cl, S.p, R * R, S.g);
        if (a.fitness && threadIdx.x == 0) {
            double x = 0.0;
            for (int r = 0; r < kCS; ++r) x += cl.map_shared_rank(S.misc, r)[0];
            S.misc[1] = x;  // <M, A_hat>
        }
        __syncthreads();
#pragma unroll 1
        for (int c = threadIdx.x; c < R; c += kNT) S.vec[c] = sqrt(S.g[c * R + c]);  // lambda
    }
    cl.sync();  // ---- 3: lambda published (rank 0's vec)
    {
        const double* l0 = cl.map_shared_rank(S.vec, 0);
#pragma unroll 1
        for (int c = threadIdx.x; c < RM; c += kNT) {
            const double l = c < R ? l0[c] : 0.0;
            S.dinv[c] = l < 1e-300 ? 0.0 : __drcp_rn(l);  // 1/lambda (U is no longer needed)
            if (rank == 0 && c < R) a.lambda[c] = l < 1e-300 ? 0.0 : l;
        }
    }
    __syncthreads();
    // A_n = A_hat / lambda (vanishing column -> e1, weight 0)
#pragma unroll 1
    for (int e = threadIdx.x; e < rows * R; e += kNT) {
        const int li = e / R, c = e % R;
        const double il = S.dinv[c];
        const double v = il == 0.0 ? ((r0 + li) == 0 ? 1.0 : 0.0) : S.w[li * ld + c] * il;
        S.w[li * ld + c] = v;
        a.a_out[(r0 + li) * R + c] = v;
    }
    __syncthreads();
    gram_dmma<kNT>(S.w, ld, rows, R, S.p, R);
    cl.sync();  // ---- 4: Gram partials of A_n
    if (rank == 0) {
        cluster_reduce(cl, S.p, R * R, S.g);
        __syncthreads();
#pragma unroll 1
        for (int e = threadIdx.x; e < R * R; e += kNT) a.g_out[e] = S.g[e];
        if (a.fitness) {
            // ||K||^2 = sum_ij Gamma_ij l_i G_ij l_j  (kruskal.hpp:97-100)
            double kk = 0.0;
#pragma unroll 1
            for (int e = threadIdx.x; e < R * R; e += kNT) {
                const int i = e / R, j = e % R;
                const double li = S.vec[i] < 1e-300 ? 0.0 : S.vec[i];
                const double lj = S.vec[j] < 1e-300 ? 0.0 : S.vec[j];
                kk += gam[e] * li * S.g[e] * lj;
            }
            kk = block_sum<kNT>(kk, red);
            if (threadIdx.x == 0) {
                const double raw = a.norm_x_sq - 2.0 * S.misc[1] + kk;
                const double rad = raw < 0.0 ? 0.0 : raw;
                a.fit_out[0] = 1.0 - sqrt(rad) / sqrt(a.norm_x_sq);
                a.fit_out[1] = raw;
            }
        }
        CPDB_TS(3);
    }
    cl.sync();  // the other ranks' smem must outlive rank 0's DSMEM reads
}

template <class Arg>
cudaError_t launch_cluster(void (*kern)(Arg), size_t smem, cudaStream_t s, const Arg& arg,
                           bool pdl) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t c{};
    c.gridDim = dim3(kCS, 1, 1);
    c.blockDim = dim3(kNT, 1, 1);
    c.dynamicSmemBytes = smem;
    c.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = attr;
    c.numAttrs = (pdl && pdl_enabled()) ? 2 : 1;
    return cudaLaunchKernelEx(&c, kern, arg);
}

int rm_of(uint32_t R) { return R <= 8 ? 8 : R <= 16 ? 16 : R <= 32 ? 32 : 64; }

template <int RM>
size_t finish_smem_rm(uint64_t I, uint32_t R) {
    return Smem<RM>::doubles(R, (I + kCS - 1) / kCS) * sizeof(double);
}

template <int RM>
size_t zqr_smem_rm(uint64_t zrows, uint32_t R, uint32_t nm) {
    return (Smem<RM>::doubles(R, (zrows + kCS - 1) / kCS) + size_t(nm) * R * R) * sizeof(double);
}

}  // namespace

size_t finish_cluster_smem(uint64_t I, uint32_t R) {
    switch (rm_of(R)) {
        case 8: return finish_smem_rm<8>(I, R);
        case 16: return finish_smem_rm<16>(I, R);
        case 32: return finish_smem_rm<32>(I, R);
        default: return finish_smem_rm<64>(I, R);
    }
}

namespace {

// Slots per lane of the row solves: as few as possible (more lanes per row,
// shorter solve steps) while every row of a CTA still gets a lane group.
int slots_for(int rm, uint64_t rows_per_cta) {
    int sl = 1;
    while (sl < 8 && (uint64_t(kNT) / uint64_t(rm / sl)) < rows_per_cta) sl *= 2;
    while (rm / sl > 32) sl *= 2;  // at most one warp per row
    return sl;
}

template <int RM, int SL>
cudaError_t finish_rs(const FinishArgs& a, size_t smem, cudaStream_t s) {
    return launch_cluster<FinishArgs>(finish_cluster_kernel<RM, SL>, smem, s, a, true);
}
template <int RM, int SL>
cudaError_t zqr_rs(const ZqrArgs& a, size_t smem, cudaStream_t s) {
    return launch_cluster<ZqrArgs>(zqr_cluster_kernel<RM, SL>, smem, s, a, a.pdl != 0);
}

template <int RM, class F8, class F4, class F2, class F1>
cudaError_t by_slots(int sl, F8 f8, F4 f4, F2 f2, F1 f1) {
    switch (sl) {
        case 1: if constexpr (RM <= 32) return f1(); else return f2();
        case 2: return f2();
        case 4: return f4();
        default: return f8();
    }
}

}  // namespace

cudaError_t launch_finish_cluster(const FinishArgs& a, cudaStream_t s) {
    if (a.R > 64) return cudaErrorInvalidValue;
    const size_t smem = finish_cluster_smem(a.I, a.R);
    if (smem > 220 * 1024) return cudaErrorInvalidValue;
    const uint64_t rows = (a.I + kCS - 1) / kCS;
    const int rm = rm_of(a.R), sl = slots_for(rm, rows);
#define CPDB_FIN(RM_)                                                                    \
    return by_slots<RM_>(                                                                \
        sl, [&] { return finish_rs<RM_, 8>(a, smem, s); },                               \
        [&] { return finish_rs<RM_, 4>(a, smem, s); },                                   \
        [&] { return finish_rs<RM_, 2>(a, smem, s); },                                   \
        [&] { return finish_rs<RM_, (RM_ <= 32 ? 1 : 2)>(a, smem, s); })
    switch (rm) {
        case 8: CPDB_FIN(8);
        case 16: CPDB_FIN(16);
        case 32: CPDB_FIN(32);
        default: CPDB_FIN(64);
    }
#undef CPDB_FIN
}

static size_t als_smem(uint64_t I, uint32_t R) {
    // Smem plan + Gamma (R x R) after the rows
    const uint64_t per = (I + kCS - 1) / kCS;
    switch (rm_of(R)) {
        case 8: return (Smem<8>::doubles(R, per) + size_t(R) * R) * sizeof(double);
        case 16: return (Smem<16>::doubles(R, per) + size_t(R) * R) * sizeof(double);
        case 32: return (Smem<32>::doubles(R, per) + size_t(R) * R) * sizeof(double);
        default: return (Smem<64>::doubles(R, per) + size_t(R) * R) * sizeof(double);
    }
}

bool als_finish_fits(uint64_t I, uint32_t R) { return R <= 64 && als_smem(I, R) <= 220 * 1024; }

namespace {
template <int RM, int SL>
cudaError_t als_rs(const AlsFinishArgs& a, size_t smem, cudaStream_t s) {
    return launch_cluster<AlsFinishArgs>(als_finish_cluster_kernel<RM, SL>, smem, s, a, true);
}
}  // namespace

cudaError_t launch_als_finish(const AlsFinishArgs& a, cudaStream_t s) {
    if (!als_finish_fits(a.I, a.R)) return cudaErrorInvalidValue;
    const size_t smem = als_smem(a.I, a.R);
    const uint64_t rows = (a.I + kCS - 1) / kCS;
    const int rm = rm_of(a.R), sl = slots_for(rm, rows);
#define CPDB_ALS(RM_)                                                                    \
    return by_slots<RM_>(                                                                \
        sl, [&] { return als_rs<RM_, 8>(a, smem, s); },                                  \
        [&] { return als_rs<RM_, 4>(a, smem, s); },                                      \
        [&] { return als_rs<RM_, 2>(a, smem, s); },                                      \
        [&] { return als_rs<RM_, (RM_ <= 32 ? 1 : 2)>(a, smem, s); })
    switch (rm) {
        case 8: CPDB_ALS(8);
        case 16: CPDB_ALS(16);
        case 32: CPDB_ALS(32);
        default: CPDB_ALS(64);
    }
#undef CPDB_ALS
}

static size_t zqr_cluster_smem(uint64_t zrows, uint32_t R, uint32_t nm) {
    switch (rm_of(R)) {
        case 8: return zqr_smem_rm<8>(zrows, R, nm);
        case 16: return zqr_smem_rm<16>(zrows, R, nm);
        case 32: return zqr_smem_rm<32>(zrows, R, nm);
        default: return zqr_smem_rm<64>(zrows, R, nm);
    }
}

bool zqr_cluster_fits(uint64_t zrows, uint32_t R, uint32_t nm) {
    return R <= 64 && zqr_cluster_smem(zrows, R, nm) <= 200 * 1024;
}

cudaError_t launch_zqr_cluster(const ZqrArgs& a, cudaStream_t s) {
    const size_t smem = zqr_cluster_smem(a.zrows, a.R, a.nm);
    const uint64_t rows = (a.zrows + kCS - 1) / kCS;
    const int rm = rm_of(a.R), sl = slots_for(rm, rows);
#define CPDB_ZQR(RM_)                                                                    \
    return by_slots<RM_>(                                                                \
        sl, [&] { return zqr_rs<RM_, 8>(a, smem, s); },                                  \
        [&] { return zqr_rs<RM_, 4>(a, smem, s); },                                      \
        [&] { return zqr_rs<RM_, 2>(a, smem, s); },                                      \
        [&] { return zqr_rs<RM_, (RM_ <= 32 ? 1 : 2)>(a, smem, s); })
    switch (rm) {
        case 8: CPDB_ZQR(8);
        case 16: CPDB_ZQR(16);
        case 32: CPDB_ZQR(32);
        default: CPDB_ZQR(64);
    }
#undef CPDB_ZQR
}

}  // namespace cpdb
