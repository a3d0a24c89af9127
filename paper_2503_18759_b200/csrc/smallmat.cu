// K4/K6: V-GEMM and the reductions of a CP-ALS-QR mode update.
//
//   launch_vgemm   V = unfold(Y,n) * Q0_hat, extrapolation fused into the
//                  operand load (solvers.hpp:260-271, 277-284)
//   reduce_splits  deterministic split-K reduction (many CTAs)
//   norm_sq        inner(x, x) (tensor.hpp:394-399)
// (Z-QR lives in zqr.cu, the per-mode tail in finish.cu.)
// All reductions use fixed partitions and fixed trees: repeated runs are
// bit-identical (solver_test.cpp:272-282 requires it).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "device.cuh"
#include "kernels.hpp"
#include "launch.hpp"
#include "rowalg.cuh"

namespace cpdb {
namespace {

namespace cg = cooperative_groups;

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

// ------------------------------------------------------------------ V-GEMM
constexpr int kVThreads = 256;
constexpr int kVBI = 64;  // rows of V per block
constexpr int kVBK = 16;  // k per smem tile

// extrapolation decision of a V-GEMM launch: the host's, or the device
// gate's when the launch carries one (uniform over the grid)
__device__ __forceinline__ bool extrap_on(const VgemmArgs& a) {
    if (!a.extrap) return false;
    return a.gate ? (a.gate[0] != 0.0 && a.gate[1] != 0.0) : true;
}
__device__ __forceinline__ double extrap_beta(const VgemmArgs& a) {
    return a.gate ? a.gate[1] : a.beta;
}

template <int RM, bool DUAL>
__global__ void __launch_bounds__(kVThreads)
vgemm_kernel(VgemmArgs a, uint64_t kchunk) {
    pdl_entry();
    __shared__ double yt[kVBI][kVBK + 1];
    __shared__ double pt[kVBK][RM];
    __shared__ double ft[DUAL ? kVBK : 1][RM];
    const int R = a.R;
    const int rbase = int(blockIdx.z) * RM;  // column block (ranks wider than RM)
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
    const bool ex = extrap_on(a);
    const double beta = extrap_beta(a);
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
                // K = R^(N-1) < 2^32: 32-bit index math (a 64-bit division per
                // element dominated this loop)
                const uint32_t k32 = uint32_t(k), J32 = uint32_t(J);
                const uint32_t o = k32 / J32, j = k32 - o * J32;
                v = a.y[(uint64_t(o) * I + i) * J + j];
            }
            yt[r_][c_] = v;
        }
        for (int e = threadIdx.x; e < kVBK * RM; e += kVThreads) {
            const int kk = e / RM, r = rbase + e % RM;
            const uint64_t k = k0 + kk;
            double q = 0.0, p = 0.0;
            if (k < ke && r < R) {
                q = a.q0[k * R + r];
                p = q;
                if (ex) p = q + beta * (q - a.alpha * a.hist[k * R + r]);
            }
            pt[kk][r - rbase] = p;
            if (DUAL) ft[kk][r - rbase] = q;
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
            const int r = rbase + rg + 4 * u;
            if (r < R) {
                vp[r] = acc[u];
                if (DUAL) fp[r] = accf[u];
            }
        }
    }
}

// V-GEMM on the FP64 tensor cores.  CTA = 64 rows of V x all R columns over a
// K-chunk; warp w owns rows 8w..8w+7 and the Rp/8 column blocks (DMMA
// m8n8k4).  Y and P tiles (16 k) are staged in padded shared memory
// (conflict-free fragment reads) with the next tile prefetched into
// registers; the extrapolation P = Q0 + beta (Q0 - alpha H) is fused into the
// P tile load, and the DUAL variant also accumulates Y Q0 for the fitness.
// Two ways to combine the K-chunks, both in a fixed order (deterministic):
//  * vgemm_cluster_kernel (very short K, C1): the 8 K-chunks of a
//    row block are one thread-block cluster and are summed through
//    distributed shared memory straight into V -- one launch, no partials;
//  * vgemm_dmma_kernel (longer K, C2-C5): split-K partials in HBM, summed by
//    reduce_splits.
constexpr int kDM = 64, kDK = 16, kDThreads = 256, kVCluster = 8;
// K-tiles per CTA up to which the cluster form is used: measured, it wins at
// C1 (K = 100: 1 tile per CTA, 6020 -> 6310 sweeps/s) and loses at C4 / C2
// (4 / 8 tiles per CTA run in sequence: -4% / -2% against 1-tile split-K
// CTAs plus the reduction kernel)
constexpr int kVClusterTiles = 2;

template <int RM, bool DUAL>
struct VAcc {
    static constexpr int RB = RM / 8 > 0 ? RM / 8 : 1;
    double v[RB][2], f[DUAL ? RB : 1][2];
};

template <int RM, bool DUAL>
__device__ __forceinline__ void vgemm_tile(const VgemmArgs& a, uint64_t i0, uint32_t kb,
                                           uint32_t ke, VAcc<RM, DUAL>& acc) {
    constexpr int RB = VAcc<RM, DUAL>::RB;
    constexpr int YLD = kDK + 4;   // (m*YLD) mod 16 spaced by 4: conflict-free A reads
    constexpr int PLD = RM + 4;    // likewise for the B reads
    constexpr int YPT = kDM * kDK / kDThreads;  // 4 Y elements per thread
    constexpr int PPT = (kDK * RM + kDThreads - 1) / kDThreads;
    __shared__ double ys[kDM * YLD];
    __shared__ double ps[kDK * PLD];
    __shared__ double fs[DUAL ? kDK * PLD : 1];
    const int R = a.R;
    const uint64_t I = a.I;
    const uint32_t J = uint32_t(a.J);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool jrun = (J % kDK) == 0;  // a 16-k tile is 16 consecutive j of one o
    const bool ex = extrap_on(a);
    const double beta = extrap_beta(a);

    // two register sets: tiles t+1 and t+2 are in flight during tile t's MMAs
    // (q0 and the history travel raw; the extrapolation is applied at the
    // stash, so the loads stay in flight during the MMAs in between)
    struct Regs {
        double y[YPT], h[PPT], q[PPT];
    };
    auto fetch = [&](Regs& rg, uint32_t k0) {
#pragma unroll
        for (int u = 0; u < YPT; ++u) {
            const int e = threadIdx.x + u * kDThreads;
            const int m = jrun ? e / kDK : e % kDM, c = jrun ? e % kDK : e / kDM;
            const uint32_t k = k0 + c;
            const uint64_t i = i0 + m;
            double v = 0.0;
            if (k < ke && i < I) {
                const uint32_t o = k / J, j = k - o * J;
                v = a.y[(uint64_t(o) * I + i) * J + j];
            }
            rg.y[u] = v;
        }
#pragma unroll
        for (int u = 0; u < PPT; ++u) {
            const int e = threadIdx.x + u * kDThreads;
            const int kk = e / RM, r = e % RM;
            const uint32_t k = k0 + kk;
            double q = 0.0, h = 0.0;
            if (e < kDK * RM && k < ke && r < R) {
                q = a.q0[uint64_t(k) * R + r];
                if (ex) h = a.hist[uint64_t(k) * R + r];
            }
            rg.q[u] = q;
            rg.h[u] = h;
        }
    };
    auto stash = [&](const Regs& rg) {
#pragma unroll
        for (int u = 0; u < YPT; ++u) {
            const int e = threadIdx.x + u * kDThreads;
            const int m = jrun ? e / kDK : e % kDM, c = jrun ? e % kDK : e / kDM;
            ys[m * YLD + c] = rg.y[u];
        }
#pragma unroll
        for (int u = 0; u < PPT; ++u) {
            const int e = threadIdx.x + u * kDThreads;
            if (e < kDK * RM) {
                const double q = rg.q[u];
                ps[(e / RM) * PLD + e % RM] = ex ? q + beta * (q - a.alpha * rg.h[u]) : q;
                if (DUAL) fs[(e / RM) * PLD + e % RM] = q;
            }
        }
    };
    auto mma = [&]() {
#pragma unroll
        for (int s4 = 0; s4 < kDK / 4; ++s4) {
            const double av = ys[(warp * 8 + (lane >> 2)) * YLD + 4 * s4 + (lane & 3)];
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                const double bv = ps[(4 * s4 + (lane & 3)) * PLD + b * 8 + (lane >> 2)];
                dmma(acc.v[b][0], acc.v[b][1], av, bv);
                if (DUAL) {
                    const double fv = fs[(4 * s4 + (lane & 3)) * PLD + b * 8 + (lane >> 2)];
                    dmma(acc.f[b][0], acc.f[b][1], av, fv);
                }
            }
        }
    };

#pragma unroll
    for (int b = 0; b < RB; ++b) acc.v[b][0] = acc.v[b][1] = 0.0;
#pragma unroll
    for (int b = 0; b < (DUAL ? RB : 1); ++b) acc.f[b][0] = acc.f[b][1] = 0.0;

    Regs ra, rb;
    if (kb < ke) fetch(ra, kb);
    if (kb + kDK < ke) fetch(rb, kb + kDK);
    for (uint32_t k0 = kb; k0 < ke; k0 += 2 * kDK) {
        stash(ra);
        __syncthreads();
        if (k0 + 2 * kDK < ke) fetch(ra, k0 + 2 * kDK);
        mma();
        __syncthreads();
        if (k0 + kDK < ke) {
            stash(rb);
            __syncthreads();
            if (k0 + 3 * kDK < ke) fetch(rb, k0 + 3 * kDK);
            mma();
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------- wide V-GEMM
// Tall-K V = Y_(n) P for R in (32, 64] (C5: I 256, K = R^3 = 262144): one CTA
// per K-chunk holds up to 256 rows of V (128 for the dual form), so P (Q0,
// extrapolated on the fly) is read once per chunk instead of once per 64-row
// block.  16 warps; warp w owns a 32-row x 32-column block of V (32 x 16 of
// V and of Vfit for the dual form): per 4-k step 4 A + 4 B fragment loads
// feed 16 DMMAs.  Y
// tiles (16 k) stream in through cp.async into a 3-stage ring; P (and F =
// Q0 for the dual form) go through registers because the extrapolation
// P = Q0 + beta (Q0 - alpha H) is applied on the way (the same expression
// as the reference, solvers.hpp:75-86).  Y layouts: J % 16 == 0 (a 16-k tile
// is 16 consecutive j of one o: rows i contiguous in k, smem [i][k]) or
// J == 1 (k = o: 16 rows of I contiguous i, smem [k][i]); other shapes use
// vgemm_dmma_kernel.  Split-K partials are summed by reduce_splits.
constexpr int kWT = 512, kWK = 16, kWStages = 3;
constexpr int kWLdA = kWK + 4;    // smem [i][k] row stride (J % 16 == 0)
constexpr int kWLdP = 64 + 4;     // P / F tile [k][c]
template <bool DUAL>
struct WideCfg {
    static constexpr int WI = DUAL ? 128 : 256;  // rows of V per CTA
    static constexpr int LdB = WI + 4;           // smem [k][i] row stride (J == 1)
    static constexpr int YS = WI * kWLdA > kWK * LdB ? WI * kWLdA : kWK * LdB;  // doubles / Y stage
    static constexpr size_t smem() {
        return (size_t(kWStages) * YS + size_t(kWStages) * kWK * kWLdP * (DUAL ? 2 : 1)) *
               sizeof(double);
    }
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <bool DUAL>
__global__ void __launch_bounds__(kWT, 1) vgemm_wide_kernel(VgemmArgs a, uint64_t kchunk) {
    constexpr int kWI = WideCfg<DUAL>::WI, kWLdB = WideCfg<DUAL>::LdB, kWYS = WideCfg<DUAL>::YS;
    extern __shared__ __align__(16) double wsm[];
    double* ys = wsm;                           // kWStages x kWYS
    double* ps = ys + kWStages * kWYS;          // kWStages x 16 x kWLdP
    double* fs = ps + kWStages * kWK * kWLdP;   // (DUAL) kWStages x 16 x kWLdP
    const int R = int(a.R);
    const uint64_t I = a.I, J = a.J;
    const uint64_t K = a.O * a.J;
    const uint64_t i0 = uint64_t(blockIdx.y) * kWI;
    const uint64_t kb = uint64_t(blockIdx.x) * kchunk;
    const uint64_t ke = min(K, kb + kchunk);
    const int ntile = int((ke - kb + kWK - 1) / kWK);
    const bool jrun = J != 1;  // J % 16 == 0 (host-checked)
    const bool ex = extrap_on(a);
    const double beta = extrap_beta(a);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = lane >> 2, kq = lane & 3;
    // warp tile: rows rw0.., cols cw0..
    constexpr int WR = 32, WC = DUAL ? 16 : 32;
    constexpr int RBW = WR / 8, CBW = WC / 8;
    const int rw0 = (warp % (kWI / WR)) * WR, cw0 = (warp / (kWI / WR)) * WC;

    // issue the loads of tile t into stage st (Y by cp.async; P/F to registers)
    auto load_y = [&](int t, int st) {
        const uint64_t k0 = kb + uint64_t(t) * kWK;
        double* dst = ys + st * kWYS;
        if (jrun) {
            // 256 rows x 16 k = 256 x 8 chunks of 16 B
            const uint64_t o = k0 / J, j0 = k0 - o * J;
#pragma unroll
            for (int u = 0; u < (kWI * kWK / 2) / kWT; ++u) {
                const int e = threadIdx.x + u * kWT;
                const int r = e >> 3, c2 = (e & 7) * 2;
                const uint64_t i = i0 + r;
                const bool ok = i < I && k0 + c2 < ke;
                const double* src = a.y + ((o * I + (ok ? i : 0)) * J + j0 + (ok ? c2 : 0));
                cp_async16(dst + r * kWLdA + c2, src, ok);
            }
        } else {
            // 16 k x 256 rows: J == 1, row o of Y is I contiguous i
#pragma unroll
            for (int u = 0; u < (kWI * kWK / 2) / kWT; ++u) {
                const int e = threadIdx.x + u * kWT;
                const int kk = e / (kWI / 2), r2 = (e % (kWI / 2)) * 2;
                const uint64_t i = i0 + r2;
                const bool ok = k0 + kk < ke && i + 1 < I + 1 && i < I;
                const double* src = a.y + ((ok ? k0 + kk : 0) * I + (ok ? i : 0));
                cp_async16(dst + kk * kWLdB + r2, src, ok);
            }
        }
    };
    constexpr int PPT = (kWK * 64 + kWT - 1) / kWT;  // 2 P elements per thread
    // raw loads only: the extrapolation is applied when the values are
    // stashed, a tile of MMAs later, so the loads' latency is hidden
    auto load_p = [&](int t, double (&pr)[PPT], double (&fr)[PPT]) {
        const uint64_t k0 = kb + uint64_t(t) * kWK;
#pragma unroll
        for (int u = 0; u < PPT; ++u) {
            const int e = threadIdx.x + u * kWT;
            const int kk = e >> 6, c = e & 63;
            const uint64_t k = k0 + kk;
            double q = 0.0, h = 0.0;
            if (k < ke && c < R) {
                q = __ldg(a.q0 + k * R + c);
                if (ex) h = __ldg(a.hist + k * R + c);
            }
            fr[u] = q;
            pr[u] = h;
        }
    };
    auto stash_p = [&](int st, const double (&pr)[PPT], const double (&fr)[PPT]) {
#pragma unroll
        for (int u = 0; u < PPT; ++u) {
            const int e = threadIdx.x + u * kWT;
            const int kk = e >> 6, c = e & 63;
            const double q = fr[u];
            ps[(st * kWK + kk) * kWLdP + c] = ex ? q + beta * (q - a.alpha * pr[u]) : q;
            if (DUAL) fs[(st * kWK + kk) * kWLdP + c] = q;
        }
    };

    double acc[RBW][CBW][2], accf[DUAL ? RBW : 1][DUAL ? CBW : 1][2];
#pragma unroll
    for (int x = 0; x < RBW; ++x)
#pragma unroll
        for (int y = 0; y < CBW; ++y) {
            acc[x][y][0] = acc[x][y][1] = 0.0;
            if (DUAL) accf[x][y][0] = accf[x][y][1] = 0.0;
        }

    double pr[PPT], fr[PPT];
    // prologue: stages 0 .. kWStages-2
#pragma unroll
    for (int t = 0; t < kWStages - 1; ++t) {
        if (t < ntile) {
            load_y(t, t);
            load_p(t, pr, fr);
            stash_p(t, pr, fr);
        }
        cp_async_commit();
    }
    for (int t = 0; t < ntile; ++t) {
        const int st = t % kWStages;
        const int tn = t + kWStages - 1;
        const bool more = tn < ntile;
        if (more) load_p(tn, pr, fr);  // registers, in flight during the MMAs
        cp_async_wait<kWStages - 2>();
        __syncthreads();  // tile t landed; stage (t-1) % S free for reuse
        if (more) load_y(tn, tn % kWStages);
        cp_async_commit();
        const double* y = ys + st * kWYS;
        const double* p = ps + st * kWK * kWLdP;
        const double* f = fs + st * kWK * kWLdP;
#pragma unroll
        for (int k4 = 0; k4 < kWK / 4; ++k4) {
            double af[RBW];
#pragma unroll
            for (int x = 0; x < RBW; ++x) {
                const int r = rw0 + x * 8 + m, kk = 4 * k4 + kq;
                af[x] = jrun ? y[r * kWLdA + kk] : y[kk * kWLdB + r];
            }
#pragma unroll
            for (int yb = 0; yb < CBW; ++yb) {
                const int c = cw0 + yb * 8 + m, kk = 4 * k4 + kq;
                const double bv = p[kk * kWLdP + c];
#pragma unroll
                for (int x = 0; x < RBW; ++x) dmma(acc[x][yb][0], acc[x][yb][1], af[x], bv);
                if (DUAL) {
                    const double fv = f[kk * kWLdP + c];
#pragma unroll
                    for (int x = 0; x < RBW; ++x) dmma(accf[x][yb][0], accf[x][yb][1], af[x], fv);
                }
            }
        }
        if (more) stash_p(tn % kWStages, pr, fr);  // its stage was last read at t - 1
    }
    cp_async_wait<0>();
    // partials of this K-chunk
    double* vp = a.vpart + uint64_t(blockIdx.x) * I * R;
    double* fp = DUAL ? a.vfitpart + uint64_t(blockIdx.x) * I * R : nullptr;
#pragma unroll
    for (int x = 0; x < RBW; ++x) {
        const uint64_t i = i0 + rw0 + x * 8 + m;
        if (i >= I) continue;
#pragma unroll
        for (int yb = 0; yb < CBW; ++yb) {
            const int c = cw0 + yb * 8 + 2 * kq;
            if (c < R) {
                vp[i * R + c] = acc[x][yb][0];
                if (DUAL) fp[i * R + c] = accf[x][yb][0];
            }
            if (c + 1 < R) {
                vp[i * R + c + 1] = acc[x][yb][1];
                if (DUAL) fp[i * R + c + 1] = accf[x][yb][1];
            }
        }
    }
}

size_t vgemm_wide_smem(bool dual) {
    return dual ? WideCfg<true>::smem() : WideCfg<false>::smem();
}

template <int RM, bool DUAL>
__global__ void __launch_bounds__(kDThreads)
vgemm_dmma_kernel(VgemmArgs a, uint64_t kchunk) {
    pdl_entry();
    constexpr int RB = VAcc<RM, DUAL>::RB;
    const int R = a.R;
    const uint64_t I = a.I;
    const uint32_t K = uint32_t(a.O * a.J);
    const uint64_t i0 = uint64_t(blockIdx.x) * kDM;
    const uint32_t kb = uint32_t(uint64_t(blockIdx.y) * kchunk);
    const uint32_t ke = uint32_t(min(uint64_t(K), uint64_t(kb) + kchunk));
    VAcc<RM, DUAL> acc;
    vgemm_tile<RM, DUAL>(a, i0, kb, ke, acc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t i = i0 + warp * 8 + (lane >> 2);
    if (i < I) {
        double* vp = a.vpart + (uint64_t(blockIdx.y) * I + i) * R;
        double* fp = DUAL ? a.vfitpart + (uint64_t(blockIdx.y) * I + i) * R : nullptr;
#pragma unroll
        for (int b = 0; b < RB; ++b) {
            const int r = b * 8 + 2 * (lane & 3);
            if (r < R) {
                vp[r] = acc.v[b][0];
                if (DUAL) fp[r] = acc.f[b][0];
            }
            if (r + 1 < R) {
                vp[r + 1] = acc.v[b][1];
                if (DUAL) fp[r + 1] = acc.f[b][1];
            }
        }
    }
}

// grid (row blocks, 8), cluster (1, 8): CTA y sums K-chunk y; the chunks'
// 64 x RM accumulators meet in shared memory and CTA y reduces rows
// 8y..8y+7 of the block over the cluster in rank order.
template <int RM, bool DUAL>
__global__ void __launch_bounds__(kDThreads)
vgemm_cluster_kernel(VgemmArgs a, uint32_t kchunk) {
    constexpr int RB = VAcc<RM, DUAL>::RB, NV = DUAL ? 2 : 1;
    extern __shared__ double red[];  // NV x kDM x RM
    cg::cluster_group cl = cg::this_cluster();
    const int R = a.R;
    const uint64_t I = a.I;
    const uint32_t K = uint32_t(a.O * a.J);
    const uint64_t i0 = uint64_t(blockIdx.x) * kDM;
    const uint32_t kb = min(K, uint32_t(blockIdx.y) * kchunk);
    const uint32_t ke = min(K, kb + kchunk);
    VAcc<RM, DUAL> acc;
    vgemm_tile<RM, DUAL>(a, i0, kb, ke, acc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = warp * 8 + (lane >> 2);
#pragma unroll
    for (int b = 0; b < RB; ++b) {
        const int c = b * 8 + 2 * (lane & 3);
        red[row * RM + c] = acc.v[b][0];
        red[row * RM + c + 1] = acc.v[b][1];
        if (DUAL) {
            red[kDM * RM + row * RM + c] = acc.f[b][0];
            red[kDM * RM + row * RM + c + 1] = acc.f[b][1];
        }
    }
    cl.sync();
    const int rank = int(cl.block_rank());
    constexpr int kRows = kDM / kVCluster;
    for (int e = threadIdx.x; e < NV * kRows * RM; e += kDThreads) {
        const int v = e / (kRows * RM), rr = (e / RM) % kRows, c = e % RM;
        const int off = v * kDM * RM + (rank * kRows + rr) * RM + c;
        double t[kVCluster];
#pragma unroll
        for (int q = 0; q < kVCluster; ++q) t[q] = cl.map_shared_rank(red, q)[off];
        const double sum = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
        const uint64_t i = i0 + rank * kRows + rr;
        if (i < I && c < R) (v ? a.vfit_out : a.v_out)[i * R + c] = sum;
    }
    cl.sync();  // keep every CTA's shared memory alive until all ranks have read it
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
    pdl_entry();
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        // eight loads in flight per step (the partials come from L2); fixed
        // summation tree -> deterministic
        double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        uint32_t p = 0;
        for (; p + 8 <= nsplit; p += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) s[u] += part[(p + u) * n + e];
        }
        for (; p < nsplit; ++p) s[0] += part[p * n + e];
        out[e] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    }
}

__global__ void permute_rows_kernel(const double* in, double* out, const uint64_t* perm,
                                    uint64_t rows, uint32_t w) {
    const uint64_t n = rows * w;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x)
        out[e] = in[perm[e / w] * w + e % w];
}

template <int RM, bool DUAL>
cudaError_t vgemm_run(VgemmArgs& a, cudaStream_t s, int sms) {
    const uint64_t K = a.O * a.J;
    a.reduced = 0;
    const bool wide = a.R > uint32_t(RM);  // column blocks of the plain kernel
    // short K: one cluster per 64-row block, chunks summed on chip
    static const bool cluster_ok = [] {
        const char* e = std::getenv("CPDB_VGEMM_CLUSTER");
        return !(e && e[0] == '0');
    }();
    if (RM >= 8 && !wide && cluster_ok && a.v_out && (!DUAL || a.vfit_out) &&
        (K + kDK - 1) / kDK <= uint64_t(kVCluster) * kVClusterTiles) {
        const uint64_t iblocks = (a.I + kDM - 1) / kDM;
        const uint64_t ktiles = (K + kDK - 1) / kDK;
        const uint32_t kchunk = uint32_t((ktiles + kVCluster - 1) / kVCluster) * kDK;
        const size_t smem = size_t(DUAL ? 2 : 1) * kDM * RM * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(vgemm_cluster_kernel<RM, DUAL>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t c{};
        c.gridDim = dim3(unsigned(iblocks), kVCluster, 1);
        c.blockDim = dim3(kDThreads, 1, 1);
        c.dynamicSmemBytes = smem;
        c.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = kVCluster;
        attr[0].val.clusterDim.z = 1;
        c.attrs = attr;
        c.numAttrs = 1;  // plain launch: V waits on the Z-QR / chain event
        a.nsplit = 1;
        a.reduced = 1;
        return cudaLaunchKernelEx(&c, vgemm_cluster_kernel<RM, DUAL>, a, kchunk);
    }
    // tall K, R in (32, 64]: the wide kernel (all rows per CTA, P read once)
    static const bool wide_ok = [] {
        const char* e = std::getenv("CPDB_VGEMM_WIDE");
        return !(e && e[0] == '0');
    }();
    if (RM == 64 && !wide && a.R > 32 && wide_ok && (a.J % kWK == 0 || a.J == 1) && K >= (1ull << 16) &&
        (a.I % 2 == 0)) {
        const uint64_t iblocks = (a.I + WideCfg<DUAL>::WI - 1) / WideCfg<DUAL>::WI;
        const uint64_t ktiles = (K + kWK - 1) / kWK;
        uint64_t nsplit = std::max<uint64_t>(1, uint64_t(sms) / iblocks);
        nsplit = std::min<uint64_t>({nsplit, ktiles, uint64_t(vgemm_max_split())});
        const uint64_t kchunk = ((ktiles + nsplit - 1) / nsplit) * kWK;
        nsplit = (K + kchunk - 1) / kchunk;
        a.nsplit = uint32_t(nsplit);
        const size_t smem = vgemm_wide_smem(DUAL);
        cudaError_t e = cudaFuncSetAttribute(vgemm_wide_kernel<DUAL>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
        const dim3 grid{unsigned(nsplit), unsigned(iblocks), 1u};
        vgemm_wide_kernel<DUAL><<<grid, kWT, smem, s>>>(a, kchunk);
        return cudaGetLastError();
    }
    if (RM >= 8 && !wide && K < (1ull << 32)) {  // DMMA path
        const uint64_t iblocks = (a.I + kDM - 1) / kDM;
        const uint64_t ktiles = (K + kDK - 1) / kDK;
        uint64_t nsplit = std::max<uint64_t>(1, (2 * uint64_t(sms)) / iblocks);
        nsplit = std::min<uint64_t>({nsplit, ktiles, uint64_t(vgemm_max_split())});
        // the cap only bites when the CTAs' K-chunks are short (C2: 2 tiles);
        // long-K V-GEMMs (C5) keep the full split
        if (a.max_split)
            nsplit = std::min<uint64_t>(nsplit, std::max<uint64_t>(a.max_split, ktiles / 8));
        const uint64_t kchunk = ((ktiles + nsplit - 1) / nsplit) * kDK;
        nsplit = (K + kchunk - 1) / kchunk;
        a.nsplit = uint32_t(nsplit);
        const dim3 grid{unsigned(iblocks), unsigned(nsplit), 1u};
        // plain launch: V waits on the Z-QR's event (side stream), which
        // programmatic serialisation must not relax
        vgemm_dmma_kernel<RM, DUAL><<<grid, kDThreads, 0, s>>>(a, kchunk);
        return cudaGetLastError();
    }
    const uint64_t iblocks = (a.I + kVBI - 1) / kVBI;
    const uint64_t ktiles = (K + kVBK - 1) / kVBK;
    uint64_t nsplit = std::max<uint64_t>(1, (2 * uint64_t(sms)) / iblocks);
    nsplit = std::min<uint64_t>({nsplit, ktiles, uint64_t(vgemm_max_split())});
    const uint64_t kchunk = ((ktiles + nsplit - 1) / nsplit) * kVBK;
    nsplit = (K + kchunk - 1) / kchunk;
    a.nsplit = uint32_t(nsplit);
    const dim3 grid{unsigned(iblocks), unsigned(nsplit), unsigned((a.R + RM - 1) / RM)};
    // plain launch: V waits on the Z-QR's event (side stream), which
    // programmatic serialisation must not relax
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

namespace {
__global__ void sum_slots_kernel(const double* slots, uint64_t stride, uint32_t world, uint64_t n,
                                 double* out) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        double v = 0.0;
        for (uint32_t r = 0; r < world; ++r) v += slots[r * stride + e];
        out[e] = v;
    }
}
}  // namespace

cudaError_t sum_slots(const double* slots, uint64_t stride, uint32_t world, uint64_t n,
                      double* out, cudaStream_t s) {
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 1024));
    sum_slots_kernel<<<std::max(grid, 1u), 256, 0, s>>>(slots, stride, world, n, out);
    return cudaGetLastError();
}

namespace {
// dst[o * chunk + j] = sum_r slots[r * stride + o * block + rank * chunk + j]
__global__ void sum_slots_scatter_kernel(const double* slots, uint64_t stride, uint32_t world,
                                         uint64_t outer, uint64_t block, uint64_t chunk,
                                         uint32_t rank, double* out) {
    const uint64_t n = outer * chunk;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t o = e / chunk, j = e % chunk;
        const uint64_t src = o * block + uint64_t(rank) * chunk + j;
        double v = 0.0;
        for (uint32_t r = 0; r < world; ++r) v += slots[r * stride + src];
        out[e] = v;
    }
}
}  // namespace

cudaError_t sum_slots_scatter(const double* slots, uint64_t stride, uint32_t world,
                              uint64_t outer, uint64_t block, uint64_t chunk, uint32_t rank,
                              double* out, cudaStream_t s) {
    const uint64_t n = outer * chunk;
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 1024));
    sum_slots_scatter_kernel<<<std::max(grid, 1u), 256, 0, s>>>(slots, stride, world, outer,
                                                                block, chunk, rank, out);
    return cudaGetLastError();
}

uint32_t vgemm_max_split() { return 296; }

namespace {
__global__ void beta_gate_kernel(double* gate, const double* fit, int allow, double gap) {
    pdl_entry();
    const double now = fit[0];
    if (allow && gate[0] == 0.0 && gate[2] != 0.0) {
        // cpdb_select_beta (solvers.hpp:92-101)
        const double prev = gate[3];
        const double p = prev < 0.0 ? 0.0 : (prev > 1.0 ? 1.0 : prev);
        const double q = now < 0.0 ? 0.0 : (now > 1.0 ? 1.0 : now);
        if (!(fabs(q - p) >= gap)) {
            gate[0] = 1.0;
            gate[1] = q > 0.90 ? 1.0 / 2000.0 : (q >= 0.70 ? 1.0 / 500.0 : 1.0 / 250.0);
        }
    }
    gate[3] = now;
    gate[2] = 1.0;
}
}  // namespace

cudaError_t beta_gate(double* gate, const double* fit, int allow, double gap, cudaStream_t s) {
    return launch_pdl(beta_gate_kernel, dim3(1), dim3(1), 0, s, gate, fit, allow, gap);
}  // 2 CTAs per SM on 148 SMs

cudaError_t launch_vgemm(VgemmArgs& a, cudaStream_t s, int sms) {
    const bool d = a.dual != 0;
    if (a.R <= 8) return d ? vgemm_run<8, true>(a, s, sms) : vgemm_run<8, false>(a, s, sms);
    if (a.R <= 16) return d ? vgemm_run<16, true>(a, s, sms) : vgemm_run<16, false>(a, s, sms);
    if (a.R <= 32) return d ? vgemm_run<32, true>(a, s, sms) : vgemm_run<32, false>(a, s, sms);
    // (wider ranks: 64-column blocks of the plain kernel, widerank.cu)
    return d ? vgemm_run<64, true>(a, s, sms) : vgemm_run<64, false>(a, s, sms);
}

cudaError_t reduce_splits(const double* part, uint32_t nsplit, uint64_t n, double* out,
                          cudaStream_t s) {
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 1024));
    return launch_pdl(reduce_splits_kernel, dim3(std::max(grid, 1u)), dim3(256), 0, s, part,
                      nsplit, n, out);
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
