// K1/K2: tensor-times-matrix on the device.
//
// Replaces cpd::ttm (/root/reference/proj/include/cpd/tensor.hpp:288-315) as
// called by execute() with B = Q_c^T (dim_tree.hpp:519-521):
//     Y[o][r][j] = sum_k X[o][k][j] * Q[k][r]
// with X viewed as [outer][K][inner] (outer = prod of extents before the
// contracted mode c, K = I_c, inner = prod after) and Y as [outer][R][inner].
//
// The contraction runs on the FP64 tensor cores (mma.sync m8n8k4 f64 ->
// DMMA.8x8x4; tcgen05 has no f64 kind).  One persistent CTA per SM streams
// X through a cp.async multi-stage shared-memory ring while 8 warps issue
// DMMAs; Q stays tiny and is re-read per stage from L2 in a pre-packed
// fragment layout.  Two X layouts cover all contraction positions:
//   kGroups  (inner % 8 == 0): 8-column groups of the flat (o, j) space; a
//            group's BK rows land as one 64 B-per-row slab -> conflict-free
//            fragment loads.  First and middle modes, and branch TTMs whose
//            trailing extent is a multiple of 8.
//   kRows    (inner == 1, K even): rows of X are contiguous in K; staged as
//            [BK/4][BM][4].  Last-mode contractions.
// Anything else (odd extents in the small reference tests) takes a plain
// one-thread-per-output kernel.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "kernels.hpp"
#include "launch.hpp"

namespace cpdb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / kWarp;

enum Layout { kGroups = 0, kRows = 1 };

template <int RB, int CB, int BK, int STAGES, int LAYOUT>
struct TtmCfg {
    static constexpr int Rp = RB * 8;
    static constexpr int BJ = kWarps * CB * 8;  // columns (kGroups) or rows (kRows) per tile
    static constexpr int XS = BK * BJ;          // doubles per X stage
    static constexpr int QS = BK * Rp;          // doubles per Q stage
    static constexpr int STAGE = XS + QS;
    static constexpr size_t SMEM = size_t(STAGES) * STAGE * sizeof(double);
    static_assert(BK % 4 == 0, "BK multiple of the MMA k");
};

template <int RB, int CB, int BK, int STAGES, int LAYOUT>
__global__ void __launch_bounds__(kThreads)
ttm_dmma_kernel(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ qp,
                uint64_t outer, uint64_t K, uint64_t inner, uint32_t R, uint64_t ntiles,
                uint32_t nk, uint32_t Rtot) {
    // (R: columns of this launch; Rtot: Y's extent in the contracted position
    // -- larger than R when a wide rank is computed in 64-column blocks, y
    // then points at the block's first column)
    pdl_entry();
    using C = TtmCfg<RB, CB, BK, STAGES, LAYOUT>;
    extern __shared__ __align__(128) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const uint64_t ncols = (LAYOUT == kGroups) ? outer * inner : outer;  // rows for kRows
    // Per-thread fixed copy coordinates.
    // kGroups: chunk = (kk, g, part); 4 chunks of 16 B per 8-double row.
    // kRows:   chunk = (m, kk pair).
    constexpr int G4 = C::BJ / 2;              // kGroups: chunks per k-row
    constexpr int HC = BK / 2;                 // kRows: chunks per X row
    constexpr int XCH = C::XS / 2;             // 16-B chunks per X stage
    constexpr int XPER = XCH / kThreads;       // per thread
    constexpr int QCH = C::QS / 2;
    static_assert(XCH % kThreads == 0, "X stage must split evenly");

    const uint64_t first = blockIdx.x;
    const uint64_t my_tiles = first < ntiles ? (ntiles - 1 - first) / gridDim.x + 1 : 0;
    const uint64_t total = my_tiles * nk;

    double acc[RB][CB][2];
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
        for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    // ---- producer: stage `t` (tile, k-chunk) -> ring slot t % STAGES ----------
    auto issue = [&](uint64_t t) {
        if (t >= total) return;
        const uint64_t tile = first + (t / nk) * gridDim.x;
        const uint32_t kc = static_cast<uint32_t>(t % nk);
        const uint64_t k0 = uint64_t(kc) * BK;
        double* sx = smem + (t % STAGES) * C::STAGE;
        double* sq = sx + C::XS;
        if (LAYOUT == kGroups) {
            static_assert(kThreads % G4 == 0 || G4 % kThreads == 0, "copy map");
            const int g = (tid % G4) / 4, part = tid % 4;
            const uint64_t c0 = tile * C::BJ + uint64_t(g) * 8;
            const bool cvalid = c0 < ncols;
            const uint64_t o = cvalid ? c0 / inner : 0, j = cvalid ? c0 % inner : 0;
            const double* base = x + (o * K) * inner + j + part * 2;
#pragma unroll
            for (int i = 0; i < XPER; ++i) {
                const int kk = tid / G4 + i * (kThreads / G4);
                const uint64_t k = k0 + kk;
                const bool ok = cvalid && k < K;
                const double* src = ok ? base + k * inner : x;
                cp_async16(sx + (g * BK + kk) * 8 + part * 2, src, ok ? 16u : 0u);
            }
        } else {
            const int kk = (tid % HC) * 2;
#pragma unroll
            for (int i = 0; i < XPER; ++i) {
                const int m = tid / HC + i * (kThreads / HC);
                const uint64_t row = tile * C::BJ + m;
                const uint64_t k = k0 + kk;
                const bool ok = row < ncols && k < K;
                const double* src = ok ? x + row * K + k : x;
                cp_async16(sx + ((kk / 4) * C::BJ + m) * 4 + (kk % 4), src, ok ? 16u : 0u);
            }
        }
        const double* qsrc = qp + k0 * C::Rp;  // packed [Kpad/4][Rp][4], contiguous per chunk
        for (int i = tid; i < QCH; i += kThreads) cp_async16(sq + 2 * i, qsrc + 2 * i, 16u);
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        issue(s);
        cp_async_commit();
    }

    for (uint64_t t = 0; t < total; ++t) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        issue(t + STAGES - 1);
        cp_async_commit();

        const double* sx = smem + (t % STAGES) * C::STAGE;
        const double* sq = sx + C::XS;
#pragma unroll
        for (int s = 0; s < BK / 4; ++s) {
            double qf[RB], xf[CB];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) qf[rb] = sq[(s * C::Rp + rb * 8) * 4 + lane];
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) {
                const int g = warp * CB + cb;
                if (LAYOUT == kGroups)
                    xf[cb] = sx[(g * BK + 4 * s + (lane & 3)) * 8 + (lane >> 2)];
                else
                    xf[cb] = sx[(s * C::BJ + g * 8) * 4 + lane];
            }
#pragma unroll
            for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                for (int cb = 0; cb < CB; ++cb) {
                    if (LAYOUT == kGroups)
                        dmma(acc[rb][cb][0], acc[rb][cb][1], qf[rb], xf[cb]);
                    else
                        dmma(acc[rb][cb][0], acc[rb][cb][1], xf[cb], qf[rb]);
                }
        }

        if (t % nk == nk - 1) {  // tile complete: epilogue straight to HBM
            const uint64_t tile = first + (t / nk) * gridDim.x;
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) {
                const int g = warp * CB + cb;
                if (LAYOUT == kGroups) {
                    const uint64_t c0 = tile * C::BJ + uint64_t(g) * 8;
                    if (c0 < ncols) {
                        const uint64_t o = c0 / inner, j = c0 % inner + 2 * (lane & 3);
#pragma unroll
                        for (int rb = 0; rb < RB; ++rb) {
                            const uint32_t r = rb * 8 + (lane >> 2);
                            if (r < R)
                                *reinterpret_cast<double2*>(y + (o * Rtot + r) * inner + j) =
                                    make_double2(acc[rb][cb][0], acc[rb][cb][1]);
                        }
                    }
                } else {
                    const uint64_t m = tile * C::BJ + uint64_t(g) * 8 + (lane >> 2);
                    if (m < ncols) {
#pragma unroll
                        for (int rb = 0; rb < RB; ++rb) {
                            const uint32_t r = rb * 8 + 2 * (lane & 3);
                            double* dst = y + m * Rtot + r;
                            if (r + 1 < R && (Rtot % 2 == 0)) {
                                *reinterpret_cast<double2*>(dst) =
                                    make_double2(acc[rb][cb][0], acc[rb][cb][1]);
                            } else {
                                if (r < R) dst[0] = acc[rb][cb][0];
                                if (r + 1 < R) dst[1] = acc[rb][cb][1];
                            }
                        }
                    }
                }
#pragma unroll
                for (int rb = 0; rb < RB; ++rb) acc[rb][cb][0] = acc[rb][cb][1] = 0.0;
            }
        }
    }
    cp_async_wait<0>();
}

// Fallback for shapes the tensor-core layouts do not cover: one thread per
// output element, ascending k (same accumulation order as the reference).
__global__ void ttm_simple_kernel(const double* __restrict__ x, double* __restrict__ y,
                                  const double* __restrict__ q, uint64_t outer, uint64_t K,
                                  uint64_t inner, uint32_t R) {
    pdl_entry();
    const uint64_t n = outer * R * inner;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < n;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t j = idx % inner, r = (idx / inner) % R, o = idx / (inner * R);
        const double* xs = x + o * K * inner + j;
        double acc = 0.0;
        for (uint64_t k = 0; k < K; ++k) acc = fma(xs[k * inner], q[k * R + r], acc);
        y[idx] = acc;
    }
}

// Q (K x R row-major) -> [Kpad/4][Rp][4] fragment order, zero padded.
__global__ void pack_q_kernel(const double* __restrict__ q, double* __restrict__ qp, uint32_t K,
                              uint32_t R, uint32_t Kpad, uint32_t Rp) {
    pdl_entry();
    const uint32_t n = Kpad * Rp;
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += gridDim.x * blockDim.x) {
        const uint32_t kq = idx % 4, r = (idx / 4) % Rp, kg = idx / (4 * Rp);
        const uint32_t k = kg * 4 + kq;
        qp[idx] = (k < K && r < R) ? q[size_t(k) * R + r] : 0.0;
    }
}

// columns [c0, c0 + Rc) of a K x ld matrix, packed like a K x Rc Q of their own
__global__ void pack_q_cols_kernel(const double* __restrict__ q, double* __restrict__ qp,
                                   uint32_t K, uint32_t ld, uint32_t c0, uint32_t Rc,
                                   uint32_t Kpad, uint32_t Rp) {
    pdl_entry();
    const uint32_t n = Kpad * Rp;
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += gridDim.x * blockDim.x) {
        const uint32_t kq = idx % 4, r = (idx / 4) % Rp, kg = idx / (4 * Rp);
        const uint32_t k = kg * 4 + kq;
        qp[idx] = (k < K && r < Rc) ? q[size_t(k) * ld + c0 + r] : 0.0;
    }
}

// R > 64: block b (columns 64b .. 64b+63) packed like a 64-column Q of its
// own, [Kpad/4][64][4], the blocks one after the other
__global__ void pack_q_blocks_kernel(const double* __restrict__ q, double* __restrict__ qp,
                                     uint32_t K, uint32_t R, uint32_t Kpad) {
    const uint32_t per = Kpad * 64, n = per * ((R + 63) / 64);
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += gridDim.x * blockDim.x) {
        const uint32_t b = idx / per, e = idx % per;
        const uint32_t kq = e % 4, r = b * 64 + (e / 4) % 64, k = (e / 256) * 4 + kq;
        qp[idx] = (k < K && r < R) ? q[size_t(k) * R + r] : 0.0;
    }
}

template <int RB, int CB, int BK, int STAGES, int LAYOUT>
cudaError_t launch_cfg(const TtmArgs& a, cudaStream_t s, int sms) {
    using C = TtmCfg<RB, CB, BK, STAGES, LAYOUT>;
    auto kern = ttm_dmma_kernel<RB, CB, BK, STAGES, LAYOUT>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const uint64_t ncols = LAYOUT == kGroups ? a.outer * a.inner : a.outer;
    const uint64_t ntiles = (ncols + C::BJ - 1) / C::BJ;
    const uint32_t nk = static_cast<uint32_t>((a.K + BK - 1) / BK);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, C::SMEM);
    per_sm = std::max(per_sm, 1);
    const uint64_t grid = std::min<uint64_t>(ntiles, uint64_t(sms) * per_sm);
    if (grid == 0) return cudaSuccess;
    return launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(kThreads), C::SMEM, s, a.x,
                      a.y, a.qp, a.outer, a.K, a.inner, a.R, ntiles, nk, a.Rtot ? a.Rtot : a.R);
}

// Tile shapes per padded rank: RB*CB accumulator tiles per warp <= 16, and an
// X stage of 32 KB (BK * BJ * 8 B).
template <int LAYOUT>
cudaError_t dispatch(const TtmArgs& a, cudaStream_t s, int sms) {
    switch (a.Rp / 8) {
        case 1: return launch_cfg<1, 8, 8, 4, LAYOUT>(a, s, sms);
        case 2: return launch_cfg<2, 8, 8, 4, LAYOUT>(a, s, sms);
        case 3: return launch_cfg<3, 4, 16, 4, LAYOUT>(a, s, sms);
        case 4: return launch_cfg<4, 4, 16, 4, LAYOUT>(a, s, sms);
        case 5: return launch_cfg<5, 2, 32, 3, LAYOUT>(a, s, sms);
        case 6: return launch_cfg<6, 2, 32, 3, LAYOUT>(a, s, sms);
        case 7: return launch_cfg<7, 2, 32, 3, LAYOUT>(a, s, sms);
        case 8: return launch_cfg<8, 2, 32, 3, LAYOUT>(a, s, sms);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

uint32_t ttm_kpad(uint64_t K) { return static_cast<uint32_t>(((K + 31) / 32) * 32); }
// (wide ranks: whole 64-column blocks, each packed on its own)
uint32_t ttm_rpad(uint32_t R) { return R <= 64 ? ((R + 7) / 8) * 8 : ((R + 63) / 64) * 64; }

cudaError_t pack_q(const double* q, double* qp, uint32_t K, uint32_t R, cudaStream_t s) {
    const uint32_t Kpad = ttm_kpad(K), Rp = ttm_rpad(R);
    if (R > 64) {
        const uint32_t n = Kpad * Rp;
        pack_q_blocks_kernel<<<(n + 255) / 256, 256, 0, s>>>(q, qp, K, R, Kpad);
        return cudaGetLastError();
    }
    const uint32_t n = Kpad * Rp;
    return launch_pdl(pack_q_kernel, dim3((n + 255) / 256), dim3(256), 0, s, q, qp, K, R, Kpad,
                      Rp);
}

cudaError_t pack_q_cols(const double* q, uint32_t ld, uint32_t c0, uint32_t Rc, double* qp,
                        uint32_t K, cudaStream_t s) {
    if (Rc > 64) return cudaErrorInvalidValue;
    const uint32_t Kpad = ttm_kpad(K), Rp = ttm_rpad(Rc);
    const uint32_t n = Kpad * Rp;
    return launch_pdl(pack_q_cols_kernel, dim3((n + 255) / 256), dim3(256), 0, s, q, qp, K, ld, c0,
                      Rc, Kpad, Rp);
}

TtmPath ttm_path(const TtmArgs& a) {
    if (a.R == 0) return TtmPath::simple;
    if (a.inner % 8 == 0) return TtmPath::groups;
    if (a.inner == 1 && a.K % 2 == 0) return TtmPath::rows;
    return TtmPath::simple;
}

cudaError_t launch_ttm(const TtmArgs& a, cudaStream_t s, int sms) {
    static const int version = [] {
        const char* v = std::getenv("CPDB_TTM");
        return v ? std::atoi(v) : 2;
    }();
    if (version >= 2 && a.qp != nullptr && !a.no_tma) {
        const cudaError_t e = launch_ttm_tma(a, s, sms);  // warp-specialised TMA path
        if (e != cudaErrorNotSupported) return e;
    }
    if (a.R > 64 && a.qp != nullptr && ttm_path(a) != TtmPath::simple) {
        // wide rank: one pass over X per 64-column block of Q (pack_q's
        // blocked layout), each writing its columns of Y
        const bool groups = ttm_path(a) == TtmPath::groups;
        const uint32_t kpad = ttm_kpad(a.K);
        for (uint32_t b = 0; b * 64 < a.R; ++b) {
            TtmArgs ab = a;
            ab.R = std::min<uint32_t>(64, a.R - b * 64);
            ab.Rp = 64;
            ab.Rtot = a.R;
            ab.qp = a.qp + size_t(b) * kpad * 64;
            ab.y = a.y + (groups ? uint64_t(b) * 64 * a.inner : uint64_t(b) * 64);
            const cudaError_t e = groups ? dispatch<kGroups>(ab, s, sms) : dispatch<kRows>(ab, s, sms);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    switch (ttm_path(a)) {
        case TtmPath::groups: return dispatch<kGroups>(a, s, sms);
        case TtmPath::rows: return dispatch<kRows>(a, s, sms);
        case TtmPath::simple: {
            const uint64_t n = a.outer * a.R * a.inner;
            const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4096));
            return launch_pdl(ttm_simple_kernel, dim3(std::max(grid, 1u)), dim3(256), 0, s, a.x,
                              a.y, a.q, a.outer, a.K, a.inner, a.R);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace cpdb
