// K1/K2 v2: warp-specialised TMA -> DMMA tensor-times-matrix (sm_100a).
//
// Same contraction as ttm.cu (cpd::ttm, tensor.hpp:288-315, with B = Q_c^T):
//     Y[o][r][j] = sum_k X[o][k][j] Q[k][r]
// One producer warp streams X through a STAGES-deep shared-memory ring with
// the Tensor Memory Accelerator (one cp.async.bulk.tensor per stage, OOB rows
// zero-filled -- that is the K and tail padding) plus a 1-D bulk copy of the
// matching packed-Q chunk; NC consumer warps wait on the stage's mbarrier,
// issue mma.sync.m8n8k4.f64 (DMMA) from the staged tiles with register double
// buffering of the fragments, and release the stage with an mbarrier arrive.
// No __syncthreads in the main loop; one persistent CTA per SM.
//
// Staging layouts (chosen so every fragment load is 256 contiguous bytes):
//   kGroups (inner % 8 == 0): tensor map over X as 4-D {8 j_lo, K, inner/8, outer};
//            smem stage = [G groups][BK][8]  (G = BJ/8; a box may cover several
//            o when inner/8 < G)
//   kRows   (inner == 1, K % 4 == 0): X as 3-D {4 k_lo, M, K/4}; smem stage =
//            [BK/4][BM][4]
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "device.cuh"
#include "kernels.hpp"
#include "launch.hpp"

namespace cpdb {
namespace {

enum Layout { kGroups = 0, kRows = 1 };

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Bulk copies into this CTA's shared memory (.shared::cta destination: the
// TTM grids are launched without a cluster).
__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cta.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <int RB, int CB, int BK, int STAGES, int NC, int LAYOUT>
struct Cfg {
    static constexpr int Rp = RB * 8;
    static constexpr int BJ = NC * CB * 8;   // tile columns (kGroups) / rows (kRows)
    static constexpr int G = BJ / 8;
    static constexpr int XS = BK * BJ;       // doubles per X stage
    static constexpr int QS = BK * Rp;       // doubles per Q stage
    static constexpr int STAGE = XS + QS;
    static constexpr int NT = (NC + 1) * 32;
    static constexpr size_t SMEM = size_t(STAGES) * STAGE * sizeof(double) + 2 * STAGES * 8 + 128;
};

template <int RB, int CB, int BK, int STAGES, int NC, int LAYOUT>
__global__ void __launch_bounds__(Cfg<RB, CB, BK, STAGES, NC, LAYOUT>::NT, 1)
ttm_tma_kernel(const __grid_constant__ CUtensorMap xmap, double* __restrict__ y,
               const double* __restrict__ qp, uint64_t outer, uint64_t K, uint64_t inner,
               uint32_t R, uint64_t ntiles, uint32_t nk) {
    pdl_entry();
    using C = Cfg<RB, CB, BK, STAGES, NC, LAYOUT>;
    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
    uint64_t* empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint64_t first = blockIdx.x;
    const uint64_t gpo = inner / 8;  // 8-column groups per o (kGroups)
    // (tile, k-block) walk with a running ring slot and phase: no 64-bit
    // division on the per-stage path

    if (warp == NC) {
        // ===================== producer: one elected lane issues TMA
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            for (uint64_t tile = first; tile < ntiles; tile += gridDim.x) {
                uint64_t g0 = tile * C::G, go = 0, gi = 0;  // kGroups: (o, group-in-o)
                if (LAYOUT == kGroups) {
                    go = g0 / gpo;
                    gi = g0 % gpo;
                }
                for (uint32_t kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[st], ph ^ 1);
                    const int k0 = int(kb * BK);
                    double* sx = smem + st * C::STAGE;
                    double* sq = sx + C::XS;
                    mbar_expect_tx(&full[st], uint32_t(C::STAGE * sizeof(double)));
                    if (LAYOUT == kGroups) {
                        if (gpo >= uint64_t(C::G)) {
                            tma_4d(sx, &xmap, &full[st], 0, k0, int(gi), int(go));
                        } else {
                            tma_4d(sx, &xmap, &full[st], 0, k0, 0, int(go));
                        }
                    } else if constexpr (C::BJ <= 256) {
                        tma_3d(sx, &xmap, &full[st], 0, int(tile * C::BJ), k0 / 4);
                    } else {
                        // box rows are capped at 256: one box per (k-quad, 256 rows)
#pragma unroll
                        for (int s = 0; s < BK / 4; ++s)
#pragma unroll
                            for (int h = 0; h < C::BJ / 256; ++h)
                                tma_3d(sx + (s * C::BJ + h * 256) * 4, &xmap, &full[st], 0,
                                       int(tile * C::BJ + h * 256), k0 / 4 + s);
                    }
                    bulk_copy(sq, qp + size_t(k0) * C::Rp, uint32_t(C::QS * sizeof(double)),
                              &full[st]);
                    if (++st == STAGES) {
                        st = 0;
                        ph ^= 1;
                    }
                }
            }
        }
        return;
    }

    // ===================== consumers
    double acc[RB][CB][2];
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
        for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    int st = 0;
    uint32_t ph = 0;
    for (uint64_t tile = first; tile < ntiles; tile += gridDim.x) {
#pragma unroll 1
        for (uint32_t kb = 0; kb < nk; ++kb) {
            mbar_wait(&full[st], ph);
            const double* sx = smem + st * C::STAGE;
            const double* sq = sx + C::XS;
            double qf[2][RB], xf[2][CB];
            auto load_frags = [&](int s, int buf) {
#pragma unroll
                for (int rb = 0; rb < RB; ++rb) qf[buf][rb] = sq[(s * C::Rp + rb * 8) * 4 + lane];
#pragma unroll
                for (int cb = 0; cb < CB; ++cb) {
                    const int g = warp * CB + cb;
                    if (LAYOUT == kGroups)
                        xf[buf][cb] = sx[(g * BK + 4 * s + (lane & 3)) * 8 + (lane >> 2)];
                    else
                        xf[buf][cb] = sx[(s * C::BJ + g * 8) * 4 + lane];
                }
            };
            load_frags(0, 0);
#pragma unroll
            for (int s = 0; s < BK / 4; ++s) {
                const int cur = s & 1;
                if (s + 1 < BK / 4) load_frags(s + 1, cur ^ 1);
#pragma unroll
                for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb) {
                        if (LAYOUT == kGroups)
                            dmma(acc[rb][cb][0], acc[rb][cb][1], qf[cur][rb], xf[cur][cb]);
                        else
                            dmma(acc[rb][cb][0], acc[rb][cb][1], xf[cur][cb], qf[cur][rb]);
                    }
            }
            // Release the stage only once its shared-memory reads have
            // RETURNED.  ptxas otherwise issues the empty-barrier arrive right
            // after the last LDS and sinks the DMMAs below it; the arrive can
            // then overtake loads still in flight, and the producer's next
            // TMA write into this slot lands before they read it.  Rare alone,
            // but every run beside CTAs of a DSMEM cluster kernel sharing the
            // SM (their remote shared-memory traffic delays local loads):
            // tools/probes/ttm_coresid.cu, profiles/r02_coresidency_probe.txt.
            // A data dependency on the last k-step's fragments (loaded last;
            // shared loads complete in order -- ptxas itself relies on that
            // when it scoreboards only the last of a run of LDS) makes the
            // arrive wait for them.  The compare is never true: the value is a
            // signalling-NaN pattern that only feeds the (never taken) trap.
            {
                constexpr int lb = (BK / 4 - 1) & 1;
                uint64_t d[RB + CB];
#pragma unroll
                for (int rb = 0; rb < RB; ++rb) d[rb] = __double_as_longlong(qf[lb][rb]);
#pragma unroll
                for (int cb = 0; cb < CB; ++cb) d[RB + cb] = __double_as_longlong(xf[lb][cb]);
#pragma unroll
                for (int w = 1; w < RB + CB; w *= 2)
#pragma unroll
                    for (int i = 0; i + w < RB + CB; i += 2 * w) d[i] ^= d[i + w];
                if (d[0] == 0x7ff400000000deadull) __trap();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == STAGES) {
                st = 0;
                ph ^= 1;
            }
        }
        // tile complete: epilogue straight to HBM
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
            const int g = warp * CB + cb;
            if (LAYOUT == kGroups) {
                const uint64_t gflat = tile * C::G + g;
                const uint64_t o = gflat / gpo, j = (gflat % gpo) * 8 + 2 * (lane & 3);
                if (o < outer) {
#pragma unroll
                    for (int rb = 0; rb < RB; ++rb) {
                        const uint32_t r = rb * 8 + (lane >> 2);
                        if (r < R)
                            *reinterpret_cast<double2*>(y + (o * R + r) * inner + j) =
                                make_double2(acc[rb][cb][0], acc[rb][cb][1]);
                    }
                }
            } else {
                const uint64_t m = tile * C::BJ + uint64_t(g) * 8 + (lane >> 2);
                if (m < outer) {
#pragma unroll
                    for (int rb = 0; rb < RB; ++rb) {
                        const uint32_t r = rb * 8 + 2 * (lane & 3);
                        double* dst = y + m * R + r;
                        if (r + 1 < R && (R % 2 == 0)) {
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
    // the output is read by later grids through TMA (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---------------------------------------------------------------- tensor maps
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

template <int RB, int CB, int BK, int STAGES, int NC, int LAYOUT>
cudaError_t launch_v2(const TtmArgs& a, cudaStream_t s, int sms) {
    using C = Cfg<RB, CB, BK, STAGES, NC, LAYOUT>;
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap map;
    CUresult r;
    if (LAYOUT == kGroups) {
        const uint64_t gpo = a.inner / 8;
        const cuuint64_t dims[4] = {8, a.K, gpo, a.outer};
        const cuuint64_t strides[3] = {a.inner * 8, 64, a.K * a.inner * 8};
        cuuint32_t box[4];
        if (gpo >= uint64_t(C::G)) {
            // a tile would straddle two o (outer == 1: the last tile's
            // columns past the end are zero-filled and not stored)
            if (gpo % C::G != 0 && a.outer != 1) return cudaErrorNotSupported;
            box[0] = 8; box[1] = BK; box[2] = C::G; box[3] = 1;
        } else {
            if (C::G % gpo != 0) return cudaErrorNotSupported;
            box[0] = 8; box[1] = BK; box[2] = cuuint32_t(gpo); box[3] = cuuint32_t(C::G / gpo);
        }
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(a.x), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        if (C::BJ > 256 && C::BJ % 256 != 0) return cudaErrorNotSupported;  // partial box
        const cuuint64_t dims[3] = {4, a.outer, a.K / 4};
        const cuuint64_t strides[2] = {a.K * 8, 32};
        const cuuint32_t box[3] = {4, cuuint32_t(C::BJ <= 256 ? C::BJ : 256),
                                   cuuint32_t(C::BJ <= 256 ? BK / 4 : 1)};
        const cuuint32_t estr[3] = {1, 1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(a.x), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
        static bool warned = false;
        if (!warned && std::getenv("CPDB_DEBUG")) {
            std::fprintf(stderr, "cpdb: tensor map encode failed (%d) layout %d outer %llu K %llu "
                         "inner %llu; using the cp.async kernel\n", int(r), LAYOUT,
                         (unsigned long long)a.outer, (unsigned long long)a.K,
                         (unsigned long long)a.inner);
            warned = true;
        }
        return cudaErrorNotSupported;
    }
    auto kern = ttm_tma_kernel<RB, CB, BK, STAGES, NC, LAYOUT>;
    // Each CTA requests its ring's shared memory only, so CTAs of other
    // grids (the 8-CTA finisher / Z-QR clusters) may share its SM.  Round 1
    // reserved the whole 227 KB instead: beside DSMEM cluster CTAs this
    // kernel's results differed run to run.  The cause was the consumer
    // release above (the empty-barrier arrive overtaking in-flight shared
    // loads); with the data dependency the probe shows 0 differing runs
    // where the old build differed in every one (profiles/
    // r02_coresidency_probe.txt).  CPDB_TTM_SMEM_WHOLE=1 restores the
    // reservation (A/B testing).
    static const bool whole_sm = [] {
        const char* e = std::getenv("CPDB_TTM_SMEM_WHOLE");
        return e && e[0] == '1';
    }();
    const size_t smem = whole_sm ? size_t(227 * 1024) : C::SMEM;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    const uint64_t ncols = LAYOUT == kGroups ? (a.outer * a.inner) / 8 : a.outer;  // groups or rows
    const uint64_t per_tile = LAYOUT == kGroups ? C::G : C::BJ;
    const uint64_t ntiles = (ncols + per_tile - 1) / per_tile;
    const uint32_t nk = static_cast<uint32_t>((a.K + BK - 1) / BK);
    // non-persistent form: two tiles per CTA (CPDB_PREFETCH_TPC), so
    // concurrent high-priority grids get SMs as CTAs retire while the per-CTA
    // prologue is paid half as often (measured, C2: 1 tile 2204 sweeps/s, 2
    // tiles 2248, 4 tiles 2116 -- the overlapped update then waits for SMs)
    const char* tpe = std::getenv("CPDB_PREFETCH_TPC");
    const uint64_t tpc = tpe ? std::max(1, std::atoi(tpe)) : (a.tiles_per_cta ? a.tiles_per_cta : 2);
    const uint64_t grid = a.one_tile_per_cta ? (ntiles + tpc - 1) / tpc
                                             : std::min<uint64_t>(ntiles, uint64_t(sms));
    if (grid == 0) return cudaSuccess;
    if (a.no_pdl) {
        kern<<<unsigned(grid), C::NT, smem, s>>>(map, a.y, a.qp, a.outer, a.K, a.inner, a.R,
                                                   ntiles, nk);
        return cudaGetLastError();
    }
    return launch_pdl(kern, dim3(unsigned(grid)), dim3(C::NT), smem, s, map, a.y, a.qp, a.outer,
                      a.K, a.inner, a.R, ntiles, nk);
}

// Tiles a launch would have with CB column blocks per consumer warp.
template <int LAYOUT>
uint64_t tiles_with(const TtmArgs& a, int cb, int nc) {
    const uint64_t per = uint64_t(nc) * cb * (LAYOUT == kGroups ? 1 : 8);
    const uint64_t cols = LAYOUT == kGroups ? (a.outer * a.inner) / 8 : a.outer;
    return (cols + per - 1) / per;
}

// Whether a tile of nc*cb 8-column groups fits the kGroups box rule (a tile
// never straddles two o unless there is only one).
template <int LAYOUT>
bool tile_ok(const TtmArgs& a, int cb, int nc) {
    // kRows boxes carry at most 256 rows: wider tiles take whole boxes
    if (LAYOUT != kGroups) return nc * cb * 8 <= 256 || (nc * cb * 8) % 256 == 0;
    const uint64_t g = uint64_t(nc) * cb, gpo = a.inner / 8;
    return gpo >= g ? (gpo % g == 0 || a.outer == 1) : (g % gpo == 0);
}

// Pick the tile (CB0, CB0/2, CB0/4 column blocks per warp; 8 or 7 consumer
// warps) that best fills the GPU: score = SM utilisation of the last wave x
// a per-CB efficiency (narrower tiles re-load Q fragments more often per
// DMMA).  Branch TTMs on the R-sized intermediates are small (C2: 16384 rows
// -> 64 tiles at CB 4, 128 at CB 2 = 86% of 148 SMs); 7 consumer warps make
// 112-row tiles, 147 of them (99%).
template <int RB, int CB0, int BK, int ST, int LAYOUT>
cudaError_t launch_adaptive(const TtmArgs& a, cudaStream_t s, int sms) {
    // Large (root-sized) TTMs: the widest tile with 16 consumer warps of half
    // the column blocks each -- the same tile, four warps per SMSP instead of
    // two, which hides the DMMA issue spacing (ncu's top stall, `wait`):
    // C2 root 265.2 -> 260.6 us (87.3 -> 88.8% of peak), C5 16.52 -> 16.30 ms
    // (89.6 -> 90.8%), C2 2501 -> 2545 sweeps/s.  CPDB_TTM_NC16=0: 8 warps;
    // =2: also the (smaller) branch TTMs.
    if constexpr (CB0 >= 2) {
        static const int nc16 = [] {
            const char* e = std::getenv("CPDB_TTM_NC16");
            return e ? std::atoi(e) : 1;
        }();
        // (CPDB_TTM_ROOTCFG=1..3: tile-shape experiments for the root)
        static const int rootcfg = [] {
            const char* e = std::getenv("CPDB_TTM_ROOTCFG");
            return e ? std::atoi(e) : 0;
        }();
        const bool root_sized = tiles_with<LAYOUT>(a, CB0, 8) >= uint64_t(2 * sms);
        if (rootcfg && root_sized) {
            if constexpr (RB == 4 && CB0 == 4) {
                if (rootcfg == 1 && tile_ok<LAYOUT>(a, 4, 16))
                    return launch_v2<4, 4, 8, 6, 16, LAYOUT>(a, s, sms);
                if (rootcfg == 2 && tile_ok<LAYOUT>(a, 4, 16))
                    return launch_v2<4, 4, 8, 5, 16, LAYOUT>(a, s, sms);
                if (rootcfg == 3 && tile_ok<LAYOUT>(a, 2, 16))
                    return launch_v2<4, 2, 8, 8, 16, LAYOUT>(a, s, sms);
            }
            if constexpr (RB == 2 && CB0 == 8) {
                if (rootcfg == 1 && tile_ok<LAYOUT>(a, 8, 16))
                    return launch_v2<2, 8, 8, 3, 16, LAYOUT>(a, s, sms);
            }
        }
        // R in (56, 64]: 16 warps of 8 x 2 accumulator blocks, 16-deep k
        // stages, five of them (C5 root 16.30 -> 15.33 ms = 96.6% of the
        // DMMA peak, 28.1 -> 29.1 sweeps/s); the other tile shapes measured
        // no better at their R (C2: 5 or 6 stages alike, wider tiles worse)
        if constexpr (RB == 8 && CB0 == 2) {
            if (nc16 > 0 && (nc16 > 1 || root_sized) && tile_ok<LAYOUT>(a, 2, 16))
                return launch_v2<8, 2, 16, 5, 16, LAYOUT>(a, s, sms);
        }
        if (nc16 > 0 && (nc16 > 1 || root_sized) && tile_ok<LAYOUT>(a, CB0 / 2, 16))
            return launch_v2<RB, CB0 / 2, BK, ST, 16, LAYOUT>(a, s, sms);
    }
    int best = CB0, best_nc = 8;
    double best_score = -1.0;
    // opt-in (CPDB_TTM_NC7=1): measured at C2, 147-CTA branch TTMs leave no
    // SMs for the concurrent 8-CTA cluster kernels and lose 1.2% sweeps/s
    // against 128-CTA ones
    static const bool nc7 = [] {
        const char* e = std::getenv("CPDB_TTM_NC7");
        return e && e[0] == '1';
    }();
    for (int nc = 8; nc >= (nc7 ? 7 : 8); --nc)
        for (int cb = CB0; cb >= 1 && cb >= CB0 / 4; cb /= 2) {
            if (!tile_ok<LAYOUT>(a, cb, nc)) continue;
            const uint64_t t = tiles_with<LAYOUT>(a, cb, nc);
            const double waves = std::ceil(double(t) / sms);
            const double util = double(t) / (waves * sms);
            const double eff = (cb == CB0 ? 1.0 : (cb == CB0 / 2 ? 0.9 : 0.7)) *
                               (nc == 8 ? 1.0 : 0.97);
            const double score = util * eff;
            if (score > best_score + 1e-9) {
                best_score = score;
                best = cb;
                best_nc = nc;
            }
        }
    if (best_nc == 7) {
        if constexpr (CB0 >= 4) {
            if (best == CB0 / 4) return launch_v2<RB, CB0 / 4, BK, ST, 7, LAYOUT>(a, s, sms);
        }
        if constexpr (CB0 >= 2) {
            if (best == CB0 / 2) return launch_v2<RB, CB0 / 2, BK, ST, 7, LAYOUT>(a, s, sms);
        }
        return launch_v2<RB, CB0, BK, ST, 7, LAYOUT>(a, s, sms);
    }
    if constexpr (CB0 >= 4) {
        if (best == CB0 / 4) return launch_v2<RB, CB0 / 4, BK, ST, 8, LAYOUT>(a, s, sms);
    }
    if constexpr (CB0 >= 2) {
        if (best == CB0 / 2) return launch_v2<RB, CB0 / 2, BK, ST, 8, LAYOUT>(a, s, sms);
    }
    return launch_v2<RB, CB0, BK, ST, 8, LAYOUT>(a, s, sms);
}

template <int LAYOUT>
cudaError_t dispatch_v2(const TtmArgs& a, cudaStream_t s, int sms) {
    // X stage ~32 KB at the widest tile; 4-5 stages in flight
    switch (a.Rp / 8) {
        case 1: return launch_adaptive<1, 8, 8, 5, LAYOUT>(a, s, sms);
        case 2: return launch_adaptive<2, 8, 8, 5, LAYOUT>(a, s, sms);
        case 3: return launch_adaptive<3, 4, 16, 5, LAYOUT>(a, s, sms);
        case 4: return launch_adaptive<4, 4, 16, 6, LAYOUT>(a, s, sms);
        case 5: return launch_adaptive<5, 2, 32, 4, LAYOUT>(a, s, sms);
        case 6: return launch_adaptive<6, 2, 32, 4, LAYOUT>(a, s, sms);
        case 7: return launch_adaptive<7, 2, 32, 4, LAYOUT>(a, s, sms);
        case 8: return launch_adaptive<8, 2, 32, 4, LAYOUT>(a, s, sms);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

// Returns cudaErrorNotSupported when the shape cannot use the TMA path (the
// caller falls back to the cp.async kernel).
cudaError_t launch_ttm_tma(const TtmArgs& a, cudaStream_t s, int sms) {
    if (a.Rp > 64 || a.R == 0) return cudaErrorNotSupported;
    if (a.inner % 8 == 0 && a.K < (1u << 31) && a.outer < (1u << 31) && a.inner / 8 < (1u << 31))
        return dispatch_v2<kGroups>(a, s, sms);
    if (a.inner == 1 && a.K % 4 == 0 && a.outer < (1u << 31)) return dispatch_v2<kRows>(a, s, sms);
    return cudaErrorNotSupported;
}

}  // namespace cpdb
