// Co-residency probe: is the TMA TTM kernel (ttm_tma.cu) bit-reproducible
// while CTAs of another grid share its SMs?  Runs the same contraction many
// times, each on a stream next to a "hog" grid, and compares every output
// with the first, isolated, run.
//
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 \
//   -I paper_2503_18759_b200/csrc -I include tools/probes/ttm_coresid.cu \
//   -L paper_2503_18759_b200 -lcpdb -Xlinker -rpath,'$ORIGIN/../../paper_2503_18759_b200' \
//   -o tools/probes/ttm_coresid
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace cg = cooperative_groups;

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e_));                \
            std::exit(1);                                                       \
        }                                                                       \
    } while (0)

// hog: each CTA holds `smem` bytes and hammers shared memory for `iters`
__global__ void hog_kernel(int iters, double* sink) {
    extern __shared__ double sh[];
    const int n = 2048;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = i;
    __syncthreads();
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        const int j = (threadIdx.x * 7 + it * 13) & (n - 1);
        acc += sh[j];
        sh[(j + 5) & (n - 1)] = acc * 1e-9;
    }
    if (acc == 1234.5) sink[0] = acc;
}

// cluster hog: 8-CTA clusters that keep a pattern in shared memory and read
// it back through DSMEM; counts words that are not what their owner wrote
__global__ void cluster_hog_kernel(int iters, unsigned long long* bad, int dsmem) {
    extern __shared__ double sh[];
    cg::cluster_group cl = cg::this_cluster();
    const int n = 4096;
    const unsigned rank = cl.block_rank();
    for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = double(blockIdx.x * 8192 + i);
    cl.sync();
    unsigned long long nb = 0;
    for (int it = 0; it < iters; ++it) {
        const unsigned peer = dsmem ? (rank + 1 + it) % 8 : rank;
        if (dsmem == 2) {  // remote writes of the peer's own pattern
            double* q = cl.map_shared_rank(sh, peer);
            const int i = (threadIdx.x * 37 + it * 101) & (n - 1);
            const unsigned pb = blockIdx.x - rank + peer;
            q[i] = double(pb * 8192 + i);
            continue;
        }
        const double* p = cl.map_shared_rank(sh, peer);
        const int i = (threadIdx.x * 37 + it * 101) & (n - 1);
        const unsigned pb = blockIdx.x - rank + peer;
        if (p[i] != double(pb * 8192 + i)) ++nb;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (sh[i] != double(blockIdx.x * 8192 + i)) ++nb;
    cl.sync();
    if (nb) atomicAdd(bad, nb);
}

__global__ void fill(double* p, uint64_t n, uint64_t seed) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
        z ^= z >> 31;
        z *= 0xBF58476D1CE4E5B9ull;
        z ^= z >> 29;
        p[i] = double(int64_t(z >> 11) - (1ll << 52)) / double(1ll << 52);
    }
}

int main(int argc, char** argv) {
    const int layout = argc > 1 ? std::atoi(argv[1]) : 0;  // 0 rows (contract last), 1 groups
    const int reps = argc > 2 ? std::atoi(argv[2]) : 30;
    const int hog_smem = argc > 3 ? std::atoi(argv[3]) : 48 * 1024;
    const int hog_ctas = argc > 4 ? std::atoi(argv[4]) : 148 * 2;
    const char* mode = argc > 5 ? argv[5] : "hog";
    const uint32_t R = 16, Rp = 16;
    cpdb::TtmArgs a{};
    if (layout == 0) {
        a.outer = 128ull * 16 * 128;
        a.K = 128;
        a.inner = 1;
    } else {
        a.outer = 1;
        a.K = 128;
        a.inner = 16ull * 128 * 16;
    }
    const uint64_t nx = a.outer * a.K * a.inner, ny = a.outer * R * a.inner;
    double *x, *y, *y0, *qp, *sink;
    CK(cudaMalloc(&x, nx * 8));
    CK(cudaMalloc(&y, ny * 8));
    CK(cudaMalloc(&y0, ny * 8));
    CK(cudaMalloc(&qp, uint64_t(cpdb::ttm_kpad(a.K)) * Rp * 8));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(sink, 0, 8));
    fill<<<1184, 256>>>(x, nx, 1);
    fill<<<1184, 256>>>(qp, uint64_t(cpdb::ttm_kpad(a.K)) * Rp, 2);
    CK(cudaDeviceSynchronize());
    a.x = x;
    a.qp = qp;
    a.R = R;
    a.Rp = Rp;
    a.no_pdl = 1;
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    a.y = y0;
    CK(cpdb::launch_ttm(a, s1, 148));
    CK(cudaDeviceSynchronize());
    CK(cudaFuncSetAttribute(hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, hog_smem));
    std::vector<double> h0(ny), h(ny);
    CK(cudaMemcpy(h0.data(), y0, ny * 8, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int rep = 0; rep < reps; ++rep) {
        CK(cudaMemset(y, 0xff, ny * 8));
        CK(cudaDeviceSynchronize());
        a.y = y;
        if (std::strcmp(mode, "cluster") == 0) {
            cudaLaunchConfig_t c{};
            c.gridDim = dim3(hog_ctas, 1, 1);
            c.blockDim = dim3(256, 1, 1);
            c.dynamicSmemBytes = 4096 * 8;
            c.stream = s2;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 8;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            c.attrs = at;
            c.numAttrs = 1;
            CK(cudaLaunchKernelEx(&c, cluster_hog_kernel, 20000 + rep * 100,
                                  reinterpret_cast<unsigned long long*>(sink),
                                  std::getenv("HOG_NO_DSMEM") ? 0 : std::getenv("HOG_WRITE") ? 2 : 1));
            CK(cpdb::launch_ttm(a, s1, 148));
        } else if (std::strcmp(mode, "hog") == 0) {
            hog_kernel<<<hog_ctas, 256, hog_smem, s2>>>(20000 + rep * 100, sink);
            CK(cpdb::launch_ttm(a, s1, 148));
        } else if (std::strcmp(mode, "self") == 0) {
            // two TTM grids at once (different outputs)
            a.y = y0 == y ? y : y;
            CK(cpdb::launch_ttm(a, s1, 148));
            cpdb::TtmArgs b = a;
            b.y = sink == nullptr ? y : y;  // same output: identical values
            CK(cpdb::launch_ttm_tma(b, s2, 148));
        } else {
            CK(cpdb::launch_ttm(a, s1, 148));
        }
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h.data(), y, ny * 8, cudaMemcpyDeviceToHost));
        uint64_t nd = 0, first = 0;
        for (uint64_t i = 0; i < ny; ++i)
            if (std::memcmp(&h[i], &h0[i], 8) != 0) {
                if (!nd) first = i;
                ++nd;
            }
        if (nd) {
            ++bad;
            if (bad <= 5)
                std::printf("rep %d: %llu of %llu differ, first %llu (%g vs %g)\n", rep,
                            (unsigned long long)nd, (unsigned long long)ny,
                            (unsigned long long)first, h[first], h0[first]);
        }
    }
    unsigned long long hb = 0;
    CK(cudaMemcpy(&hb, sink, 8, cudaMemcpyDeviceToHost));
    std::printf("layout %d mode %s hog_smem %d ctas %d: %d of %d reps differ (hog bad words %llu)\n",
                layout, mode, hog_smem, hog_ctas, bad, reps, hb);
    return 0;
}
