// Device versions of the reference's dense primitives that the drop-in C++
// API exposes one by one (tensor.hpp / linalg.hpp / solvers.hpp / kruskal.hpp).
// The solver does not call these -- it has fused equivalents -- but the
// reference tests call the primitives directly, so each has a device kernel.
#include <algorithm>

#include "device.cuh"
#include "cpdt.hpp"
#include "prims.hpp"
#include "runtime.hpp"

namespace cpdb {
namespace {

__global__ void transpose_kernel(const double* in, uint64_t rows, uint64_t cols, double* out) {
    const uint64_t n = rows * cols;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = e / cols, j = e % cols;
        out[j * rows + i] = in[e];
    }
}

// unfold (tensor.hpp:217-250): element lin -> (row = idx[mode], col with the
// earliest other mode fastest)
__global__ void unfold_kernel(const double* t, Dims8 d, uint32_t mode, double* out) {
    uint64_t total = 1;
    for (uint32_t k = 0; k < d.order; ++k) total *= d.v[k];
    const uint64_t cols = total / d.v[mode];
    for (uint64_t lin = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; lin < total;
         lin += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t rem = lin, idx[8];
        for (int k = int(d.order) - 1; k >= 0; --k) {
            idx[k] = rem % d.v[k];
            rem /= d.v[k];
        }
        uint64_t col = 0, w = 1;
        for (uint32_t k = 0; k < d.order; ++k)
            if (k != mode) {
                col += idx[k] * w;
                w *= d.v[k];
            }
        out[idx[mode] * cols + col] = t[lin];
    }
}

// khatri_rao (tensor.hpp:343-368): row index digits with the LAST list
// element fastest; products formed left to right like the reference fold.
__global__ void khatri_rao_kernel(const double* const* mats, Dims8 rows, uint64_t cols,
                                  double* out) {
    uint64_t total = 1;
    for (uint32_t k = 0; k < rows.order; ++k) total *= rows.v[k];
    const uint64_t n = total * cols;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = e / cols, j = e % cols;
        uint64_t rem = row, idx[8];
        for (int k = int(rows.order) - 1; k >= 0; --k) {
            idx[k] = rem % rows.v[k];
            rem /= rows.v[k];
        }
        double p = mats[0][idx[0] * cols + j];
        for (uint32_t k = 1; k < rows.order; ++k) p = __dmul_rn(p, mats[k][idx[k] * cols + j]);
        out[e] = p;
    }
}

// solve_rows_lower_triangular (linalg.hpp:192-216): one thread per row,
// back substitution; status = column+1 of the first singular diagonal.
__global__ void solve_rows_lower_kernel(const double* l, uint32_t n, double* x, uint64_t rows,
                                        int* status) {
    __shared__ int bad;
    if (threadIdx.x == 0) {
        double mx = 0.0;
        for (uint32_t i = 0; i < n; ++i) mx = fmax(mx, fabs(l[i * n + i]));
        bad = 0;
        for (uint32_t i = 0; i < n; ++i)
            if (fabs(l[i * n + i]) <= 1e-14 * mx) {
                bad = int(i) + 1;
                break;
            }
        if (blockIdx.x == 0) *status = bad;
    }
    __syncthreads();
    if (bad) return;
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
         r += uint64_t(gridDim.x) * blockDim.x) {
        double* xr = x + r * n;
        for (int c = int(n) - 1; c >= 0; --c) {
            double s = xr[c];
            for (uint32_t j = c + 1; j < n; ++j) s -= xr[j] * l[j * n + c];
            xr[c] = s / l[c * n + c];
        }
    }
}

__global__ void extrapolate_kernel(const double* now, const double* prev, uint64_t n, double beta,
                                   double alpha, double* out) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x)
        out[e] = beta == 0.0 ? now[e] : now[e] + beta * (now[e] - alpha * prev[e]);
}

// fitness_fast_qr (kruskal.hpp:109-128), one block
__global__ void __launch_bounds__(256)
fitness_kernel(double nx2, const double* v, const double* ah, uint64_t rows, const double* r0,
               const double* rn, const double* lam, uint32_t r, double* out) {
    __shared__ double red[8];
    double s = 0.0;
    for (uint64_t e = threadIdx.x; e < rows * r; e += 256) {
        const uint64_t i = e / r, j = e % r;
        double m = 0.0;
        for (uint32_t p = 0; p < r; ++p) m = fma(ah[i * r + p], r0[j * r + p], m);
        s = fma(v[e], m, s);
    }
    double k = 0.0;
    for (uint32_t e = threadIdx.x; e < r * r; e += 256) {
        const uint32_t i = e / r, j = e % r;
        double g0 = 0.0, gn = 0.0;
        for (uint32_t p = 0; p < r; ++p) {
            g0 = fma(r0[p * r + i], r0[p * r + j], g0);
            gn = fma(rn[p * r + i], rn[p * r + j], gn);
        }
        k += g0 * lam[i] * gn * lam[j];
    }
    for (int pass = 0; pass < 2; ++pass) {
        double v0 = warp_sum(pass == 0 ? s : k);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v0;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += red[w];
            out[pass] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double raw = nx2 - 2.0 * out[0] + out[1];
        const double rad = raw < 0.0 ? 0.0 : raw;
        out[2] = 1.0 - sqrt(rad) / sqrt(nx2);
        out[3] = raw;
    }
}

unsigned grid_for(uint64_t n) {
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 8192)));
}

}  // namespace

cudaError_t transpose_dev(const double* in, uint64_t rows, uint64_t cols, double* out,
                          cudaStream_t s) {
    transpose_kernel<<<grid_for(rows * cols), 256, 0, s>>>(in, rows, cols, out);
    return cudaGetLastError();
}

cudaError_t unfold_dev(const double* t, const Dims8& d, uint32_t mode, double* out,
                       cudaStream_t s) {
    uint64_t total = 1;
    for (uint32_t k = 0; k < d.order; ++k) total *= d.v[k];
    unfold_kernel<<<grid_for(total), 256, 0, s>>>(t, d, mode, out);
    return cudaGetLastError();
}

cudaError_t khatri_rao_dev(const double* const* mats_dev, const Dims8& rows, uint64_t cols,
                           double* out, cudaStream_t s) {
    uint64_t total = cols;
    for (uint32_t k = 0; k < rows.order; ++k) total *= rows.v[k];
    khatri_rao_kernel<<<grid_for(total), 256, 0, s>>>(mats_dev, rows, cols, out);
    return cudaGetLastError();
}

cudaError_t solve_rows_lower_dev(const double* l, uint32_t n, double* x, uint64_t rows,
                                 int* status, cudaStream_t s) {
    solve_rows_lower_kernel<<<grid_for(rows), 256, 0, s>>>(l, n, x, rows, status);
    return cudaGetLastError();
}

cudaError_t extrapolate_dev(const double* now, const double* prev, uint64_t n, double beta,
                            double alpha, double* out, cudaStream_t s) {
    extrapolate_kernel<<<grid_for(n), 256, 0, s>>>(now, prev, n, beta, alpha, out);
    return cudaGetLastError();
}

cudaError_t fitness_dev(double nx2, const double* v, const double* ah, uint64_t rows,
                        const double* r0, const double* rn, const double* lam, uint32_t r,
                        double* out4, cudaStream_t s) {
    fitness_kernel<<<1, 256, 0, s>>>(nx2, v, ah, rows, r0, rn, lam, r, out4);
    return cudaGetLastError();
}

namespace {
__global__ void nonfinite_kernel(const double* x, uint64_t n, unsigned long long* out) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        c += isfinite(x[i]) ? 0ull : 1ull;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);  // integer: order-free
}
}  // namespace

uint64_t count_nonfinite(const double* x, uint64_t n, cudaStream_t s) {
    unsigned long long* d = nullptr;
    unsigned long long h = 0;
    CPDB_CK(cudaMallocAsync(&d, sizeof h, s));
    CPDB_CK(cudaMemsetAsync(d, 0, sizeof h, s));
    nonfinite_kernel<<<1184, 256, 0, s>>>(x, n, d);
    CPDB_CK(cudaGetLastError());
    CPDB_CK(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s));
    CPDB_CK(cudaFreeAsync(d, s));
    CPDB_CK(cudaStreamSynchronize(s));
    return h;
}

}  // namespace cpdb

namespace cpdb {
namespace {
// Order-free integer hash of a buffer (diagnostic, CPDB_FINGERPRINT): every
// word is mixed with its index, the mixes are summed mod 2^64.
__global__ void fingerprint_kernel(const unsigned long long* x, uint64_t n,
                                   unsigned long long* out) {
    unsigned long long h = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        unsigned long long v = x[i] ^ (i * 0x9E3779B97F4A7C15ull);
        v ^= v >> 31;
        v *= 0xBF58476D1CE4E5B9ull;
        v ^= v >> 29;
        h += v;
    }
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}
}  // namespace

cudaError_t fingerprint(const double* x, uint64_t n, unsigned long long* out, cudaStream_t s) {
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 148));
    fingerprint_kernel<<<std::max(grid, 1u), 256, 0, s>>>(
        reinterpret_cast<const unsigned long long*>(x), n, out);
    return cudaGetLastError();
}

}  // namespace cpdb
