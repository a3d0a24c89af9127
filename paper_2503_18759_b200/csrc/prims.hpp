// Launchers of the single-primitive kernels (prims.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cpdb {

struct Dims8 {
    uint64_t v[8];
    uint32_t order;
};

cudaError_t transpose_dev(const double* in, uint64_t rows, uint64_t cols, double* out,
                          cudaStream_t s);
cudaError_t unfold_dev(const double* t, const Dims8& d, uint32_t mode, double* out,
                       cudaStream_t s);
cudaError_t khatri_rao_dev(const double* const* mats_dev, const Dims8& rows, uint64_t cols,
                           double* out, cudaStream_t s);
cudaError_t solve_rows_lower_dev(const double* l, uint32_t n, double* x, uint64_t rows,
                                 int* status, cudaStream_t s);
cudaError_t extrapolate_dev(const double* now, const double* prev, uint64_t n, double beta,
                            double alpha, double* out, cudaStream_t s);
// out4 = {<V, A_hat R0^T>, ||K||^2, fitness, raw radicand}
cudaError_t fitness_dev(double nx2, const double* v, const double* ah, uint64_t rows,
                        const double* r0, const double* rn, const double* lam, uint32_t r,
                        double* out4, cudaStream_t s);

// Order-free integer hash of n doubles added into *out (diagnostic).
cudaError_t fingerprint(const double* x, uint64_t n, unsigned long long* out, cudaStream_t s);

}  // namespace cpdb
