// Drop-in for /root/reference/proj/include/cpd/linalg.hpp on libcpdb.
//
//   thin_qr                      linalg.hpp:39-99   device Householder (same
//                                                   reflector signs, backward
//                                                   Q accumulation, diag R >= 0)
//   solve_rows_lower_triangular  linalg.hpp:192-216 device row solves, same
//                                                   1e-14 relative singularity test
//   normalize_columns            linalg.hpp:225-242 device, the reference's exact
//                                                   summation order
//   solve_spd                    linalg.hpp:132-187 device Cholesky (+ the
//                                                   1e-12 trace/n ridge retry) and
//                                                   row solves (CP-ALS normal equations)
#pragma once

#include <cstddef>
#include <stdexcept>
#include <utility>
#include <vector>

#include "cpd/abi.hpp"
#include "cpd/tensor.hpp"

namespace cpd {

struct QrPair {
    Matrix q;  // m x n, orthonormal columns
    Matrix r;  // n x n, upper triangular, diag >= 0
};

inline QrPair thin_qr(const Matrix& a) {
    if (a.rows() < a.cols()) throw std::invalid_argument("thin_qr: requires rows >= cols");
    QrPair out{Matrix(a.rows(), a.cols()), Matrix(a.cols(), a.cols())};
    abi::check(cpdb_thin_qr(abi::ctx(), a.data(), a.rows(), a.cols(), out.q.data(),
                            out.r.data()));
    return out;
}

// Row-wise back substitution: X with X L^T = RHS (the reference passes R0^T as
// L, solvers.hpp:272).  Throws singular_triangular_error naming the column.
inline Matrix solve_rows_lower_triangular(const Matrix& l, const Matrix& rhs) {
    const std::size_t n = l.rows();
    if (l.cols() != n)
        throw std::invalid_argument("solve_rows_lower_triangular: L must be square");
    if (rhs.cols() != n)
        throw std::invalid_argument("solve_rows_lower_triangular: RHS columns must match L");
    Matrix x(rhs.rows(), n);
    int64_t bad = -1;
    const int st = cpdb_solve_rows_lower(abi::ctx(), l.data(), n, rhs.data(), rhs.rows(),
                                         x.data(), &bad);
    if (st == CPDB_SINGULAR_TRIANGULAR && bad >= 0)
        throw singular_triangular_error(std::size_t(bad), l(std::size_t(bad), std::size_t(bad)));
    abi::check(st);
    return x;
}

struct NormalizedColumns {
    Matrix matrix;
    std::vector<double> weights;
};

inline NormalizedColumns normalize_columns(const Matrix& a) {
    NormalizedColumns out{Matrix(a.rows(), a.cols()), std::vector<double>(a.cols(), 0.0)};
    abi::check(cpdb_normalize_columns(abi::ctx(), a.data(), a.rows(), a.cols(),
                                      out.matrix.data(), out.weights.data()));
    return out;
}

struct SpdSolveResult {
    Matrix x;
    bool regularized = false;
};

// X G = RHS with G symmetric positive (semi)definite (linalg.hpp:132-187):
// symmetric check, Cholesky, one ridge retry, singular_system_error.
inline SpdSolveResult solve_spd(const Matrix& g, const Matrix& rhs) {
    SpdSolveResult out{Matrix(rhs.rows(), rhs.cols()), false};
    int32_t reg = 0;
    abi::check(cpdb_solve_spd(abi::ctx(), g.data(), g.rows(), g.cols(), rhs.data(), rhs.rows(),
                              rhs.cols(), out.x.data(), &reg));
    out.regularized = reg != 0;
    return out;
}

}  // namespace cpd
