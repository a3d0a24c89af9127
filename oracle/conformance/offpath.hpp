// TEST INFRASTRUCTURE ONLY (force-included into the conformance binaries by
// oracle/conformance/Makefile; never part of libcpdb or include/cpd).
//
// The reference's unit-test files for the hot path (linalg_test, tensor_test,
// kruskal_test, solver_test) also exercise the CP-ALS normal-equation solver,
// which this library does not ship.  So that those
// files compile UNCHANGED against the drop-in headers, this shim supplies the
// missing off-path entry points with straightforward host implementations of
// the reference's documented algorithms:
//   solve_spd          linalg.hpp:114-171  Cholesky (+ one 1e-12 trace/n ridge retry)
//   mttkrp(_materialized) tensor.hpp:453-518  unfold(X, n) * KR(descending)
//                                            (unfold and Khatri-Rao on the device)
//   fitness_fast_als   kruskal.hpp:78-94
//   cp_als             solvers.hpp:149-208
// Test cases that reach these report on the shim, not on the product; the
// conformance summary (tools/conformance.py) lists them separately.
#pragma once

#include <algorithm>
#include <cmath>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cpd/kruskal.hpp"
#include "cpd/linalg.hpp"
#include "cpd/solvers.hpp"
#include "cpd/tensor.hpp"

namespace cpd {

struct SpdSolveResult {
    Matrix x;
    bool regularized = false;
};

namespace offpath {

inline std::optional<Matrix> chol_lower(const Matrix& g) {
    const std::size_t n = g.rows();
    Matrix l(n, n);
    for (std::size_t j = 0; j < n; ++j) {
        double d = g(j, j);
        for (std::size_t k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
        if (!(d > 0.0)) return std::nullopt;
        l(j, j) = std::sqrt(d);
        for (std::size_t i = j + 1; i < n; ++i) {
            double s = g(i, j);
            for (std::size_t k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
            l(i, j) = s / l(j, j);
        }
    }
    return l;
}

}  // namespace offpath

// X G = RHS with G symmetric positive (semi)definite.
inline SpdSolveResult solve_spd(const Matrix& g, const Matrix& rhs) {
    const std::size_t n = g.rows();
    if (g.cols() != n) throw std::invalid_argument("solve_spd: G must be square");
    if (rhs.cols() != n) throw std::invalid_argument("solve_spd: RHS columns must match G");
    double big = 0.0, asym = 0.0;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) {
            big = std::max(big, std::fabs(g(i, j)));
            asym = std::max(asym, std::fabs(g(i, j) - g(j, i)));
        }
    if (asym > 1e-10 * big) throw std::invalid_argument("solve_spd: G is not symmetric");
    SpdSolveResult out{rhs, false};
    std::optional<Matrix> l = offpath::chol_lower(g);
    if (!l) {
        double tr = 0.0;
        for (std::size_t i = 0; i < n; ++i) tr += g(i, i);
        Matrix shifted = g;
        for (std::size_t i = 0; i < n; ++i) shifted(i, i) += 1e-12 * tr / double(n);
        l = offpath::chol_lower(shifted);
        out.regularized = true;
        if (!l) throw singular_system_error("solve_spd: factorization failed after ridge");
    }
    for (std::size_t r = 0; r < rhs.rows(); ++r) {
        double* x = out.x.data() + r * n;
        for (std::size_t c = 0; c < n; ++c) {  // W L^T = RHS (W = X L), forward
            double s = x[c];
            for (std::size_t j = 0; j < c; ++j) s -= x[j] * (*l)(c, j);
            x[c] = s / (*l)(c, c);
        }
        for (std::size_t c = n; c-- > 0;) {  // X L = W, backward
            double s = x[c];
            for (std::size_t j = c + 1; j < n; ++j) s -= x[j] * (*l)(j, c);
            x[c] = s / (*l)(c, c);
        }
    }
    return out;
}

inline Matrix mttkrp_materialized(const DenseTensor& t, std::span<const Matrix* const> factors,
                                  std::size_t mode) {
    const auto& dims = t.shape().dims();
    if (mode >= dims.size()) throw std::invalid_argument("mttkrp: mode out of range");
    if (factors.size() != dims.size())
        throw std::invalid_argument("mttkrp: need one factor per mode");
    std::size_t rank = 0;
    for (std::size_t k = 0; k < dims.size(); ++k) {
        if (k == mode) continue;
        if (factors[k] == nullptr) throw std::invalid_argument("mttkrp: missing factor");
        if (rank == 0) rank = factors[k]->cols();
        if (factors[k]->cols() != rank) throw std::invalid_argument("mttkrp: mismatched ranks");
        if (factors[k]->rows() != dims[k])
            throw std::invalid_argument("mttkrp: factor rows do not match mode extent");
    }
    if (rank == 0) throw std::invalid_argument("mttkrp: order must be >= 2");
    std::vector<const Matrix*> desc;
    for (std::size_t k = dims.size(); k-- > 0;)
        if (k != mode) desc.push_back(factors[k]);
    return matmul(unfold(t, mode), khatri_rao(std::span<const Matrix* const>(desc)));
}

inline Matrix mttkrp(const DenseTensor& t, std::span<const Matrix* const> factors,
                     std::size_t mode) {
    return mttkrp_materialized(t, factors, mode);
}
inline Matrix mttkrp(const DenseTensor& t, const std::vector<const Matrix*>& factors,
                     std::size_t mode) {
    return mttkrp_materialized(t, std::span<const Matrix* const>(factors), mode);
}
inline Matrix mttkrp_materialized(const DenseTensor& t, const std::vector<const Matrix*>& factors,
                                  std::size_t mode) {
    return mttkrp_materialized(t, std::span<const Matrix* const>(factors), mode);
}

inline FitnessResult fitness_fast_als(double norm_x_sq, const Matrix& m_last,
                                      const Matrix& a_hat_last, const Matrix& gamma_last,
                                      const std::vector<double>& lambda, const Matrix& s_last) {
    if (!(norm_x_sq > 0.0)) throw std::invalid_argument("fitness_fast_als: zero-norm tensor");
    const double xk = dot(m_last, a_hat_last);
    const std::size_t r = lambda.size();
    if (gamma_last.rows() != r || s_last.rows() != r)
        throw std::invalid_argument("fitness_fast_als: dimension mismatch");
    double kk = 0.0;
    for (std::size_t i = 0; i < r; ++i)
        for (std::size_t j = 0; j < r; ++j)
            kk += gamma_last(i, j) * lambda[i] * s_last(i, j) * lambda[j];
    const double raw = norm_x_sq - 2.0 * xk + kk;
    return {1.0 - std::sqrt(raw < 0.0 ? 0.0 : raw) / std::sqrt(norm_x_sq), raw};
}

inline SolveResult cp_als(const DenseTensor& x, const SolverConfig& cfg,
                          const std::optional<KruskalModel>& init = {}) {
    cfg.validate();
    if (cfg.algorithm != Algorithm::als)
        throw std::invalid_argument("cp_als: config algorithm must be als");
    if (x.order() < 2) throw std::invalid_argument("cp_als: tensor order must be >= 2");
    const double nx2 = inner(x, x);
    if (nx2 == 0.0) throw std::invalid_argument("cp_als: zero-norm tensor");
    const std::size_t order = x.order(), rank = cfg.rank;
    std::vector<Matrix> fs = detail::initial_factors(x, cfg, init);
    std::vector<double> lambda = detail::initial_lambda(init, rank);
    std::vector<Matrix> grams;
    for (const Matrix& f : fs) grams.push_back(gram(f));
    const std::uint64_t per_mode = 2ull * x.size() * rank;
    std::uint64_t flops = 0;
    std::vector<std::size_t> ord(order);
    for (std::size_t k = 0; k < order; ++k) ord[k] = k;
    SolveResult res;
    for (std::size_t sweep = 1; sweep <= cfg.max_iterations; ++sweep) {
        Matrix m_last, a_last, g_last;
        bool reg = false;
        for (std::size_t n = 0; n < order; ++n) {
            Matrix g(rank, rank, std::vector<double>(rank * rank, 1.0));
            for (std::size_t k = 0; k < order; ++k)
                if (k != n) g = hadamard(g, grams[k]);
            std::vector<const Matrix*> ptrs;
            for (const Matrix& f : fs) ptrs.push_back(&f);
            Matrix m = mttkrp(x, ptrs, n);
            SpdSolveResult s = solve_spd(g, m);
            reg = reg || s.regularized;
            NormalizedColumns nc = normalize_columns(s.x);
            fs[n] = std::move(nc.matrix);
            lambda = std::move(nc.weights);
            grams[n] = gram(fs[n]);
            flops += per_mode;
            if (n + 1 == order) {
                m_last = std::move(m);
                a_last = std::move(s.x);
                g_last = std::move(g);
            }
        }
        const FitnessResult fit =
            fitness_fast_als(nx2, m_last, a_last, g_last, lambda, grams[order - 1]);
        res.trace.push_back({sweep, ord, fit.fitness, fit.raw_radicand, 0.0, 0, flops, 0.0, reg});
        if (fit.fitness >= cfg.fitness_threshold) break;
    }
    res.model = {std::move(lambda), std::move(fs)};
    return res;
}

}  // namespace cpd
