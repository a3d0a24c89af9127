// Drop-in for /root/reference/proj/include/cpd/tensor.hpp on libcpdb.
//
// Value types (Shape, Matrix, DenseTensor) keep the reference's public API and
// row-major layout (last index fastest, tensor.hpp:42-47) so that the
// reference's callers and tests compile unchanged.  The contractions on the
// CP-ALS-QR path -- ttm (tensor.hpp:288-315), multi_ttm, unfold
// (tensor.hpp:217-250), khatri_rao (tensor.hpp:343-368) and inner
// (tensor.hpp:394-399) -- run on the B200 through the C ABI.  Small dense
// helpers that the reference uses for bookkeeping and checks (matmul of
// R-sized matrices, transpose, gram, dot, hadamard, kronecker, fold) are plain
// host loops here as they are there; none of them is on the sweep's hot path.
//
// MTTKRP (tensor.hpp:415-518), the kernel of the CP-ALS normal-equation
// solver, also runs on the device: mttkrp /
// mttkrp_materialized below go through cpdb_mttkrp.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "cpd/abi.hpp"

namespace cpd {

// ------------------------------------------------------------------ Shape
class Shape {
public:
    Shape() = default;
    explicit Shape(std::vector<std::size_t> extents) : dims_(std::move(extents)) {
        if (dims_.empty()) throw std::invalid_argument("Shape: order must be >= 1");
        count_ = 1;
        for (const std::size_t e : dims_) {
            if (e == 0) throw std::invalid_argument("Shape: every extent must be >= 1");
            if (count_ > std::numeric_limits<std::size_t>::max() / e)
                throw std::invalid_argument("Shape: element count overflows");
            count_ *= e;
        }
    }
    Shape(std::initializer_list<std::size_t> extents)
        : Shape(std::vector<std::size_t>(extents.begin(), extents.end())) {}

    std::size_t order() const { return dims_.size(); }
    std::size_t extent(std::size_t mode) const { return dims_.at(mode); }
    const std::vector<std::size_t>& dims() const { return dims_; }
    std::size_t element_count() const { return count_; }

    // Horner form of the row-major offset.
    std::size_t linear_index(std::span<const std::size_t> idx) const {
        std::size_t off = 0;
        for (std::size_t k = 0; k < dims_.size(); ++k) off = off * dims_[k] + idx[k];
        return off;
    }

    friend bool operator==(const Shape& a, const Shape& b) { return a.dims_ == b.dims_; }
    friend bool operator!=(const Shape& a, const Shape& b) { return !(a == b); }

private:
    std::vector<std::size_t> dims_;
    std::size_t count_ = 0;
};

// ------------------------------------------------------------------ Matrix
class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols) : m_(rows), n_(cols) {
        if (m_ == 0 || n_ == 0) throw std::invalid_argument("Matrix: zero dimension");
        v_.assign(m_ * n_, 0.0);
    }
    Matrix(std::size_t rows, std::size_t cols, std::vector<double> values)
        : m_(rows), n_(cols), v_(std::move(values)) {
        if (m_ == 0 || n_ == 0) throw std::invalid_argument("Matrix: zero dimension");
        if (v_.size() != m_ * n_)
            throw std::invalid_argument("Matrix: value count does not match rows*cols");
    }
    static Matrix identity(std::size_t n) {
        Matrix e(n, n);
        for (std::size_t i = 0; i < n; ++i) e.v_[i * n + i] = 1.0;
        return e;
    }

    std::size_t rows() const { return m_; }
    std::size_t cols() const { return n_; }
    std::size_t size() const { return v_.size(); }
    double& operator()(std::size_t i, std::size_t j) { return v_[i * n_ + j]; }
    double operator()(std::size_t i, std::size_t j) const { return v_[i * n_ + j]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    const std::vector<double>& values() const { return v_; }

private:
    std::size_t m_ = 0, n_ = 0;
    std::vector<double> v_;
};

// ------------------------------------------------------------------ DenseTensor
class DenseTensor {
public:
    DenseTensor() = default;
    explicit DenseTensor(Shape s) : shape_(std::move(s)), v_(shape_.element_count(), 0.0) {}
    DenseTensor(Shape s, std::vector<double> values) : shape_(std::move(s)), v_(std::move(values)) {
        if (v_.size() != shape_.element_count())
            throw std::invalid_argument("DenseTensor: value count does not match shape");
    }

    const Shape& shape() const { return shape_; }
    std::size_t order() const { return shape_.order(); }
    std::size_t size() const { return v_.size(); }
    double at(std::span<const std::size_t> idx) const { return v_[shape_.linear_index(idx)]; }
    double& at(std::span<const std::size_t> idx) { return v_[shape_.linear_index(idx)]; }
    double at(std::initializer_list<std::size_t> idx) const {
        return v_[shape_.linear_index(std::span<const std::size_t>(idx.begin(), idx.size()))];
    }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    const std::vector<double>& values() const { return v_; }
    std::vector<double>& values() { return v_; }

private:
    Shape shape_;
    std::vector<double> v_;
};

// ------------------------------------------------------------------ small host helpers
inline Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols() != b.rows()) throw std::invalid_argument("matmul: inner dimensions differ");
    Matrix c(a.rows(), b.cols());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t k = 0; k < a.cols(); ++k) {
            const double s = a(i, k);
            for (std::size_t j = 0; j < b.cols(); ++j) c(i, j) += s * b(k, j);
        }
    return c;
}

inline Matrix transpose(const Matrix& a) {
    Matrix t(a.cols(), a.rows());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) t(j, i) = a(i, j);
    return t;
}

// A^T A
inline Matrix gram(const Matrix& a) {
    Matrix g(a.cols(), a.cols());
    for (std::size_t r = 0; r < a.rows(); ++r)
        for (std::size_t i = 0; i < a.cols(); ++i)
            for (std::size_t j = 0; j < a.cols(); ++j) g(i, j) += a(r, i) * a(r, j);
    return g;
}

inline double dot(const Matrix& a, const Matrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols())
        throw std::invalid_argument("dot: dimension mismatch");
    double s = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a.data()[i] * b.data()[i];
    return s;
}

inline Matrix hadamard(const Matrix& a, const Matrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols())
        throw std::invalid_argument("hadamard: dimension mismatch");
    Matrix c(a.rows(), a.cols());
    for (std::size_t i = 0; i < a.size(); ++i) c.data()[i] = a.data()[i] * b.data()[i];
    return c;
}

inline Matrix kronecker(const Matrix& a, const Matrix& b) {
    Matrix c(a.rows() * b.rows(), a.cols() * b.cols());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j)
            for (std::size_t p = 0; p < b.rows(); ++p)
                for (std::size_t q = 0; q < b.cols(); ++q)
                    c(i * b.rows() + p, j * b.cols() + q) = a(i, j) * b(p, q);
    return c;
}

inline double frobenius_norm(const Matrix& m) {
    double s = 0.0;
    for (const double v : m.values()) s += v * v;
    return std::sqrt(s);
}

// ------------------------------------------------------------------ device-backed ops
// Mode-n unfolding: rows = mode n, columns ordered with the EARLIEST other
// mode fastest (tensor.hpp:213-233).  Device permutation kernel.
inline Matrix unfold(const DenseTensor& t, std::size_t mode) {
    if (mode >= t.order()) throw std::invalid_argument("unfold: mode out of range");
    const std::size_t rows = t.shape().extent(mode);
    Matrix out(rows, t.size() / rows);
    const auto d = abi::u64(t.shape().dims());
    abi::check(cpdb_unfold(abi::ctx(), t.data(), d.data(), uint32_t(d.size()),
                           uint32_t(mode), out.data()));
    return out;
}

// Inverse of unfold (host index walk; only used by callers outside the sweep).
inline DenseTensor fold(const Matrix& m, std::size_t mode, const Shape& shape) {
    const std::size_t order = shape.order();
    if (mode >= order) throw std::invalid_argument("fold: mode out of range");
    if (m.rows() != shape.extent(mode) || m.rows() * m.cols() != shape.element_count())
        throw std::invalid_argument("fold: matrix dimensions do not match shape");
    DenseTensor t(shape);
    std::vector<std::size_t> idx(order, 0);
    for (std::size_t lin = 0; lin < t.size(); ++lin) {
        // column index: other modes, earliest fastest
        std::size_t col = 0, stride = 1;
        for (std::size_t k = 0; k < order; ++k) {
            if (k == mode) continue;
            col += idx[k] * stride;
            stride *= shape.extent(k);
        }
        t.values()[lin] = m(idx[mode], col);
        for (std::size_t k = order; k-- > 0;) {  // row-major increment
            if (++idx[k] < shape.extent(k)) break;
            idx[k] = 0;
        }
    }
    return t;
}

// Y = T x_mode B, B is (new extent) x I_mode; tensor.hpp:288-315.
inline DenseTensor ttm(const DenseTensor& t, const Matrix& b, std::size_t mode) {
    if (mode >= t.order()) throw std::invalid_argument("ttm: mode out of range");
    if (b.cols() != t.shape().extent(mode))
        throw std::invalid_argument("ttm: matrix columns do not match mode extent");
    std::vector<std::size_t> od = t.shape().dims();
    od[mode] = b.rows();
    DenseTensor y{Shape(od)};
    const auto d = abi::u64(t.shape().dims());
    abi::check(cpdb_ttm(abi::ctx(), t.data(), d.data(), uint32_t(d.size()), b.data(), b.rows(),
                        uint32_t(mode), y.data()));
    return y;
}

struct ModeMatrix {
    std::size_t mode;
    const Matrix* matrix;
};

inline DenseTensor multi_ttm(const DenseTensor& t, std::span<const ModeMatrix> pairs) {
    std::vector<bool> used(t.order(), false);
    for (const ModeMatrix& p : pairs) {
        if (p.mode >= t.order()) throw std::invalid_argument("multi_ttm: mode out of range");
        if (used[p.mode]) throw std::invalid_argument("multi_ttm: duplicate mode");
        used[p.mode] = true;
    }
    DenseTensor y = t;
    for (const ModeMatrix& p : pairs) y = ttm(y, *p.matrix, p.mode);
    return y;
}

inline DenseTensor multi_ttm(const DenseTensor& t, std::initializer_list<ModeMatrix> pairs) {
    return multi_ttm(t, std::span<const ModeMatrix>(pairs.begin(), pairs.size()));
}

// Column-wise Kronecker product; the LAST matrix's row index varies fastest
// (tensor.hpp:343-368).  Device kernel.
inline Matrix khatri_rao(std::span<const Matrix* const> mats) {
    if (mats.empty()) throw std::invalid_argument("khatri_rao: empty list");
    const std::size_t r = mats[0]->cols();
    std::vector<const double*> ptrs;
    std::vector<uint64_t> rows;
    std::size_t prod = 1;
    for (const Matrix* m : mats) {
        if (m->cols() != r) throw std::invalid_argument("khatri_rao: mismatched column counts");
        ptrs.push_back(m->data());
        rows.push_back(m->rows());
        prod *= m->rows();
    }
    Matrix out(prod, r);
    abi::check(cpdb_khatri_rao(abi::ctx(), ptrs.data(), rows.data(), uint32_t(ptrs.size()), r,
                               out.data()));
    return out;
}

inline Matrix khatri_rao(std::initializer_list<const Matrix*> mats) {
    return khatri_rao(std::span<const Matrix* const>(mats.begin(), mats.size()));
}

// Matricized tensor times Khatri-Rao product (tensor.hpp:453-488): one
// device TTM of X with the factor of another mode plus a Khatri-Rao
// contraction of the rest; factors[mode] is not read (tensor.hpp:415-431).
inline Matrix mttkrp(const DenseTensor& t, std::span<const Matrix* const> factors,
                     std::size_t mode) {
    const std::size_t order = t.order();
    if (mode >= order) throw std::invalid_argument("mttkrp: mode out of range");
    if (factors.size() != order) throw std::invalid_argument("mttkrp: need one factor per mode");
    std::vector<const double*> ptrs(order, nullptr);
    std::vector<uint64_t> rows(order, 0), cols(order, 0);
    std::size_t rank = 0;
    for (std::size_t k = 0; k < order; ++k) {
        if (k == mode || factors[k] == nullptr) continue;
        ptrs[k] = factors[k]->data();
        rows[k] = factors[k]->rows();
        cols[k] = factors[k]->cols();
        if (rank == 0) rank = factors[k]->cols();
    }
    Matrix out(t.shape().extent(mode), rank == 0 ? 1 : rank);
    const std::vector<uint64_t> dims = abi::u64(t.shape().dims());
    abi::check(cpdb_mttkrp(abi::ctx(), t.data(), dims.data(), uint32_t(order), ptrs.data(),
                           rows.data(), cols.data(), uint32_t(mode), out.data()));
    return out;
}

// The reference keeps a materialising variant as an independent check of the
// streaming path (tensor.hpp:494-518); both name the same product, which the
// device computes one way.  Same argument checks.
inline Matrix mttkrp_materialized(const DenseTensor& t, std::span<const Matrix* const> factors,
                                  std::size_t mode) {
    const std::size_t order = t.order();
    if (mode >= order) throw std::invalid_argument("mttkrp: mode out of range");
    if (factors.size() != order) throw std::invalid_argument("mttkrp: need one factor per mode");
    for (std::size_t k = 0; k < order; ++k)
        if (k != mode && factors[k] == nullptr)
            throw std::invalid_argument("mttkrp: missing factor");
    return mttkrp(t, factors, mode);
}

// <A, B> (tensor.hpp:394-399), deterministic device reduction.
inline double inner(const DenseTensor& a, const DenseTensor& b) {
    if (a.shape() != b.shape()) throw std::invalid_argument("inner: shape mismatch");
    double s = 0.0;
    abi::check(cpdb_inner(abi::ctx(), a.data(), b.data(), a.size(), &s));
    return s;
}

inline double frobenius_norm(const DenseTensor& t) { return std::sqrt(inner(t, t)); }

}  // namespace cpd
