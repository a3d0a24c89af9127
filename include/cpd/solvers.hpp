// Drop-in for /root/reference/proj/include/cpd/solvers.hpp on libcpdb.
//
//   cp_als_qr   solvers.hpp:317-322  \  one device-resident run (cpdb_solve):
//   als_qr_bre  solvers.hpp:329-336  /  X, the intermediate cache, Q/R, the Q0
//                                       history and V never leave HBM; the host
//                                       sees one fitness scalar per sweep.
//   extrapolate_q0  solvers.hpp:75-86   device elementwise kernel
//   select_beta     solvers.hpp:92-101  the same scalar table (cpdb_select_beta)
// SolverConfig / TraceRow / SolveResult keep the reference's fields, including
// q0_observer (called with Q0 in the reference's Khatri-Rao row order).
//
//   cp_als      solvers.hpp:149-208  device-resident normal-equation ALS (the
//                                    paper's comparison solver): per mode
//                                    MTTKRP, Gamma, solve_spd, normalisation
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <optional>
#include <stdexcept>
#include <utility>
#include <vector>

#include "cpd/abi.hpp"
#include "cpd/dim_tree.hpp"
#include "cpd/factor_state.hpp"
#include "cpd/kruskal.hpp"
#include "cpd/linalg.hpp"
#include "cpd/rng.hpp"
#include "cpd/tensor.hpp"

namespace cpd {

enum class Algorithm { als, als_qr };

struct SolverConfig {
    std::size_t rank = 1;
    std::size_t max_iterations = 1;
    double fitness_threshold = 1.0;
    Algorithm algorithm = Algorithm::als;
    Strategy strategy = Strategy::naive;
    bool extrapolation_enabled = false;
    double alpha = 0.1;
    std::optional<double> beta_override;
    double activation_gap = 0.03;
    std::uint64_t seed = 0;
    std::function<void(std::size_t sweep, std::size_t mode, const Matrix& q0)> q0_observer;

    void validate() const {
        if (rank == 0) throw std::invalid_argument("SolverConfig: rank must be >= 1");
        if (max_iterations == 0)
            throw std::invalid_argument("SolverConfig: need at least one iteration");
        if (!(fitness_threshold >= 0.0 && fitness_threshold <= 1.0))
            throw std::invalid_argument("SolverConfig: fitness threshold must be in [0,1]");
        if (!std::isfinite(alpha) || !std::isfinite(activation_gap))
            throw std::invalid_argument("SolverConfig: alpha and activation gap must be finite");
    }
};

struct TraceRow {
    std::size_t iteration = 0;              // 1-based sweep
    std::vector<std::size_t> update_order;  // 0-based modes
    double fitness = 0.0;
    double raw_radicand = 0.0;
    double wall_seconds = 0.0;  // device clock since the solve began
    std::uint64_t root_ttm_count = 0;
    std::uint64_t flops = 0;
    double beta_used = 0.0;
    bool regularized = false;
};

struct SolveResult {
    KruskalModel model;
    std::vector<TraceRow> trace;
};

inline Matrix extrapolate_q0(const Matrix& q0_now, const Matrix& q0_prev, double beta,
                             double alpha) {
    if (q0_now.rows() != q0_prev.rows() || q0_now.cols() != q0_prev.cols())
        throw std::invalid_argument("extrapolate_q0: shape mismatch");
    if (beta == 0.0) return q0_now;  // bit-identical (solvers.hpp:79)
    Matrix out(q0_now.rows(), q0_now.cols());
    abi::check(cpdb_extrapolate_q0(abi::ctx(), q0_now.data(), q0_prev.data(), q0_now.rows(),
                                   q0_now.cols(), beta, alpha, out.data()));
    return out;
}

inline std::optional<double> select_beta(double fitness_prev, double fitness_now,
                                         double gap_threshold) {
    double beta = 0.0;
    if (cpdb_select_beta(fitness_prev, fitness_now, gap_threshold, &beta) == 0)
        return std::nullopt;
    return beta;
}

namespace detail {

// N(0,1) from Rng(seed), mode by mode, row-major, then unit columns
// (solvers.hpp:105-124).  The device run draws the same stream itself; this
// host copy serves callers that want the initial model.
inline std::vector<Matrix> initial_factors(const DenseTensor& x, const SolverConfig& cfg,
                                           const std::optional<KruskalModel>& init) {
    if (init) {
        if (init->order() != x.order() || init->rank() != cfg.rank)
            throw std::invalid_argument("solver: init model does not match tensor/config");
        for (std::size_t k = 0; k < x.order(); ++k)
            if (init->factors[k].rows() != x.shape().extent(k))
                throw std::invalid_argument("solver: init factor rows do not match tensor");
        return init->factors;
    }
    Rng rng(cfg.seed);
    std::vector<Matrix> fs;
    for (std::size_t k = 0; k < x.order(); ++k) {
        Matrix f(x.shape().extent(k), cfg.rank);
        for (std::size_t i = 0; i < f.size(); ++i) f.data()[i] = rng.normal();
        fs.push_back(normalize_columns(f).matrix);
    }
    return fs;
}

inline std::vector<double> initial_lambda(const std::optional<KruskalModel>& init,
                                          std::size_t rank) {
    return init ? init->lambda : std::vector<double>(rank, 1.0);
}

struct ObserverBridge {
    const SolverConfig* cfg;
    static void call(void* user, uint64_t sweep, uint32_t mode, const double* q0, uint64_t rows,
                     uint64_t cols) {
        const auto* self = static_cast<const ObserverBridge*>(user);
        const Matrix m(rows, cols, std::vector<double>(q0, q0 + rows * cols));
        self->cfg->q0_observer(std::size_t(sweep), std::size_t(mode), m);
    }
};

// One run on a context that already holds X (dims = its global extents):
// the device-resident loop of run_qr (solvers.hpp:215-309).
inline SolveResult run_on_context(cpdb_ctx* ctx, const std::vector<std::size_t>& dims,
                                  const SolverConfig& cfg, const std::vector<double>* init_f,
                                  const std::vector<double>* init_l, bool extrapolate) {
    cpdb_config c{};
    c.rank = cfg.rank;
    c.max_iterations = cfg.max_iterations;
    c.fitness_threshold = cfg.fitness_threshold;
    c.strategy = int32_t(cfg.strategy);
    c.extrapolate = extrapolate ? 1 : 0;
    c.alpha = cfg.alpha;
    c.has_beta_override = cfg.beta_override.has_value() ? 1 : 0;
    c.beta_override = cfg.beta_override.value_or(0.0);
    c.activation_gap = cfg.activation_gap;
    c.seed = cfg.seed;

    cpdb_state st{};
    std::vector<double> f_copy, l_copy;
    if (init_f) {
        f_copy = *init_f;
        l_copy = *init_l;
        st.factors = f_copy.data();
        st.lambda = l_copy.data();
    }
    std::size_t nfac = 0;
    for (const std::size_t d : dims) nfac += d * cfg.rank;
    std::vector<cpdb_trace_row> rows(cfg.max_iterations);
    std::vector<double> lam(cfg.rank), fac(nfac);
    uint64_t n = 0;
    ObserverBridge bridge{&cfg};
    abi::check(cpdb_solve(ctx, &c, init_f ? &st : nullptr, rows.data(), &n, lam.data(),
                          fac.data(), nullptr, nullptr,
                          cfg.q0_observer ? &ObserverBridge::call : nullptr, &bridge));

    SolveResult out;
    for (uint64_t i = 0; i < n; ++i) {
        const cpdb_trace_row& r = rows[i];
        TraceRow t;
        t.iteration = std::size_t(r.iteration);
        t.update_order.assign(r.update_order, r.update_order + r.order);
        t.fitness = r.fitness;
        t.raw_radicand = r.raw_radicand;
        t.wall_seconds = r.wall_seconds;
        t.root_ttm_count = r.root_ttm_count;
        t.flops = r.flops;
        t.beta_used = r.beta_used;
        t.regularized = r.regularized != 0;
        out.trace.push_back(std::move(t));
    }
    out.model.lambda = std::move(lam);
    std::size_t off = 0;
    for (const std::size_t d : dims) {
        out.model.factors.emplace_back(
            d, cfg.rank, std::vector<double>(fac.begin() + off, fac.begin() + off + d * cfg.rank));
        off += d * cfg.rank;
    }
    return out;
}

// One solve on a private device context (run_qr, solvers.hpp:215-309).
inline SolveResult run_qr(const DenseTensor& x, const SolverConfig& cfg,
                          const std::optional<KruskalModel>& init, bool extrapolate) {
    cfg.validate();
    const std::size_t order = x.order();
    if (order < 2) throw std::invalid_argument("cp_als_qr: tensor order must be >= 2");
    for (std::size_t k = 0; k < order; ++k)
        if (cfg.rank > x.shape().extent(k))
            throw std::invalid_argument(
                "cp_als_qr: rank must not exceed any mode extent (compact QR)");
    std::vector<double> init_f, init_l;
    if (init) {
        for (const Matrix& f : initial_factors(x, cfg, init))
            init_f.insert(init_f.end(), f.values().begin(), f.values().end());
        init_l = initial_lambda(init, cfg.rank);
    }
    cpdb_ctx* ctx = nullptr;
    const char* env = std::getenv("CPD_DEVICE");
    abi::check(cpdb_create(env ? std::atoi(env) : 0, &ctx));
    struct Guard {
        cpdb_ctx* c;
        ~Guard() { cpdb_destroy(c); }
    } guard{ctx};
    const std::vector<uint64_t> dims = abi::u64(x.shape().dims());
    abi::check(cpdb_tensor_set(ctx, x.data(), dims.data(), uint32_t(order)));
    return run_on_context(ctx, x.shape().dims(), cfg, init ? &init_f : nullptr,
                          init ? &init_l : nullptr, extrapolate);
}

}  // namespace detail

namespace detail {

// cp_als on a context whose tensor is already in HBM (cpdb_als_solve):
// shared by cp_als and the command line (which streams X straight to HBM)
inline SolveResult run_als_on_context(cpdb_ctx* ctx, const std::vector<std::size_t>& dims,
                                      const SolverConfig& cfg, const double* init_f,
                                      const double* init_l) {
    cpdb_config c{};
    c.rank = cfg.rank;
    c.max_iterations = cfg.max_iterations;
    c.fitness_threshold = cfg.fitness_threshold;
    c.alpha = cfg.alpha;
    c.activation_gap = cfg.activation_gap;
    c.seed = cfg.seed;
    std::size_t nfac = 0;
    for (const std::size_t d : dims) nfac += d * cfg.rank;
    std::vector<cpdb_trace_row> rows(cfg.max_iterations);
    std::vector<double> lam(cfg.rank), fac(nfac);
    uint64_t n = 0;
    abi::check(cpdb_als_solve(ctx, &c, init_l, init_f, rows.data(), &n, lam.data(), fac.data()));
    SolveResult out;
    for (uint64_t i = 0; i < n; ++i) {
        const cpdb_trace_row& r = rows[i];
        TraceRow t;
        t.iteration = std::size_t(r.iteration);
        t.update_order.assign(r.update_order, r.update_order + r.order);
        t.fitness = r.fitness;
        t.raw_radicand = r.raw_radicand;
        t.wall_seconds = r.wall_seconds;
        t.root_ttm_count = r.root_ttm_count;
        t.flops = r.flops;
        t.beta_used = r.beta_used;
        t.regularized = r.regularized != 0;
        out.trace.push_back(std::move(t));
    }
    out.model.lambda = std::move(lam);
    std::size_t off = 0;
    for (const std::size_t d : dims) {
        out.model.factors.emplace_back(
            d, cfg.rank, std::vector<double>(fac.begin() + off, fac.begin() + off + d * cfg.rank));
        off += d * cfg.rank;
    }
    return out;
}

}  // namespace detail

inline SolveResult cp_als(const DenseTensor& x, const SolverConfig& cfg,
                          const std::optional<KruskalModel>& init = {}) {
    cfg.validate();
    if (cfg.algorithm != Algorithm::als)
        throw std::invalid_argument("cp_als: config algorithm must be als");
    if (x.order() < 2) throw std::invalid_argument("cp_als: tensor order must be >= 2");
    std::vector<double> init_f, init_l;
    if (init) {
        for (const Matrix& f : detail::initial_factors(x, cfg, init))
            init_f.insert(init_f.end(), f.values().begin(), f.values().end());
        init_l = detail::initial_lambda(init, cfg.rank);
    }
    cpdb_ctx* ctx = nullptr;
    const char* env = std::getenv("CPD_DEVICE");
    abi::check(cpdb_create(env ? std::atoi(env) : 0, &ctx));
    struct Guard {
        cpdb_ctx* c;
        ~Guard() { cpdb_destroy(c); }
    } guard{ctx};
    const std::vector<uint64_t> dims = abi::u64(x.shape().dims());
    abi::check(cpdb_tensor_set(ctx, x.data(), dims.data(), uint32_t(x.order())));
    return detail::run_als_on_context(ctx, x.shape().dims(), cfg, init ? init_f.data() : nullptr,
                                      init ? init_l.data() : nullptr);
}

inline SolveResult cp_als_qr(const DenseTensor& x, const SolverConfig& cfg,
                             const std::optional<KruskalModel>& init = {}) {
    if (cfg.algorithm != Algorithm::als_qr)
        throw std::invalid_argument("cp_als_qr: config algorithm must be als-qr");
    return detail::run_qr(x, cfg, init, false);
}

inline SolveResult als_qr_bre(const DenseTensor& x, const SolverConfig& cfg,
                              const std::optional<KruskalModel>& init = {}) {
    SolverConfig bre = cfg;
    bre.algorithm = Algorithm::als_qr;
    bre.strategy = Strategy::branch_reuse;
    bre.extrapolation_enabled = true;
    return detail::run_qr(x, bre, init, true);
}

}  // namespace cpd
