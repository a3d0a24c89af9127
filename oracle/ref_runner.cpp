// Reference runner: a C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/cpd, compiled in place by oracle/Makefile into
// oracle/_ref/libcpdref.so).  It is the pin for the C restatement
// (oracle/cpd_oracle.c) and the `kind: "reference"` CPU baseline in bench.py.
//
// TEST INFRASTRUCTURE ONLY.  Nothing on the product path links this library;
// only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs load it.  No reference source is copied: the build passes
// -I /root/reference/proj/include.
//
// Entry points follow the reference functions they wrap (file:line relative to
// /root/reference/proj/include/cpd):
//   cpdref_ttm              tensor.hpp:288-315   ttm
//   cpdref_thin_qr          linalg.hpp:39-99     thin_qr
//   cpdref_khatri_rao       tensor.hpp:343-368   khatri_rao
//   cpdref_unfold           tensor.hpp:217-250   unfold
//   cpdref_solve_rows_lower linalg.hpp:192-216   solve_rows_lower_triangular
//   cpdref_normalize_columns linalg.hpp:225-242  normalize_columns
//   cpdref_extrapolate_q0   solvers.hpp:75-86    extrapolate_q0
//   cpdref_select_beta      solvers.hpp:92-101   select_beta
//   cpdref_fitness_fast_qr  kruskal.hpp:109-128  fitness_fast_qr
//   cpdref_schedule         dim_tree.hpp:386-426 build_schedule (flattened)
//   cpdref_measured_cost    dim_tree.hpp:549-570 measured_cost
//   cpdref_closed_form_cost dim_tree.hpp:579-621 closed_form_cost
//   cpdref_execute_run      dim_tree.hpp:473-544 execute, driven as in
//                           dim_tree_test.cpp:37-73 (random factor refresh)
//   cpdref_solve            solvers.hpp:317-336  cp_als_qr / als_qr_bre, or a
//                           loop-for-loop mirror of run_qr (solvers.hpp:215-309)
//                           when a resume state or per-sweep dumps are requested
//   cpdref_cp_als           solvers.hpp:149-208  cp_als (normal equations)
//   cpdref_mttkrp           tensor.hpp:453-488   mttkrp (streaming path)
//   cpdref_solve_spd        linalg.hpp:132-187   solve_spd
//   cpdref_fitness_fast_als kruskal.hpp:88-104   fitness_fast_als
//   cpdref_synth_baseline   BASELINE.json configs built from rng.hpp +
//                           kruskal.hpp:54-67 reconstruct
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cpd/dim_tree.hpp"
#include "cpd/factor_state.hpp"
#include "cpd/io.hpp"
#include "cpd/synth.hpp"
#include "cpd/kruskal.hpp"
#include "cpd/linalg.hpp"
#include "cpd/rng.hpp"
#include "cpd/solvers.hpp"
#include "cpd/tensor.hpp"

#include "cpd_abi_types.h"

namespace {

thread_local std::string g_error;

// Status codes shared with the product ABI (include/cpdb.h).
enum : int {
    kOk = 0,
    kInvalidArgument = 1,
    kStale = 2,
    kSingularTriangular = 3,
    kLogic = 4,
    kOther = 5,
    kSingularSystem = 10,
};

template <class F>
int guarded(F&& body) {
    try {
        body();
        return kOk;
    } catch (const cpd::stale_intermediate_error& e) {
        g_error = e.what();
        return kStale;
    } catch (const cpd::singular_triangular_error& e) {
        g_error = e.what();
        return kSingularTriangular;
    } catch (const cpd::singular_system_error& e) {
        g_error = e.what();
        return kSingularSystem;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return kInvalidArgument;
    } catch (const std::logic_error& e) {
        g_error = e.what();
        return kLogic;
    } catch (const std::exception& e) {
        g_error = e.what();
        return kOther;
    }
}

cpd::Shape make_shape(const uint64_t* dims, uint32_t order) {
    std::vector<std::size_t> d(dims, dims + order);
    return cpd::Shape(d);
}

cpd::DenseTensor make_tensor(const double* data, const uint64_t* dims, uint32_t order) {
    cpd::Shape s = make_shape(dims, order);
    std::vector<double> v(data, data + s.element_count());
    return cpd::DenseTensor(std::move(s), std::move(v));
}

cpd::Matrix make_matrix(const double* data, uint64_t rows, uint64_t cols) {
    return cpd::Matrix(rows, cols, std::vector<double>(data, data + rows * cols));
}

void put(const cpd::Matrix& m, double* out) {
    std::memcpy(out, m.data(), m.size() * sizeof(double));
}

cpd::Strategy strategy_of(int32_t s) {
    switch (s) {
        case 0: return cpd::Strategy::naive;
        case 1: return cpd::Strategy::dim_tree;
        case 2: return cpd::Strategy::branch_reuse;
    }
    throw std::invalid_argument("strategy code out of range");
}

cpd::SolverConfig config_of(const cpdo_config& c) {
    cpd::SolverConfig cfg;
    cfg.rank = c.rank;
    cfg.max_iterations = c.max_iterations;
    cfg.fitness_threshold = c.fitness_threshold;
    cfg.algorithm = cpd::Algorithm::als_qr;
    cfg.strategy = strategy_of(c.strategy);
    cfg.extrapolation_enabled = c.extrapolate != 0;
    cfg.alpha = c.alpha;
    if (c.has_beta_override) cfg.beta_override = c.beta_override;
    cfg.activation_gap = c.activation_gap;
    cfg.seed = c.seed;
    return cfg;
}

void put_row(const cpd::TraceRow& t, cpdo_trace_row* out) {
    std::memset(out, 0, sizeof *out);
    out->iteration = t.iteration;
    out->order = static_cast<uint32_t>(t.update_order.size());
    for (std::size_t i = 0; i < t.update_order.size() && i < CPDO_MAX_ORDER; ++i)
        out->update_order[i] = static_cast<uint32_t>(t.update_order[i]);
    out->fitness = t.fitness;
    out->raw_radicand = t.raw_radicand;
    out->wall_seconds = t.wall_seconds;
    out->root_ttm_count = t.root_ttm_count;
    out->flops = t.flops;
    out->beta_used = t.beta_used;
    out->regularized = t.regularized ? 1 : 0;
}

// X contracted with Q_k^T for every mode k outside `key`, descending mode
// order: rebuilds a retained branch-reuse intermediate from the current
// factors (legal by the freshness invariant, dim_tree.hpp:109-111).
cpd::DenseTensor rebuild_entry(const cpd::DenseTensor& x, const cpd::FactorState& st,
                               cpd::ModeSet key) {
    cpd::DenseTensor t = x;
    for (std::size_t k = x.order(); k-- > 0;)
        if (!(key & cpd::mode_bit(k))) t = cpd::ttm(t, cpd::transpose(st.q(k)), k);
    return t;
}

// Loop-for-loop mirror of detail::run_qr (solvers.hpp:215-309) that can start
// from a sweep-boundary state and dump per-sweep factors.  With sweeps_done ==
// 0 it reproduces cp_als_qr / als_qr_bre bit for bit (checked in
// tests/test_oracle_ref.py).
void mirror_run(const cpd::DenseTensor& x, const cpdo_config& c, cpdo_state* st,
                cpdo_trace_row* trace, uint64_t* trace_len, double* factors_per_sweep,
                double* lambda_per_sweep, cpdo_q0_observer observer, void* observer_user) {
    const cpd::SolverConfig cfg = config_of(c);
    cfg.validate();
    const bool extrapolate = c.extrapolate != 0;
    const std::size_t order = x.order();
    const std::size_t rank = cfg.rank;
    const double norm_x_sq = cpd::inner(x, x);
    if (norm_x_sq == 0.0) throw std::invalid_argument("cp_als_qr: zero-norm tensor");
    for (std::size_t k = 0; k < order; ++k)
        if (rank > x.shape().extent(k))
            throw std::invalid_argument("cp_als_qr: rank must not exceed any mode extent");

    const uint64_t done = st ? st->sweeps_done : 0;
    std::vector<cpd::Matrix> init;
    if (st && st->factors) {
        const double* p = st->factors;
        for (std::size_t k = 0; k < order; ++k) {
            init.push_back(make_matrix(p, x.shape().extent(k), rank));
            p += x.shape().extent(k) * rank;
        }
    } else {
        init = cpd::detail::initial_factors(x, cfg, std::nullopt);
    }
    cpd::FactorState state = cpd::FactorState::from_factors(init);
    state.lambda.assign(rank, 1.0);
    if (st && st->lambda) state.lambda.assign(st->lambda, st->lambda + rank);

    const cpd::Strategy strategy = extrapolate ? cpd::Strategy::branch_reuse : cfg.strategy;
    const cpd::Schedule schedule = cpd::build_schedule(order, strategy, done + cfg.max_iterations);
    cpd::IntermediateCache cache;
    if (done > 0) {
        for (cpd::ModeSet key : cpd::detail::retained_keys(schedule, done - 1, order - 1)) {
            if (cache.find(key)) continue;
            cpd::IntermediateCache::Entry e;
            e.tensor = rebuild_entry(x, state, key);
            for (std::size_t k = 0; k < order; ++k)
                if (!(key & cpd::mode_bit(k))) e.stamps[k] = state.version(k);
            cache.put(key, std::move(e));
        }
    }

    std::size_t zrows = 1;
    for (std::size_t k = 1; k < order; ++k) zrows *= rank;
    std::vector<std::optional<cpd::Matrix>> history(order);
    if (st && st->q0_history) {
        for (std::size_t n = 0; n < order; ++n)
            if (st->history_mask & (1u << n))
                history[n] = make_matrix(st->q0_history + n * zrows * rank, zrows, rank);
    }
    std::optional<double> active_beta;
    if (extrapolate && cfg.beta_override) active_beta = *cfg.beta_override;
    if (extrapolate && st && st->has_active_beta && !active_beta) active_beta = st->active_beta;
    std::optional<double> prev_fitness;
    if (st && st->has_prev_fitness) prev_fitness = st->prev_fitness;

    cpd::CostReport total =
        done > 0 ? cpd::measured_cost(schedule, x.shape().dims(), rank, done) : cpd::CostReport{};

    cpd::detail::WallClock clock;
    uint64_t rows = 0;
    for (uint64_t sweep = done + 1; sweep <= done + cfg.max_iterations; ++sweep) {
        cpd::Matrix v_last, a_hat_last, r0_last;
        std::size_t last_mode = 0;
        double beta_used = 0.0;
        const std::vector<std::size_t> update_order = schedule.update_order(sweep - 1);
        for (std::size_t n : update_order) {
            std::vector<const cpd::Matrix*> r_desc;
            for (std::size_t k = order; k-- > 0;)
                if (k != n) r_desc.push_back(&state.r(k));
            const cpd::Matrix z = cpd::khatri_rao(
                std::span<const cpd::Matrix* const>(r_desc.data(), r_desc.size()));
            cpd::QrPair zq = cpd::thin_qr(z);
            if (observer) observer(observer_user, sweep, static_cast<uint32_t>(n), zq.q.data(),
                                   zq.q.rows(), zq.q.cols());
            const cpd::Matrix* q_used = &zq.q;
            cpd::Matrix q_ex;
            if (extrapolate && active_beta && *active_beta != 0.0 && history[n]) {
                q_ex = cpd::extrapolate_q0(zq.q, *history[n], *active_beta, cfg.alpha);
                q_used = &q_ex;
                beta_used = *active_beta;
            }
            if (extrapolate) history[n] = zq.q;

            auto [y, cost] = cpd::execute(schedule, x, state, cache, sweep - 1, n);
            total.merge(cost);
            const cpd::Matrix y_n = cpd::unfold(y, n);
            cpd::Matrix v = cpd::matmul(y_n, *q_used);
            cpd::Matrix a_hat = cpd::solve_rows_lower_triangular(cpd::transpose(zq.r), v);
            auto normalized = cpd::normalize_columns(a_hat);
            state.lambda = std::move(normalized.weights);
            state.update(n, std::move(normalized.matrix));
            if (n == update_order.back() && q_used != &zq.q) v = cpd::matmul(y_n, zq.q);
            v_last = std::move(v);
            a_hat_last = std::move(a_hat);
            r0_last = std::move(zq.r);
            last_mode = n;
        }
        const cpd::FitnessResult fit = cpd::fitness_fast_qr(
            norm_x_sq, v_last, a_hat_last, r0_last, state.r(last_mode), state.lambda);
        cpd::TraceRow row{sweep, update_order, fit.fitness, fit.raw_radicand, clock.seconds(),
                          total.root_ttm_count, total.total_flops, beta_used, false};
        if (trace) put_row(row, trace + rows);
        if (factors_per_sweep) {
            std::size_t per = 0;
            for (std::size_t k = 0; k < order; ++k) per += state.modes[k].factor.size();
            double* p = factors_per_sweep + rows * per;
            for (std::size_t k = 0; k < order; ++k) {
                put(state.modes[k].factor, p);
                p += state.modes[k].factor.size();
            }
        }
        if (lambda_per_sweep)
            std::memcpy(lambda_per_sweep + rows * rank, state.lambda.data(), rank * sizeof(double));
        ++rows;
        if (extrapolate && !active_beta && !cfg.beta_override && sweep >= 2 && prev_fitness)
            active_beta = cpd::select_beta(*prev_fitness, fit.fitness, cfg.activation_gap);
        prev_fitness = fit.fitness;
        if (fit.fitness >= cfg.fitness_threshold) break;
    }
    if (trace_len) *trace_len = rows;

    if (st) {
        st->sweeps_done = done + rows;
        if (st->lambda) std::memcpy(st->lambda, state.lambda.data(), rank * sizeof(double));
        if (st->factors) {
            double* p = st->factors;
            for (std::size_t k = 0; k < order; ++k) {
                put(state.modes[k].factor, p);
                p += state.modes[k].factor.size();
            }
        }
        if (st->q0_history) {
            st->history_mask = 0;
            for (std::size_t n = 0; n < order; ++n)
                if (history[n]) {
                    put(*history[n], st->q0_history + n * zrows * rank);
                    st->history_mask |= 1u << n;
                }
        }
        st->has_active_beta = active_beta ? 1 : 0;
        st->active_beta = active_beta ? *active_beta : 0.0;
        st->has_prev_fitness = prev_fitness ? 1 : 0;
        st->prev_fitness = prev_fitness ? *prev_fitness : 0.0;
    }
}

}  // namespace

extern "C" {

const char* cpdref_last_error(void) { return g_error.c_str(); }

int cpdref_rng_normals(uint64_t seed, uint64_t n, double* out) {
    cpd::Rng rng(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng.normal();
    return kOk;
}

int cpdref_rng_uniforms(uint64_t seed, uint64_t n, double* out) {
    cpd::Rng rng(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng.uniform();
    return kOk;
}

int cpdref_ttm(const double* t, const uint64_t* dims, uint32_t order, const double* b,
               uint64_t b_rows, uint32_t mode, double* out) {
    return guarded([&] {
        const cpd::DenseTensor x = make_tensor(t, dims, order);
        if (mode >= order) throw std::invalid_argument("ttm: mode out of range");
        const cpd::Matrix m = make_matrix(b, b_rows, dims[mode]);
        const cpd::DenseTensor y = cpd::ttm(x, m, mode);
        std::memcpy(out, y.data(), y.size() * sizeof(double));
    });
}

int cpdref_unfold(const double* t, const uint64_t* dims, uint32_t order, uint32_t mode,
                  double* out) {
    return guarded([&] { put(cpd::unfold(make_tensor(t, dims, order), mode), out); });
}

int cpdref_thin_qr(const double* a, uint64_t m, uint64_t n, double* q, double* r) {
    return guarded([&] {
        const cpd::QrPair p = cpd::thin_qr(make_matrix(a, m, n));
        put(p.q, q);
        put(p.r, r);
    });
}

int cpdref_khatri_rao(const double* const* mats, const uint64_t* rows, uint32_t count,
                      uint64_t cols, double* out) {
    return guarded([&] {
        std::vector<cpd::Matrix> ms;
        for (uint32_t i = 0; i < count; ++i) ms.push_back(make_matrix(mats[i], rows[i], cols));
        std::vector<const cpd::Matrix*> ptrs;
        for (auto& m : ms) ptrs.push_back(&m);
        put(cpd::khatri_rao(std::span<const cpd::Matrix* const>(ptrs.data(), ptrs.size())), out);
    });
}

int cpdref_solve_rows_lower(const double* l, uint64_t n, const double* rhs, uint64_t rows,
                            double* out, int64_t* bad_column) {
    if (bad_column) *bad_column = -1;
    return guarded([&] {
        try {
            put(cpd::solve_rows_lower_triangular(make_matrix(l, n, n), make_matrix(rhs, rows, n)),
                out);
        } catch (const cpd::singular_triangular_error& e) {
            if (bad_column) *bad_column = static_cast<int64_t>(e.column);
            throw;
        }
    });
}

int cpdref_normalize_columns(const double* a, uint64_t m, uint64_t n, double* out,
                             double* weights) {
    return guarded([&] {
        auto nc = cpd::normalize_columns(make_matrix(a, m, n));
        put(nc.matrix, out);
        std::memcpy(weights, nc.weights.data(), n * sizeof(double));
    });
}

int cpdref_extrapolate_q0(const double* now, const double* prev, uint64_t rows, uint64_t cols,
                          double beta, double alpha, double* out) {
    return guarded([&] {
        put(cpd::extrapolate_q0(make_matrix(now, rows, cols), make_matrix(prev, rows, cols), beta,
                                alpha),
            out);
    });
}

int cpdref_select_beta(double prev, double now, double gap, double* beta) {
    const auto b = cpd::select_beta(prev, now, gap);
    *beta = b ? *b : 0.0;
    return b ? 1 : 0;
}

int cpdref_fitness_fast_qr(double norm_x_sq, const double* v, const double* a_hat, uint64_t rows,
                           const double* r0, const double* r_n, const double* lambda, uint64_t r,
                           double* fitness, double* raw) {
    return guarded([&] {
        const auto f = cpd::fitness_fast_qr(norm_x_sq, make_matrix(v, rows, r),
                                            make_matrix(a_hat, rows, r), make_matrix(r0, r, r),
                                            make_matrix(r_n, r, r),
                                            std::vector<double>(lambda, lambda + r));
        *fitness = f.fitness;
        *raw = f.raw_radicand;
    });
}

// Flattened schedule: per step {iteration, block, mode, source, contract, produces}.
int cpdref_schedule(uint32_t order, int32_t strategy, uint64_t iterations, int64_t* out,
                    uint64_t cap_steps, uint64_t* n_steps, uint64_t* cycle) {
    return guarded([&] {
        const cpd::Schedule s = cpd::build_schedule(order, strategy_of(strategy), iterations);
        uint64_t n = 0;
        for (std::size_t i = 0; i < s.num_iterations(); ++i) {
            const auto& it = s.iteration(i);
            for (std::size_t b = 0; b < it.updates.size(); ++b)
                for (const auto& st : it.updates[b].steps) {
                    if (n < cap_steps) {
                        int64_t* row = out + 6 * n;
                        row[0] = static_cast<int64_t>(i);
                        row[1] = static_cast<int64_t>(b);
                        row[2] = static_cast<int64_t>(it.updates[b].mode);
                        row[3] = st.source;
                        row[4] = static_cast<int64_t>(st.contract_mode);
                        row[5] = st.produces;
                    }
                    ++n;
                }
        }
        *n_steps = n;
        cycle[0] = s.cycle_start();
        cycle[1] = s.cycle_length();
    });
}

int cpdref_retained_keys(uint32_t order, int32_t strategy, uint64_t iterations, uint64_t iter,
                         uint64_t block, uint32_t* out, uint64_t cap, uint64_t* n) {
    return guarded([&] {
        const cpd::Schedule s = cpd::build_schedule(order, strategy_of(strategy), iterations);
        const auto keys = cpd::detail::retained_keys(s, iter, block);
        *n = keys.size();
        for (std::size_t i = 0; i < keys.size() && i < cap; ++i) out[i] = keys[i];
    });
}

int cpdref_measured_cost(uint32_t order, int32_t strategy, const uint64_t* dims, uint64_t rank,
                         uint64_t iterations, uint64_t* total_flops, uint64_t* roots) {
    return guarded([&] {
        const cpd::Schedule s = cpd::build_schedule(order, strategy_of(strategy), iterations);
        const auto c =
            cpd::measured_cost(s, std::vector<std::size_t>(dims, dims + order), rank, iterations);
        *total_flops = c.total_flops;
        *roots = c.root_ttm_count;
    });
}

int cpdref_closed_form_cost(uint32_t order, int32_t strategy, const uint64_t* dims, uint64_t rank,
                            uint64_t* total) {
    return guarded([&] {
        *total = cpd::closed_form_cost(order, strategy_of(strategy),
                                       std::vector<std::size_t>(dims, dims + order), rank);
    });
}

// execute() driven like dim_tree_test.cpp:37-73: for `iterations` sweeps of the
// plan, run every scheduled update, write its Y (concatenated), then refresh
// that mode's factor with normalize_columns(random) from the same Rng stream.
int cpdref_execute_run(const double* x, const uint64_t* dims, uint32_t order, uint64_t rank,
                       int32_t strategy, uint64_t iterations, uint64_t seed,
                       const double* init_factors, double* y_out, uint64_t* flops_out) {
    return guarded([&] {
        const cpd::DenseTensor t = make_tensor(x, dims, order);
        std::vector<cpd::Matrix> f;
        const double* p = init_factors;
        for (uint32_t k = 0; k < order; ++k) {
            f.push_back(make_matrix(p, dims[k], rank));
            p += dims[k] * rank;
        }
        cpd::FactorState state = cpd::FactorState::from_factors(f);
        const cpd::Schedule s = cpd::build_schedule(order, strategy_of(strategy), iterations);
        cpd::IntermediateCache cache;
        cpd::Rng rng(seed);
        double* out = y_out;
        uint64_t u = 0;
        for (uint64_t it = 0; it < iterations; ++it)
            for (std::size_t mode : s.update_order(it)) {
                auto [y, cost] = cpd::execute(s, t, state, cache, it, mode);
                std::memcpy(out, y.data(), y.size() * sizeof(double));
                out += y.size();
                if (flops_out) flops_out[u] = cost.total_flops;
                ++u;
                cpd::Matrix m(dims[mode], rank);
                for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = rng.normal();
                state.update(mode, cpd::normalize_columns(m).matrix);
            }
    });
}

int cpdref_solve(const double* x, const uint64_t* dims, uint32_t order, const cpdo_config* cfg,
                 cpdo_state* state, cpdo_trace_row* trace, uint64_t* trace_len,
                 double* out_lambda, double* out_factors, double* factors_per_sweep,
                 double* lambda_per_sweep, cpdo_q0_observer observer, void* observer_user) {
    return guarded([&] {
        const cpd::DenseTensor t = make_tensor(x, dims, order);
        const bool mirror = state != nullptr || factors_per_sweep != nullptr ||
                            lambda_per_sweep != nullptr;
        if (mirror) {
            cpdo_state local{};
            std::vector<double> lam(cfg->rank), fac;
            for (uint32_t k = 0; k < order; ++k) fac.resize(fac.size() + dims[k] * cfg->rank);
            cpdo_state* st = state;
            if (!st) {
                st = &local;
                local.lambda = lam.data();
                local.factors = nullptr;
            }
            mirror_run(t, *cfg, st, trace, trace_len, factors_per_sweep, lambda_per_sweep,
                       observer, observer_user);
            if (out_lambda && st->lambda) std::memcpy(out_lambda, st->lambda, cfg->rank * 8);
            if (out_factors && st->factors)
                std::memcpy(out_factors, st->factors, fac.size() * sizeof(double));
            if (out_factors && !st->factors && factors_per_sweep && trace_len && *trace_len)
                std::memcpy(out_factors, factors_per_sweep + (*trace_len - 1) * fac.size(),
                            fac.size() * sizeof(double));
            return;
        }
        cpd::SolverConfig c = config_of(*cfg);
        if (observer)
            c.q0_observer = [&](std::size_t sweep, std::size_t mode, const cpd::Matrix& q0) {
                observer(observer_user, sweep, static_cast<uint32_t>(mode), q0.data(), q0.rows(),
                         q0.cols());
            };
        const cpd::SolveResult r = cfg->extrapolate ? cpd::als_qr_bre(t, c) : cpd::cp_als_qr(t, c);
        for (std::size_t i = 0; i < r.trace.size(); ++i)
            if (trace) put_row(r.trace[i], trace + i);
        if (trace_len) *trace_len = r.trace.size();
        if (out_lambda)
            std::memcpy(out_lambda, r.model.lambda.data(), r.model.lambda.size() * sizeof(double));
        if (out_factors) {
            double* p = out_factors;
            for (const auto& f : r.model.factors) {
                put(f, p);
                p += f.size();
            }
        }
    });
}

// kruskal.hpp:54-67 reconstruct through the reference itself
int cpdref_reconstruct(const uint64_t* dims, uint32_t order, uint64_t rank, const double* lambda,
                       const double* factors, double* out) {
    return guarded([&] {
        const cpd::Shape shape = make_shape(dims, order);
        cpd::KruskalModel m;
        m.lambda.assign(lambda, lambda + rank);
        const double* p = factors;
        for (uint32_t k = 0; k < order; ++k) {
            cpd::Matrix f(dims[k], rank);
            std::memcpy(f.data(), p, dims[k] * rank * sizeof(double));
            p += dims[k] * rank;
            m.factors.push_back(std::move(f));
        }
        const cpd::DenseTensor xt = cpd::reconstruct(m, shape);
        std::memcpy(out, xt.data(), xt.size() * sizeof(double));
    });
}

// BASELINE.json synthetic construction.
// kind 0: i.i.d. N(0,1) factors drawn mode by mode, row-major.
// kind 1: per mode a shared g ~ N(0,1)^I, then per column j: U ~ U(0,1),
//         h_j ~ N(0,1)^I, column = 10^(-3U) (sqrt(0.9) g + sqrt(0.1) h_j).
// X = reconstruct(lambda = 1, factors) + rho ||X|| / ||E|| E, E ~ N(0,1) drawn
// after the factors from the same stream.
int cpdref_synth_baseline(int32_t kind, const uint64_t* dims, uint32_t order, uint64_t rank,
                          double rho, uint64_t seed, double* out, double* truth_factors) {
    return guarded([&] {
        cpd::Rng rng(seed);
        const cpd::Shape shape = make_shape(dims, order);
        cpd::KruskalModel truth;
        truth.lambda.assign(rank, 1.0);
        for (uint32_t k = 0; k < order; ++k) {
            cpd::Matrix f(dims[k], rank);
            if (kind == 0) {
                for (std::size_t i = 0; i < f.size(); ++i) f.data()[i] = rng.normal();
            } else if (kind == 1) {
                std::vector<double> g(dims[k]);
                for (auto& v : g) v = rng.normal();
                for (uint64_t j = 0; j < rank; ++j) {
                    const double s = std::pow(10.0, -3.0 * rng.uniform());
                    for (uint64_t i = 0; i < dims[k]; ++i)
                        f(i, j) = s * (std::sqrt(0.9) * g[i] + std::sqrt(0.1) * rng.normal());
                }
            } else {
                throw std::invalid_argument("synth: unknown kind");
            }
            truth.factors.push_back(std::move(f));
        }
        cpd::DenseTensor xt = cpd::reconstruct(truth, shape);
        if (rho > 0.0) {
            cpd::DenseTensor noise(shape);
            for (double& v : noise.values()) v = rng.normal();
            const double scale = rho * cpd::frobenius_norm(xt) / cpd::frobenius_norm(noise);
            for (std::size_t i = 0; i < xt.size(); ++i) xt.data()[i] += scale * noise.data()[i];
        }
        std::memcpy(out, xt.data(), xt.size() * sizeof(double));
        if (truth_factors) {
            double* p = truth_factors;
            for (const auto& f : truth.factors) {
                put(f, p);
                p += f.size();
            }
        }
    });
}

// ---- .cpdt files through the reference's own codec (io.hpp:93-121, 176-209) ----
// 8 = file_error, 9 = format_error (the CLI's exit codes 2 / 3 distinguish them)
int cpdref_write_tensor_file(const char* path, const double* data, const uint64_t* dims,
                             uint32_t order) {
    try {
        cpd::write_tensor_file(path, make_tensor(data, dims, order));
        return kOk;
    } catch (const cpd::file_error& e) {
        g_error = e.what();
        return 8;
    } catch (const std::exception& e) {
        g_error = e.what();
        return kOther;
    }
}

int cpdref_read_tensor_file(const char* path, uint32_t* order, uint64_t* dims, double* out,
                            uint64_t cap) {
    try {
        const cpd::DenseTensor t = cpd::read_tensor_file(path);
        *order = uint32_t(t.order());
        for (std::size_t k = 0; k < t.order() && k < 8; ++k) dims[k] = t.shape().extent(k);
        if (out && t.size() <= cap) std::memcpy(out, t.data(), t.size() * sizeof(double));
        return kOk;
    } catch (const cpd::file_error& e) {
        g_error = e.what();
        return 8;
    } catch (const cpd::format_error& e) {
        g_error = e.what();
        return 9;
    } catch (const std::exception& e) {
        g_error = e.what();
        return kOther;
    }
}

// ---- the reference's synthetic generator (synth.hpp:80-106, CLI `synth`) ----
int cpdref_assemble_noisy(const uint64_t* dims, uint32_t order, uint64_t rank,
                          const double* collinearity, double l1, double l2, uint64_t seed,
                          double* out) {
    return guarded([&] {
        cpd::SynthSpec spec;
        spec.dims = make_shape(dims, order);
        spec.true_rank = rank;
        spec.collinearity.assign(collinearity, collinearity + order);
        spec.l1 = l1;
        spec.l2 = l2;
        spec.seed = seed;
        const cpd::SynthResult r = cpd::assemble_noisy_tensor(spec);
        std::memcpy(out, r.tensor.data(), r.tensor.size() * sizeof(double));
    });
}

int cpdref_cp_als(const double* x, const uint64_t* dims, uint32_t order, const cpdo_config* cfg,
                  const double* init_lambda, const double* init_factors, cpdo_trace_row* trace,
                  uint64_t* trace_len, double* out_lambda, double* out_factors) {
    return guarded([&] {
        const cpd::DenseTensor t = make_tensor(x, dims, order);
        cpd::SolverConfig c = config_of(*cfg);
        c.algorithm = cpd::Algorithm::als;
        std::optional<cpd::KruskalModel> init;
        if (init_factors) {
            cpd::KruskalModel m;
            m.lambda.assign(init_lambda, init_lambda + cfg->rank);
            const double* p = init_factors;
            for (uint32_t k = 0; k < order; ++k) {
                m.factors.push_back(make_matrix(p, dims[k], cfg->rank));
                p += dims[k] * cfg->rank;
            }
            init = std::move(m);
        }
        const cpd::SolveResult r = cpd::cp_als(t, c, init);
        for (std::size_t i = 0; i < r.trace.size(); ++i)
            if (trace) put_row(r.trace[i], trace + i);
        if (trace_len) *trace_len = r.trace.size();
        if (out_lambda)
            std::memcpy(out_lambda, r.model.lambda.data(), r.model.lambda.size() * sizeof(double));
        if (out_factors) {
            double* p = out_factors;
            for (const auto& f : r.model.factors) {
                put(f, p);
                p += f.size();
            }
        }
    });
}

int cpdref_mttkrp(const double* t, const uint64_t* dims, uint32_t order,
                  const double* const* factors, uint64_t rank, uint32_t mode, double* out) {
    return guarded([&] {
        const cpd::DenseTensor x = make_tensor(t, dims, order);
        std::vector<cpd::Matrix> mats(order);
        std::vector<const cpd::Matrix*> ptrs(order, nullptr);
        for (uint32_t k = 0; k < order; ++k) {
            if (k == mode || !factors[k]) continue;
            mats[k] = make_matrix(factors[k], dims[k], rank);
            ptrs[k] = &mats[k];
        }
        put(cpd::mttkrp(x, std::span<const cpd::Matrix* const>(ptrs.data(), ptrs.size()), mode),
            out);
    });
}

int cpdref_solve_spd(const double* g, uint64_t n, const double* rhs, uint64_t rows, double* x,
                     int32_t* regularized) {
    return guarded([&] {
        const auto r = cpd::solve_spd(make_matrix(g, n, n), make_matrix(rhs, rows, n));
        put(r.x, x);
        if (regularized) *regularized = r.regularized ? 1 : 0;
    });
}

int cpdref_fitness_fast_als(double nx2, const double* m, const double* a_hat, uint64_t rows,
                            uint64_t cols, const double* gamma, const double* lambda, uint64_t r,
                            const double* s_last, double* fitness, double* raw) {
    return guarded([&] {
        const cpd::FitnessResult f = cpd::fitness_fast_als(
            nx2, make_matrix(m, rows, cols), make_matrix(a_hat, rows, cols),
            make_matrix(gamma, r, r), std::vector<double>(lambda, lambda + r),
            make_matrix(s_last, r, r));
        *fitness = f.fitness;
        *raw = f.raw_radicand;
    });
}

}  // extern "C"
