// cp_als (/root/reference/proj/include/cpd/solvers.hpp:149-208) on the device,
// and the MTTKRP / solve_spd / fitness_fast_als primitives behind the drop-in
// headers.  X, the factors, their Grams and every intermediate stay in HBM;
// the host reads one fitness row per sweep.  Sharded contexts (mode 0 split
// across ranks) reduce the I_n x R MTTKRP partials: an
// all-reduce for n != 0, an all-gather of the local rows for n = 0.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "cpd/rng.hpp"
#include "kernels.hpp"
#include "runtime.hpp"

namespace cpdb {

namespace {

struct MttkrpBufs {
    DevBuf t, w, part;
};

// M (I_n x R, local rows for n = 0 on a sharded context, else partial sums
// that the caller reduces) = X_(n) KR(A_k, k != n) of the device tensor x
// with local extents ld.  fac[k] / qp[k]: A_k (its local rows for k = 0) and
// its packed copy for the TTM kernel.
void mttkrp_dev(cpdb_ctx* c, const double* x, const std::vector<uint64_t>& ld,
                const std::vector<const double*>& fac, const std::vector<const double*>& qp,
                uint32_t R, uint32_t n, MttkrpBufs& b, double* m_out, cudaStream_t s) {
    const uint32_t N = uint32_t(ld.size());
    const uint32_t cm = (n == N - 1) ? 0 : N - 1;  // contraction mode of the TTM
    std::vector<uint64_t> td = ld;
    td[cm] = R;
    double* t = b.t.ensure(numel(td));
    run_ttm(c, x, ld, cm, fac[cm], qp[cm], R, t, s);
    KrcArgs a{};
    a.t = t;
    a.R = R;
    for (uint32_t k = 0; k < N; ++k) {
        a.fac[k] = fac[k];
        a.dims[k] = ld[k];
    }
    a.rows_w = 1;
    for (uint32_t k = 0; k < N; ++k)
        if (k != n && k != cm) {
            a.km[a.nkm++] = k;
            a.rows_w *= ld[k];
        }
    a.In = ld[n];
    if (cm == N - 1) {
        a.router = 0;
        a.P = 1;
        a.Q = 1;
        for (uint32_t k = 0; k < n; ++k) a.P *= ld[k];
        for (uint32_t k = n + 1; k < N - 1; ++k) a.Q *= ld[k];
    } else {
        a.router = 1;
        a.P = 1;
        a.Q = 1;
        for (uint32_t k = 1; k < N - 1; ++k) a.Q *= ld[k];
    }
    double* w = b.w.ensure(std::max<uint64_t>(a.rows_w, 1) * R);
    CPDB_CK(launch_kr_table(a, w, s));
    const uint64_t split = krc_split(a, c->sms);
    double* out = split > 1 ? b.part.ensure(split * a.In * R) : m_out;
    CPDB_CK(launch_krc(a, w, out, split, s));
    c->launches += 3;
    if (split > 1) {
        CPDB_CK(reduce_splits(out, uint32_t(split), a.In * R, m_out, s));
        c->launches += 1;
    }
}

// Reduce the rank-local MTTKRP into the full M on every rank.
void mttkrp_combine(cpdb_ctx* c, uint32_t n, double* m_full, uint32_t R) {
    if (c->world <= 1) return;
    if (n == 0) {
        allgather(c, m_full, c->rows * R);
    } else {
        allreduce_sum(c, m_full, c->dims[n] * R);
    }
}

}  // namespace

// ---------------------------------------------------------------- cp_als
void als_solve(cpdb_ctx* c, const cpdb_config& cfg, const double* init_lambda,
               const double* init_factors, cpdb_trace_row* trace, uint64_t* trace_len,
               double* out_lambda, double* out_factors) {
    // SolverConfig::validate (solvers.hpp:41-49) and cp_als's own checks (:152-156)
    if (cfg.rank == 0) fail(CPDB_INVALID_ARGUMENT, "SolverConfig: rank must be >= 1");
    if (cfg.max_iterations == 0)
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: need at least one iteration");
    if (!(cfg.fitness_threshold >= 0.0 && cfg.fitness_threshold <= 1.0))
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: fitness threshold must be in [0,1]");
    if (!std::isfinite(cfg.alpha) || !std::isfinite(cfg.activation_gap))
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: alpha and activation gap must be finite");
    require_tensor(c);
    const uint32_t N = uint32_t(c->dims.size());
    if (N < 2) fail(CPDB_INVALID_ARGUMENT, "cp_als: tensor order must be >= 2");
    const double nx2 = ctx_norm_sq(c);
    if (nx2 == 0.0) fail(CPDB_INVALID_ARGUMENT, "cp_als: zero-norm tensor");
    if (cfg.rank > 1024)
        fail(CPDB_INVALID_ARGUMENT, "cp_als: ranks above 1024 are not supported on the device");
    const uint32_t R = uint32_t(cfg.rank);
    cudaStream_t s = c->stream;
    const bool sharded = c->world > 1;

    // factors, lambda (initial_factors / initial_lambda, solvers.hpp:105-130)
    std::vector<DevBuf> A(N), AP(N), G(N);
    uint64_t nfac = 0;
    for (uint64_t d : c->dims) nfac += d * R;
    {
        std::vector<double> init(nfac);
        if (init_factors) {
            std::memcpy(init.data(), init_factors, nfac * sizeof(double));
        } else {
            cpd::Rng rng(cfg.seed);
            for (double& v : init) v = rng.normal();
        }
        uint64_t off = 0;
        for (uint32_t k = 0; k < N; ++k) {
            const uint64_t I = c->dims[k];
            A[k].ensure(I * R);
            CPDB_CK(cudaMemcpyAsync(A[k].p, init.data() + off, I * R * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
            if (!init_factors) CPDB_CK(normalize_exact(A[k].p, I, R, nullptr, s));
            off += I * R;
        }
        CPDB_CK(cudaStreamSynchronize(s));
    }
    DevBuf lam, M, fit, reg, uwork, gam, ahat;
    lam.ensure(R);
    {
        std::vector<double> l(R, 1.0);
        if (init_lambda) l.assign(init_lambda, init_lambda + R);
        CPDB_CK(cudaMemcpyAsync(lam.p, l.data(), R * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    uint64_t maxI = 0;
    for (uint64_t d : c->dims) maxI = std::max(maxI, d);
    for (uint32_t k = 0; k < N; ++k) {
        G[k].ensure(uint64_t(R) * R);
        CPDB_CK(gram_dev(A[k].p, c->dims[k], R, G[k].p, s));
        const uint64_t rows = (k == 0 && sharded) ? c->rows : c->dims[k];
        AP[k].ensure(uint64_t(ttm_kpad(rows)) * ttm_rpad(R));
        CPDB_CK(pack_q(A[k].p + ((k == 0 && sharded) ? c->row_begin * R : 0), AP[k].p,
                       uint32_t(rows), R, s));
    }
    M.ensure(maxI * R);
    fit.ensure(8);
    int* dreg = reinterpret_cast<int*>(reg.ensure(1));
    MttkrpBufs bufs;

    cudaEvent_t t0, te;
    CPDB_CK(cudaEventCreate(&t0));
    CPDB_CK(cudaEventCreate(&te));
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } evg{t0, te};
    CPDB_CK(cudaEventRecord(t0, s));

    // MTTKRP kernel flops per mode, as the reference counts them (:164)
    const uint64_t mttkrp_flops = 2ull * numel(c->dims) * R;
    uint64_t flops = 0, rows_out = 0;
    for (uint64_t sweep = 1; sweep <= cfg.max_iterations; ++sweep) {
        CPDB_CK(cudaMemsetAsync(c->dstatus, 0, sizeof(int), s));
        CPDB_CK(cudaMemsetAsync(dreg, 0, sizeof(int), s));
        for (uint32_t n = 0; n < N; ++n) {
            std::vector<const double*> fac(N), qp(N);
            for (uint32_t k = 0; k < N; ++k) {
                fac[k] = A[k].p + ((k == 0 && sharded) ? c->row_begin * R : 0);
                qp[k] = AP[k].p;
            }
            double* m_local = M.p + ((n == 0 && sharded) ? c->row_begin * R : 0);
            mttkrp_dev(c, c->x, c->ldims, fac, qp, R, n, bufs, m_local, s);
            mttkrp_combine(c, n, M.p, R);
            const uint64_t I = c->dims[n];
            const bool last = (n + 1 == N);
            if (als_finish_fits(I, R)) {
                AlsFinishArgs f{};
                f.m = M.p;
                for (uint32_t k = 0; k < N; ++k)
                    if (k != n) f.grams[f.ng++] = G[k].p;
                f.I = I;
                f.R = R;
                f.a_out = A[n].p;
                f.g_out = G[n].p;
                f.lambda = lam.p;
                f.fitness = last ? 1 : 0;
                f.norm_x_sq = nx2;
                f.fit_out = fit.p;
                f.status = c->dstatus;
                f.regularized = dreg;
                CPDB_CK(launch_als_finish(f, s));
                c->launches += 1;
            } else {
                // long modes: Gamma, solve_spd, normalize_columns, gram, fitness
                GramList gl{};
                for (uint32_t k = 0; k < N; ++k)
                    if (k != n) gl.g[gl.n++] = G[k].p;
                double* gp = gam.ensure(uint64_t(R) * R);
                double* ah = ahat.ensure(I * R);
                CPDB_CK(hadamard_dev(gl, R, gp, s));
                CPDB_CK(cudaMemcpyAsync(ah, M.p, I * R * sizeof(double), cudaMemcpyDeviceToDevice,
                                        s));
                const size_t uw = spd_work_doubles(R);
                int* dreg_n = reinterpret_cast<int*>(uwork.ensure(uw + 2)) + 2 * uw;
                CPDB_CK(launch_spd_solve(gp, R, uwork.p, ah, I, c->dstatus, dreg_n, s, c->sms));
                CPDB_CK(cudaMemcpyAsync(A[n].p, ah, I * R * sizeof(double),
                                        cudaMemcpyDeviceToDevice, s));
                CPDB_CK(normalize_exact(A[n].p, I, R, lam.p, s));
                CPDB_CK(gram_dev(A[n].p, I, R, G[n].p, s));
                // fold this mode's ridge flag into the sweep's
                CPDB_CK(launch_or_flag(dreg_n, dreg, s));
                if (last)
                    CPDB_CK(launch_fitness_als(nx2, M.p, ah, I * R, gp, lam.p, G[n].p, R, fit.p,
                                               s));
                c->launches += 7;
            }
            const uint64_t rows = (n == 0 && sharded) ? c->rows : I;
            CPDB_CK(pack_q(A[n].p + ((n == 0 && sharded) ? c->row_begin * R : 0), AP[n].p,
                           uint32_t(rows), R, s));
            c->launches += 1;
            flops += mttkrp_flops;
        }
        CPDB_CK(cudaEventRecord(te, s));
        CPDB_CK(cudaMemcpyAsync(c->pinned, fit.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CPDB_CK(cudaMemcpyAsync(c->pinned + 2, c->dstatus, sizeof(int), cudaMemcpyDeviceToHost, s));
        CPDB_CK(cudaMemcpyAsync(reinterpret_cast<int*>(c->pinned + 2) + 1, dreg, sizeof(int),
                                cudaMemcpyDeviceToHost, s));
        CPDB_CK(cudaStreamSynchronize(s));
        int status, regularized;
        std::memcpy(&status, c->pinned + 2, sizeof(int));
        std::memcpy(&regularized, reinterpret_cast<int*>(c->pinned + 2) + 1, sizeof(int));
        if (status == 5) fail(CPDB_INVALID_ARGUMENT, "solve_spd: G is not symmetric");
        if (status)
            fail(CPDB_SINGULAR_SYSTEM, "solve_spd: factorization failed after ridge");
        float ms = 0.f;
        CPDB_CK(cudaEventElapsedTime(&ms, t0, te));
        const double f = c->pinned[0];
        if (trace) {
            cpdb_trace_row& row = trace[rows_out];
            std::memset(&row, 0, sizeof row);
            row.iteration = sweep;
            row.order = N;
            for (uint32_t k = 0; k < N; ++k) row.update_order[k] = k;
            row.fitness = f;
            row.raw_radicand = c->pinned[1];
            row.wall_seconds = ms * 1e-3;
            row.root_ttm_count = 0;
            row.flops = flops;
            row.beta_used = 0.0;
            row.regularized = regularized ? 1 : 0;
        }
        ++rows_out;
        if (f >= cfg.fitness_threshold) break;  // (:200)
    }
    if (trace_len) *trace_len = rows_out;
    if (out_lambda)
        CPDB_CK(cudaMemcpy(out_lambda, lam.p, R * sizeof(double), cudaMemcpyDeviceToHost));
    if (out_factors) {
        uint64_t off = 0;
        for (uint32_t k = 0; k < N; ++k) {
            CPDB_CK(cudaMemcpy(out_factors + off, A[k].p, c->dims[k] * R * sizeof(double),
                               cudaMemcpyDeviceToHost));
            off += c->dims[k] * R;
        }
    }
}

// ---------------------------------------------------------------- primitives
void mttkrp_primitive(cpdb_ctx* c, const double* x, const std::vector<uint64_t>& dims,
                      const std::vector<const double*>& fac_dev, uint32_t R, uint32_t n,
                      double* m_out) {
    const uint32_t N = uint32_t(dims.size());
    std::vector<DevBuf> AP(N);
    std::vector<const double*> qp(N, nullptr);
    for (uint32_t k = 0; k < N; ++k) {
        if (k == n) continue;
        AP[k].ensure(uint64_t(ttm_kpad(dims[k])) * ttm_rpad(R));
        CPDB_CK(pack_q(fac_dev[k], AP[k].p, uint32_t(dims[k]), R, c->stream));
        qp[k] = AP[k].p;
    }
    MttkrpBufs b;
    mttkrp_dev(c, x, dims, fac_dev, qp, R, n, b, m_out, c->stream);
    CPDB_CK(cudaStreamSynchronize(c->stream));
}

}  // namespace cpdb
