// Device-resident CP-ALS-QR driver (the B200 replacement of detail::run_qr,
// /root/reference/proj/include/cpd/solvers.hpp:215-309).
//
// The host keeps exactly what the reference keeps on the host -- the plan,
// factor versions and cache stamps (freshness is checked before every cached
// read, dim_tree.hpp:506-513), the beta state machine and the stop test --
// and every tensor and matrix lives in HBM.  Per mode update n (solvers.hpp:
// 249-289) the stream carries:
//   launch_zqr     Q0, R0 of Khatri-Rao(R_k, k != n)           (:250-255)
//   launch_ttm...  the scheduled TTM chain, cache in HBM        (:267)
//   launch_vgemm   V = Y_(n) Q0_hat, extrapolation fused        (:258-271,277-284)
//   launch_finish  A_hat, normalise, lambda, factor QR, fitness (:272-275,291)
// and the host synchronises once per sweep to read the fitness scalar.
#include "runtime.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "comm.hpp"
#include "cpd/rng.hpp"

namespace cpdb {

void fail(int code, const std::string& what) { throw Fail{code, what}; }

void check_cuda(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return;
    cudaGetLastError();
    throw Fail{e == cudaErrorMemoryAllocation ? CPDB_OUT_OF_MEMORY : CPDB_CUDA_ERROR,
               std::string(where) + ": " + cudaGetErrorString(e)};
}

DevBuf::~DevBuf() {
    if (p) cudaFree(p);
}

double* DevBuf::ensure(size_t d) {
    if (p && d <= n) return p;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    CPDB_CK(cudaMalloc(&p, std::max<size_t>(d, 1) * sizeof(double)));
    n = std::max<size_t>(d, 1);
    return p;
}

uint64_t numel(const std::vector<uint64_t>& d) {
    uint64_t n = 1;
    for (uint64_t v : d) n *= v;
    return n;
}

void require_tensor(cpdb_ctx* c) {
    if (!c->x) fail(CPDB_INVALID_ARGUMENT, "no tensor set on this context (cpdb_tensor_set)");
}

void allreduce_sum(cpdb_ctx* c, double* dev, size_t n) {
    if (c->world <= 1) return;
    const Nccl& N = nccl();
    const ncclResult_t r =
        N.AllReduce(dev, dev, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->comm), c->stream);
    if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, std::string("ncclAllReduce: ") + N.GetErrorString(r));
}

void allgather(cpdb_ctx* c, double* dev_full, size_t per_rank) {
    if (c->world <= 1) return;
    const Nccl& N = nccl();
    const ncclResult_t r = N.AllGather(dev_full + per_rank * c->rank, dev_full, per_rank,
                                       ncclDouble, static_cast<ncclComm_t>(c->comm), c->stream);
    if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, std::string("ncclAllGather: ") + N.GetErrorString(r));
}

double ctx_norm_sq(cpdb_ctx* c) {
    require_tensor(c);
    if (c->norm_valid) return c->norm_x_sq;
    double* part = c->partials.ensure(kNormBlocks + 8);
    CPDB_CK(norm_sq(c->x, numel(c->ldims), part, part + kNormBlocks, c->stream));
    c->launches += 2;
    allreduce_sum(c, part + kNormBlocks, 1);
    CPDB_CK(cudaMemcpyAsync(c->pinned, part + kNormBlocks, sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
    CPDB_CK(cudaStreamSynchronize(c->stream));
    c->norm_x_sq = c->pinned[0];
    c->norm_valid = true;
    return c->norm_x_sq;
}

std::vector<uint64_t> natural_to_reference(uint32_t order, uint64_t R) {
    const uint32_t m = order - 1;
    uint64_t rows = 1;
    for (uint32_t t = 0; t < m; ++t) rows *= R;
    std::vector<uint64_t> perm(rows);
    for (uint64_t nat = 0; nat < rows; ++nat) {
        uint64_t rem = nat, ref = 0, w = 1;
        // nat: digit t=0 slowest; ref: digit t=0 fastest
        std::vector<uint64_t> d(m);
        for (uint32_t t = m; t-- > 0;) {
            d[t] = rem % R;
            rem /= R;
        }
        for (uint32_t t = 0; t < m; ++t) {
            ref += d[t] * w;
            w *= R;
        }
        perm[nat] = ref;
    }
    return perm;
}

void run_ttm(cpdb_ctx* ctx, const double* src, const std::vector<uint64_t>& sd, uint32_t c,
             const double* q, const double* qp, uint32_t R, double* dst) {
    TtmArgs a{};
    a.x = src;
    a.y = dst;
    a.q = q;
    a.qp = qp;
    a.outer = 1;
    a.inner = 1;
    for (uint32_t k = 0; k < c; ++k) a.outer *= sd[k];
    for (uint32_t k = c + 1; k < sd.size(); ++k) a.inner *= sd[k];
    a.K = sd[c];
    a.R = R;
    a.Rp = ttm_rpad(R);
    CPDB_CK(launch_ttm(a, ctx->stream, ctx->sms));
    ctx->launches += 1;
}

namespace {

struct FactorBufs {
    DevBuf a, q, qp, r;
};

struct EventPool {
    std::vector<cudaEvent_t> free_, used;
    cudaEvent_t get() {
        cudaEvent_t e;
        if (!free_.empty()) {
            e = free_.back();
            free_.pop_back();
        } else {
            CPDB_CK(cudaEventCreate(&e));
        }
        used.push_back(e);
        return e;
    }
    void recycle() {
        free_.insert(free_.end(), used.begin(), used.end());
        used.clear();
    }
    ~EventPool() {
        for (auto e : free_) cudaEventDestroy(e);
        for (auto e : used) cudaEventDestroy(e);
    }
};

std::string set_name(uint32_t s, uint32_t order) {
    std::string out = "Y(";
    bool first = true;
    for (uint32_t m = 0; m < order; ++m)
        if (s & (1u << m)) {
            if (!first) out += ',';
            out += std::to_string(m + 1);
            first = false;
        }
    return out + ")";
}

}  // namespace

void solve(cpdb_ctx* c, const cpdb_config& cfg, cpdb_state* state, cpdb_trace_row* trace,
           uint64_t* trace_len, double* out_lambda, double* out_factors, double* fps,
           double* lps, cpdb_q0_observer observer, void* user) {
    // ---- SolverConfig::validate (solvers.hpp:41-49) and run_qr guards (:217-224)
    if (cfg.rank == 0) fail(CPDB_INVALID_ARGUMENT, "SolverConfig: rank must be >= 1");
    if (cfg.max_iterations == 0)
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: need at least one iteration");
    if (!(cfg.fitness_threshold >= 0.0 && cfg.fitness_threshold <= 1.0))
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: fitness threshold must be in [0,1]");
    if (!std::isfinite(cfg.alpha) || !std::isfinite(cfg.activation_gap))
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: alpha and activation gap must be finite");
    if (cfg.strategy < 0 || cfg.strategy > 2) fail(CPDB_INVALID_ARGUMENT, "unknown strategy");
    require_tensor(c);
    const uint32_t order = static_cast<uint32_t>(c->dims.size());
    if (order < 2) fail(CPDB_INVALID_ARGUMENT, "cp_als_qr: tensor order must be >= 2");
    if (order > CPDB_MAX_ORDER) fail(CPDB_INVALID_ARGUMENT, "cp_als_qr: order above 8");
    const double nx2 = ctx_norm_sq(c);
    if (nx2 == 0.0) fail(CPDB_INVALID_ARGUMENT, "cp_als_qr: zero-norm tensor");
    const uint32_t R = static_cast<uint32_t>(cfg.rank);
    for (uint32_t k = 0; k < order; ++k)
        if (cfg.rank > c->dims[k])
            fail(CPDB_INVALID_ARGUMENT,
                 "cp_als_qr: rank must not exceed any mode extent (compact QR)");
    if (R > 64) fail(CPDB_INVALID_ARGUMENT, "cp_als_qr: rank above 64 is not supported on the device path");
    const bool extrap = cfg.extrapolate != 0;
    const Strategy strategy = extrap ? Strategy::branch_reuse : static_cast<Strategy>(cfg.strategy);
    const uint64_t done = state ? state->sweeps_done : 0;
    Plan plan;
    try {
        plan = build_plan(order, strategy, done + cfg.max_iterations);
    } catch (const SchedError& e) {
        fail(e.code, e.what);
    }
    const bool sharded = c->world > 1;
    cudaStream_t s = c->stream;
    const uint32_t Rp = ttm_rpad(R);
    uint64_t zrows = 1;
    for (uint32_t k = 1; k < order; ++k) zrows *= R;
    uint64_t maxI = 0;
    for (uint64_t d : c->dims) maxI = std::max(maxI, d);
    uint64_t nfac = 0;
    for (uint64_t d : c->dims) nfac += d * R;

    c->prof = cpdb_profile{};
    const uint64_t launches0 = c->launches;

    // ---- factor state (factor_state.hpp:28-34) -----------------------------
    std::vector<FactorBufs> fb(order);
    for (uint32_t k = 0; k < order; ++k) {
        const uint64_t I = c->dims[k];
        fb[k].a.ensure(I * R);
        fb[k].q.ensure(I * R);
        fb[k].qp.ensure(uint64_t(ttm_kpad(I)) * Rp);
        fb[k].r.ensure(uint64_t(R) * R);
    }
    DevBuf lam;
    lam.ensure(R);
    {
        std::vector<double> init(nfac);
        if (state && state->factors) {
            std::memcpy(init.data(), state->factors, nfac * sizeof(double));
        } else {
            cpd::Rng rng(cfg.seed);  // solvers.hpp:116-122
            for (double& v : init) v = rng.normal();
        }
        uint64_t off = 0;
        for (uint32_t k = 0; k < order; ++k) {
            const uint64_t I = c->dims[k];
            CPDB_CK(cudaMemcpyAsync(fb[k].a.p, init.data() + off, I * R * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
            if (!(state && state->factors)) {
                CPDB_CK(normalize_exact(fb[k].a.p, I, R, nullptr, s));
                c->launches += 1;
            }
            off += I * R;
        }
        std::vector<double> l(R, 1.0);
        if (state && state->lambda) l.assign(state->lambda, state->lambda + R);
        CPDB_CK(cudaMemcpyAsync(lam.p, l.data(), R * sizeof(double), cudaMemcpyHostToDevice, s));
        CPDB_CK(cudaStreamSynchronize(s));
    }
    DevBuf fscratch, vpart, vfitpart, vfull, vfitfull, vout, fitbuf, q0buf, q1buf, r0buf, zwork;
    fscratch.ensure(maxI * (R + 1));
    vout.ensure(maxI * R);
    fitbuf.ensure(8);
    q0buf.ensure(zrows * R);
    q1buf.ensure(zrows * R);
    r0buf.ensure(uint64_t(R) * R);
    zwork.ensure(zqr_work_doubles(R) + uint64_t(4 * c->sms) * R * R);
    vfull.ensure(maxI * R);
    vfitfull.ensure(maxI * R);
    std::vector<uint64_t> versions(order, 1);

    CPDB_CK(cudaMemsetAsync(c->dstatus, 0, sizeof(int), s));
    auto qr_factor = [&](uint32_t k) {
        FinishArgs f{};
        f.init = 1;
        f.I = c->dims[k];
        f.R = R;
        f.a_out = fb[k].a.p;
        f.q_out = fb[k].q.p;
        f.qp_out = fb[k].qp.p;
        f.r_out = fb[k].r.p;
        f.lambda = lam.p;
        f.scratch = fscratch.p;
        f.status = c->dstatus;
        f.v_out = vout.p;
        CPDB_CK(launch_finish(f, s));
        c->launches += 1;
    };
    for (uint32_t k = 0; k < order; ++k) qr_factor(k);
    // Sharded runs contract the leading mode with this rank's rows of Q_0
    // only; they get their own packed copy (no row-alignment constraint).
    DevBuf qp0_local;
    auto pack_local0 = [&]() {
        if (!sharded) return;
        qp0_local.ensure(uint64_t(ttm_kpad(c->rows)) * Rp);
        CPDB_CK(pack_q(fb[0].q.p + c->row_begin * R, qp0_local.p, uint32_t(c->rows), R, s));
        c->launches += 1;
    };
    pack_local0();

    // ---- Q0 history (reference row order on the host side) -----------------
    const std::vector<uint64_t> perm = natural_to_reference(order, R);
    std::vector<DevBuf> hist(order);
    std::vector<bool> has_hist(order, false);
    for (uint32_t n = 0; n < order; ++n) hist[n].ensure(zrows * R);
    if (state && state->q0_history) {
        std::vector<double> nat(zrows * R);
        for (uint32_t n = 0; n < order; ++n) {
            if (!(state->history_mask & (1u << n))) continue;
            const double* ref = state->q0_history + uint64_t(n) * zrows * R;
            for (uint64_t i = 0; i < zrows; ++i)
                std::memcpy(&nat[i * R], ref + perm[i] * R, R * sizeof(double));
            CPDB_CK(cudaMemcpyAsync(hist[n].p, nat.data(), zrows * R * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
            CPDB_CK(cudaStreamSynchronize(s));
            has_hist[n] = true;
        }
    }
    bool has_beta = false;
    double beta = 0.0;
    if (extrap && cfg.has_beta_override) {
        has_beta = true;
        beta = cfg.beta_override;
    }
    if (extrap && state && state->has_active_beta && !has_beta) {
        has_beta = true;
        beta = state->active_beta;
    }
    bool has_prev = state && state->has_prev_fitness;
    double prev_fit = has_prev ? state->prev_fitness : 0.0;

    // ---- cost accounting (dim_tree.hpp:523-526) -------------------------------
    Cost total = done > 0 ? measured_cost(plan, c->dims, R, done) : Cost{};

    // ---- the intermediate cache ---------------------------------------------
    std::map<uint32_t, Slot> cache;
    const uint32_t root = plan.root();
    auto local_dims_of = [&](uint32_t key) {
        std::vector<uint64_t> d(order);
        for (uint32_t k = 0; k < order; ++k) d[k] = (key & (1u << k)) ? c->ldims[k] : R;
        return d;
    };
    auto q_rows_for = [&](uint32_t k, bool src_sharded, const double*& q, const double*& qp) {
        q = fb[k].q.p;
        qp = fb[k].qp.p;
        if (k == 0 && src_sharded) {
            q += c->row_begin * R;
            qp = qp0_local.p;
        }
    };
    EventPool events;
    std::vector<Timer> timers;
    auto ttm_step = [&](const double* src, const std::vector<uint64_t>& sd, bool src_sharded,
                        uint32_t k, double* dst, bool is_root) {
        const double* q;
        const double* qp;
        q_rows_for(k, src_sharded, q, qp);
        Timer t;
        if (c->timing) {
            t.a = events.get();
            t.b = events.get();
            t.kind = is_root ? 0 : 1;
            CPDB_CK(cudaEventRecord(t.a, s));
        }
        run_ttm(c, src, sd, k, q, qp, R, dst);
        if (c->timing) {
            CPDB_CK(cudaEventRecord(t.b, s));
            const uint64_t nin = numel(sd);
            const uint64_t nout = nin / sd[k] * R;
            t.flops = 2.0 * double(nout) * double(sd[k]);
            t.bytes = 8.0 * (double(nin) + double(nout) + double(sd[k]) * R);
            timers.push_back(t);
        }
        if (src_sharded && k == 0 && sharded) {
            Timer tc;
            if (c->timing) {
                tc.a = events.get();
                tc.b = events.get();
                tc.kind = 2;
                CPDB_CK(cudaEventRecord(tc.a, s));
            }
            allreduce_sum(c, dst, numel(sd) / sd[k] * R);
            if (c->timing) {
                CPDB_CK(cudaEventRecord(tc.b, s));
                timers.push_back(tc);
            }
        }
    };
    if (done > 0) {
        // rebuild the retained intermediates from X and the current factors
        for (uint32_t key : retained_keys(plan, done - 1, order - 1)) {
            if (cache.count(key)) continue;
            std::vector<uint64_t> d = c->ldims;
            const double* cur = c->x;
            bool cur_sharded = sharded;
            DevBuf tmp[2];
            int w = 0;
            for (uint32_t k = order; k-- > 0;) {
                if (key & (1u << k)) continue;
                std::vector<uint64_t> nd = d;
                nd[k] = R;
                double* out = tmp[w].ensure(numel(nd));
                ttm_step(cur, d, cur_sharded, k, out, cur == c->x);
                if (k == 0) cur_sharded = false;
                cur = out;
                d = nd;
                w ^= 1;
            }
            Slot& sl = cache[key];
            sl.buf.ensure(numel(d));
            CPDB_CK(cudaMemcpyAsync(sl.buf.p, cur, numel(d) * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
            sl.valid = true;
            sl.dims = d;
            sl.sharded = sharded && (key & 1u);
            sl.stamps.assign(order, 0);
            for (uint32_t k = 0; k < order; ++k)
                if (!(key & (1u << k))) sl.stamps[k] = versions[k];
            CPDB_CK(cudaStreamSynchronize(s));
        }
        events.recycle();
        timers.clear();
    }

    std::vector<DevBuf> ybuf(order);
    for (uint32_t n = 0; n < order; ++n) ybuf[n].ensure(numel(local_dims_of(1u << n)));

    struct StartEvent {
        cudaEvent_t e = nullptr;
        ~StartEvent() {
            if (e) cudaEventDestroy(e);
        }
    } start;
    CPDB_CK(cudaEventCreate(&start.e));
    const cudaEvent_t t_start = start.e;
    CPDB_CK(cudaEventRecord(t_start, s));
    uint64_t rows_out = 0;
    double last_ms = 0.0;
    for (uint64_t sweep = done + 1; sweep <= done + cfg.max_iterations; ++sweep) {
        const Sweep& sw = plan.sweeps[sweep - 1];
        double beta_used = 0.0;
        CPDB_CK(cudaMemsetAsync(c->dstatus, 0, sizeof(int), s));
        for (uint32_t b = 0; b < order; ++b) {
            const uint32_t n = sw.updates[b].mode;
            const bool last = (b == order - 1);
            // 1-2. Khatri-Rao + QR of the other R_k -> Q0, R0 (solvers.hpp:250-255)
            ZqrArgs z{};
            uint32_t t = 0;
            for (uint32_t k = 0; k < order; ++k)
                if (k != n) z.rmats[t++] = fb[k].r.p;
            z.nm = order - 1;
            z.R = R;
            z.zrows = zrows;
            z.q1 = q1buf.p;
            z.q0 = q0buf.p;
            z.r0 = r0buf.p;
            z.work = zwork.p;
            z.status = c->dstatus;
            CPDB_CK(launch_zqr(z, s, c->sms));
            c->launches += 4;
            if (observer) {
                std::vector<double> nat(zrows * R), ref(zrows * R);
                CPDB_CK(cudaMemcpyAsync(nat.data(), q0buf.p, zrows * R * sizeof(double),
                                        cudaMemcpyDeviceToHost, s));
                CPDB_CK(cudaStreamSynchronize(s));
                for (uint64_t i = 0; i < zrows; ++i)
                    std::memcpy(&ref[perm[i] * R], &nat[i * R], R * sizeof(double));
                observer(user, sweep, n, ref.data(), zrows, R);
            }
            // 3. extrapolation gate (solvers.hpp:260-265)
            const bool use_ex = extrap && has_beta && beta != 0.0 && has_hist[n];
            if (use_ex) beta_used = beta;

            // 4. the scheduled TTM chain (execute, dim_tree.hpp:496-541)
            for (const Step& st : sw.updates[b].steps) {
                const double* src;
                std::vector<uint64_t> sd;
                std::vector<uint64_t> stamp(order, 0);
                bool src_sh;
                if (st.source == root) {
                    src = c->x;
                    sd = c->ldims;
                    src_sh = sharded;
                } else {
                    auto it = cache.find(st.source);
                    if (it == cache.end() || !it->second.valid)
                        fail(CPDB_LOGIC_ERROR, "execute: scheduled source " +
                                                   set_name(st.source, order) +
                                                   " missing from cache");
                    for (uint32_t m = 0; m < order; ++m)
                        if (it->second.stamps[m] && it->second.stamps[m] != versions[m])
                            fail(CPDB_STALE_INTERMEDIATE,
                                 "execute: stale intermediate " + set_name(st.source, order));
                    src = it->second.buf.p;
                    sd = it->second.dims;
                    stamp = it->second.stamps;
                    src_sh = it->second.sharded;
                }
                std::vector<uint64_t> od = sd;
                od[st.contract] = R;
                double* dst;
                if (st.produces == (1u << n)) {
                    dst = ybuf[n].p;
                } else {
                    Slot& sl = cache[st.produces];
                    dst = sl.buf.ensure(numel(od));
                }
                ttm_step(src, sd, src_sh, st.contract, dst, st.source == root);
                // global-extent flop count, as the reference counts it
                uint64_t gout = 1;
                for (uint32_t k = 0; k < order; ++k)
                    gout *= (st.produces & (1u << k)) ? c->dims[k] : uint64_t(R);
                total.flops += 2ull * gout * c->dims[st.contract];
                if (st.source == root) ++total.roots;
                stamp[st.contract] = versions[st.contract];
                if (st.produces != (1u << n)) {
                    Slot& sl = cache[st.produces];
                    sl.valid = true;
                    sl.dims = od;
                    sl.stamps = stamp;
                    sl.sharded = src_sh && st.contract != 0;
                }
            }
            const std::vector<ModeSet> keep = retained_keys(plan, sweep - 1, b);
            for (auto& kv : cache)
                if (std::find(keep.begin(), keep.end(), kv.first) == keep.end()) kv.second.valid = false;

            // 5. V = Y_(n) Q0_hat (+ unextrapolated V for the fitness)
            const std::vector<uint64_t> yd = local_dims_of(1u << n);
            VgemmArgs v{};
            v.y = ybuf[n].p;
            v.q0 = q0buf.p;
            v.hist = use_ex ? hist[n].p : nullptr;
            v.beta = beta;
            v.alpha = cfg.alpha;
            v.extrap = use_ex ? 1 : 0;
            v.dual = (last && use_ex) ? 1 : 0;
            v.I = yd[n];
            v.O = 1;
            for (uint32_t k = 0; k < n; ++k) v.O *= R;
            v.J = 1;
            for (uint32_t k = n + 1; k < order; ++k) v.J *= R;
            v.R = R;
            const size_t part = size_t(vgemm_max_split()) * v.I * R;
            v.vpart = vpart.ensure(part);
            v.vfitpart = v.dual ? vfitpart.ensure(part) : nullptr;
            CPDB_CK(launch_vgemm(v, s, c->sms));
            c->launches += 1;
            const double* vsrc = v.vpart;
            const double* vfsrc = v.vfitpart;
            uint32_t nsplit = v.nsplit;
            if (sharded && n == 0) {
                // local rows of V -> gather the full V on every rank
                CPDB_CK(reduce_splits(v.vpart, nsplit, v.I * R, vfull.p + c->row_begin * R, s));
                allgather(c, vfull.p, v.I * R);
                vsrc = vfull.p;
                if (v.dual) {
                    CPDB_CK(reduce_splits(v.vfitpart, nsplit, v.I * R,
                                          vfitfull.p + c->row_begin * R, s));
                    allgather(c, vfitfull.p, v.I * R);
                    vfsrc = vfitfull.p;
                }
                c->launches += v.dual ? 2 : 1;
                nsplit = 1;
            }
            // 6-9. A_hat, lambda, factor QR, fitness (solvers.hpp:272-292)
            FinishArgs f{};
            f.init = 0;
            f.vpart = vsrc;
            f.vfitpart = vfsrc;
            f.nsplit = nsplit;
            f.dual = v.dual;
            f.r0 = r0buf.p;
            f.I = c->dims[n];
            f.R = R;
            f.v_out = vout.p;
            f.a_out = fb[n].a.p;
            f.q_out = fb[n].q.p;
            f.qp_out = fb[n].qp.p;
            f.r_out = fb[n].r.p;
            f.lambda = lam.p;
            f.scratch = fscratch.p;
            f.fitness = last ? 1 : 0;
            f.norm_x_sq = nx2;
            f.fit_out = fitbuf.p;
            f.status = c->dstatus;
            CPDB_CK(launch_finish(f, s));
            c->launches += 1;
            if (n == 0) pack_local0();
            ++versions[n];
            if (extrap) {
                hist[n].swap(q0buf);  // history keeps the unextrapolated Q0
                has_hist[n] = true;
            }
        }
        cudaEvent_t e_end = events.get();
        CPDB_CK(cudaEventRecord(e_end, s));
        CPDB_CK(cudaMemcpyAsync(c->pinned, fitbuf.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CPDB_CK(cudaMemcpyAsync(c->pinned + 2, c->dstatus, sizeof(int), cudaMemcpyDeviceToHost, s));
        CPDB_CK(cudaStreamSynchronize(s));
        int status;
        std::memcpy(&status, c->pinned + 2, sizeof(int));
        if (status) {
            if ((status & 0xFF) == 1)
                fail(CPDB_SINGULAR_TRIANGULAR,
                     "triangular solve: diagonal entry of column " + std::to_string(status >> 8) +
                         " is ~0 (rank-deficient Khatri-Rao factor)");
            fail(CPDB_SINGULAR_TRIANGULAR,
                 "Cholesky QR breakdown: rank-deficient Khatri-Rao or factor matrix");
        }
        const double fit = c->pinned[0], raw = c->pinned[1];
        float ms = 0.f;
        CPDB_CK(cudaEventElapsedTime(&ms, t_start, e_end));
        if (sweep == done + 1) c->prof.sweep1_ms = ms;
        last_ms = ms;
        for (const Timer& t : timers) {
            float tm = 0.f;
            CPDB_CK(cudaEventElapsedTime(&tm, t.a, t.b));
            if (t.kind == 0) {
                c->prof.root_ttms += 1;
                c->prof.root_ttm_ms += tm;
                c->prof.root_ttm_flops += t.flops;
                c->prof.root_ttm_bytes += t.bytes;
            } else if (t.kind == 1) {
                c->prof.branch_ttm_ms += tm;
            } else {
                c->prof.comm_ms += tm;
            }
        }
        timers.clear();
        if (trace) {
            cpdb_trace_row& row = trace[rows_out];
            std::memset(&row, 0, sizeof row);
            row.iteration = sweep;
            row.order = order;
            for (uint32_t b = 0; b < order; ++b) row.update_order[b] = sw.updates[b].mode;
            row.fitness = fit;
            row.raw_radicand = raw;
            row.wall_seconds = ms * 1e-3;
            row.root_ttm_count = total.roots;
            row.flops = total.flops;
            row.beta_used = beta_used;
        }
        if (fps) {
            uint64_t off = 0;
            for (uint32_t k = 0; k < order; ++k) {
                CPDB_CK(cudaMemcpy(fps + rows_out * nfac + off, fb[k].a.p,
                                   c->dims[k] * R * sizeof(double), cudaMemcpyDeviceToHost));
                off += c->dims[k] * R;
            }
        }
        if (lps)
            CPDB_CK(cudaMemcpy(lps + rows_out * R, lam.p, R * sizeof(double), cudaMemcpyDeviceToHost));
        ++rows_out;
        // beta gate (solvers.hpp:297-300)
        if (extrap && !has_beta && !cfg.has_beta_override && sweep >= 2 && has_prev) {
            const double cl_prev = prev_fit < 0.0 ? 0.0 : (prev_fit > 1.0 ? 1.0 : prev_fit);
            const double cl_now = fit < 0.0 ? 0.0 : (fit > 1.0 ? 1.0 : fit);
            if (!(std::fabs(cl_now - cl_prev) >= cfg.activation_gap)) {
                has_beta = true;
                beta = cl_now > 0.90 ? 1.0 / 2000.0 : (cl_now >= 0.70 ? 1.0 / 500.0 : 1.0 / 250.0);
            }
        }
        prev_fit = fit;
        has_prev = true;
        events.recycle();
        if (fit >= cfg.fitness_threshold) break;
    }
    c->prof.sweeps = rows_out;
    c->prof.solve_ms = last_ms;
    c->prof.mode_update_ms = last_ms - c->prof.root_ttm_ms - c->prof.branch_ttm_ms - c->prof.comm_ms;
    c->prof.kernel_launches = c->launches - launches0;
    if (trace_len) *trace_len = rows_out;

    auto get_factors = [&](double* dst) {
        uint64_t off = 0;
        for (uint32_t k = 0; k < order; ++k) {
            CPDB_CK(cudaMemcpy(dst + off, fb[k].a.p, c->dims[k] * R * sizeof(double),
                               cudaMemcpyDeviceToHost));
            off += c->dims[k] * R;
        }
    };
    if (out_lambda) CPDB_CK(cudaMemcpy(out_lambda, lam.p, R * sizeof(double), cudaMemcpyDeviceToHost));
    if (out_factors) get_factors(out_factors);
    if (state) {
        state->sweeps_done = done + rows_out;
        if (state->lambda)
            CPDB_CK(cudaMemcpy(state->lambda, lam.p, R * sizeof(double), cudaMemcpyDeviceToHost));
        if (state->factors) get_factors(state->factors);
        if (state->q0_history) {
            state->history_mask = 0;
            std::vector<double> nat(zrows * R);
            for (uint32_t n = 0; n < order; ++n) {
                if (!has_hist[n]) continue;
                CPDB_CK(cudaMemcpy(nat.data(), hist[n].p, zrows * R * sizeof(double),
                                   cudaMemcpyDeviceToHost));
                double* ref = state->q0_history + uint64_t(n) * zrows * R;
                for (uint64_t i = 0; i < zrows; ++i)
                    std::memcpy(ref + perm[i] * R, &nat[i * R], R * sizeof(double));
                state->history_mask |= 1u << n;
            }
        }
        state->has_active_beta = has_beta ? 1 : 0;
        state->active_beta = has_beta ? beta : 0.0;
        state->has_prev_fitness = has_prev ? 1 : 0;
        state->prev_fitness = has_prev ? prev_fit : 0.0;
    }
}

}  // namespace cpdb

cpdb_ctx::~cpdb_ctx() {
    if (stream) cudaStreamSynchronize(stream);
    if (comm) {
        const cpdb::Nccl& N = cpdb::nccl();
        if (N.ok) N.CommDestroy(static_cast<ncclComm_t>(comm));
    }
    if (dstatus) cudaFree(dstatus);
    if (pinned) cudaFreeHost(pinned);
    if (stream) cudaStreamDestroy(stream);
}
