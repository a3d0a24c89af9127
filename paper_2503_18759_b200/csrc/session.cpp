// The device-resident CP-ALS-QR driver (B200 replacement of detail::run_qr,
// /root/reference/proj/include/cpd/solvers.hpp:215-309) as a resumable
// session: begin() is the run_qr setup (:217-241), run(n) executes n sweeps of
// the loop (:243-302), end() returns the model (:304-308) and the
// sweep-boundary state.  cpdb_solve = begin + run(max_iterations) + end.
//
// The host keeps exactly what the reference keeps on the host -- the plan,
// factor versions and cache stamps (freshness is checked before every cached
// read, dim_tree.hpp:506-513), the beta state machine and the stop test --
// and every tensor and matrix lives in HBM.  Per mode update n (solvers.hpp:
// 249-289) the stream carries
//   launch_zqr     Q0, R0 of Khatri-Rao(R_k, k != n)           (:250-255)
//   launch_ttm...  the scheduled TTM chain, cache in HBM        (:267)
//   launch_vgemm   V = Y_(n) Q0_hat, extrapolation fused        (:258-271,277-284)
//   launch_finish  A_hat, normalise, lambda, factor QR, fitness (:272-275,291)
// and the host reads one fitness scalar per sweep.
//
// Streams and ordering (unsharded; sharded runs keep the simple form:
// Z-QR on `side`, chain + collectives + tail on `stream`):
//   stream (main, high)  V-GEMM, finisher, beta gate; the Z-QR of an update
//                        whose mode differs from the previous one (launched
//                        programmatically right behind that finisher)
//   side   (high - 1)    chains (below the latency-bound kernels)
//   zq     (high)        the Z-QR of a sweep-boundary update
//   mid    (high - 1)    the chain of a sweep-boundary update (waits only for
//                        its cached source, not for the previous chain)
//   aux    (high)        the next sweep's first V-GEMM + finisher, issued
//                        before the host reads this sweep's fitness (third
//                        order: and the second update's Z-QR right behind)
//   lo     (low)         the prefetched root TTM (prefetch_root /
//                        launch_prefetch), two tiles per CTA (one if short)
// Dependencies are explicit events: ev_fac[k] (the finisher that last
// changed A_k/Q_k/R_k), ev_v[2n+p] (the V-GEMM that last read ybuf[2n+p]),
// ev_zread[p] (last readers of Z-QR buffer set p), ev_zq / ev_zqr (this
// update's Z-QR / chain done), ev_hist[n] (the Z-QR that produced the Q0
// history of mode n), slot_ready (a cache slot's producer), pf.ev
// (prefetched root done).  Buffers that
// consecutive updates may touch concurrently are doubled (factors + lambda,
// Z-QR outputs, Y_(n), V partials, scratch), so a speculative update can be
// undone by swapping back (undo_speculative_update).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "comm.hpp"
#include "prims.hpp"
#include "cpd/rng.hpp"
#include "runtime.hpp"
#include "session.hpp"

namespace cpdb {

static const char* const kBreakdownMessage =
    "Cholesky QR breakdown: rank-deficient Khatri-Rao or factor matrix";
namespace {

// Stream/event calls of the session go through these so the happens-before
// checker (hb.hpp, CPDB_HBCHECK=1) sees the same ordering the GPU does.
inline cudaError_t hb_rec(HbCheck& h, cudaEvent_t e, cudaStream_t s) {
    h.record(e, s);
    return cudaEventRecord(e, s);
}
inline cudaError_t hb_wait(HbCheck& h, cudaStream_t s, cudaEvent_t e, unsigned f) {
    h.wait(s, e);
    return cudaStreamWaitEvent(s, e, f);
}
inline cudaError_t hb_ssync(HbCheck& h, cudaStream_t s) {
    cudaError_t r = cudaStreamSynchronize(s);
    h.sync_stream(s);
    return r;
}
inline cudaError_t hb_esync(HbCheck& h, cudaEvent_t e) {
    cudaError_t r = cudaEventSynchronize(e);
    h.sync_event(e);
    return r;
}
inline cudaError_t hb_dsync(HbCheck& h) {
    cudaError_t r = cudaDeviceSynchronize();
    h.sync_all();
    return r;
}
#define cudaEventRecord(e, st) ::cpdb::hb_rec(hb, (e), (st))
#define cudaStreamWaitEvent(st, e, f) ::cpdb::hb_wait(hb, (st), (e), (f))
#define cudaStreamSynchronize(st) ::cpdb::hb_ssync(hb, (st))
#define cudaEventSynchronize(e) ::cpdb::hb_esync(hb, (e))
#define cudaDeviceSynchronize() ::cpdb::hb_dsync(hb)
using Rg = HbCheck::Rg;
inline Rg rg(const void* p, uint64_t doubles) { return Rg{p, size_t(doubles) * sizeof(double)}; }

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

cudaEvent_t EventPool::get() {
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

void EventPool::recycle() {
    free_.insert(free_.end(), used.begin(), used.end());
    used.clear();
}

void EventPool::recycle_prefix(size_t n) {
    n = std::min(n, used.size());
    free_.insert(free_.end(), used.begin(), used.begin() + long(n));
    used.erase(used.begin(), used.begin() + long(n));
}

EventPool::~EventPool() {
    for (auto e : free_) cudaEventDestroy(e);
    for (auto e : used) cudaEventDestroy(e);
}

Session::~Session() {
    if (c && c->stream) cudaStreamSynchronize(c->stream);
    if (c && c->side) cudaStreamSynchronize(c->side);
    if (c && c->side_hi) cudaStreamSynchronize(c->side_hi);
    if (c && c->lo) cudaStreamSynchronize(c->lo);
    if (c && c->mid) cudaStreamSynchronize(c->mid);
    if (c && c->aux) cudaStreamSynchronize(c->aux);
    if (c && c->zq) cudaStreamSynchronize(c->zq);
    if (c && c->tailq) cudaStreamSynchronize(c->tailq);
    if (ev_fin) cudaEventDestroy(ev_fin);
    if (pf.ev) cudaEventDestroy(pf.ev);
    if (t_start) cudaEventDestroy(t_start);
    if (ev_ready) cudaEventDestroy(ev_ready);
    if (ev_zqr) cudaEventDestroy(ev_zqr);
    if (ev_zq) cudaEventDestroy(ev_zq);
    if (ev_aux) cudaEventDestroy(ev_aux);
    if (ev_tail) cudaEventDestroy(ev_tail);
    for (cudaEvent_t e : ev_fac)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_v)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_zread)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_zread_b)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_v_b)
        if (e) cudaEventDestroy(e);
    for (auto& kv : slot_ready) cudaEventDestroy(kv.second);
    for (cudaEvent_t e : ev_hist)
        if (e) cudaEventDestroy(e);
    if (ev_zq_pending) cudaEventDestroy(ev_zq_pending);
}

// ---------------------------------------------------------------- timeline
cudaEvent_t Session::tl_begin(cudaStream_t st) {
    if (!timeline) return nullptr;
    cudaEvent_t a;
    CPDB_CK(cudaEventCreate(&a));
    CPDB_CK(cudaEventRecord(a, st));
    return a;
}

void Session::tl_end(cudaEvent_t a, cudaStream_t st, const char* label) {
    if (!timeline) return;
    cudaEvent_t b;
    CPDB_CK(cudaEventCreate(&b));
    CPDB_CK(cudaEventRecord(b, st));
    const int sid = st == side ? 1 : st == c->lo ? 2 : st == c->mid ? 3 : st == c->aux ? 4 : st == c->zq ? 5 : st == c->tailq ? 6 : 0;
    marks.push_back(Mark{label, sid, tl_sweep, tl_mode, a, b});
}

void Session::tl_flush() {
    if (!timeline || marks.empty()) return;
    CPDB_CK(cudaDeviceSynchronize());
    FILE* f = std::fopen(timeline, "a");
    for (const Mark& m : marks) {
        float t0 = 0.f, t1 = 0.f;
        CPDB_CK(cudaEventElapsedTime(&t0, t_start, m.a));
        CPDB_CK(cudaEventElapsedTime(&t1, t_start, m.b));
        if (f)
            std::fprintf(f, "%s,%d,%llu,%u,%.2f,%.2f\n", m.label, m.stream,
                         (unsigned long long)m.sweep, m.mode, t0 * 1e3, t1 * 1e3);
        cudaEventDestroy(m.a);
        cudaEventDestroy(m.b);
    }
    if (f) std::fclose(f);
    marks.clear();
}

// ---------------------------------------------------------------- setup
void Session::begin(cpdb_ctx* ctx, const cpdb_config& config, const cpdb_state* state) {
    c = ctx;
    cfg = config;
    {
        const char* e = std::getenv("CPDB_HBCHECK");
        hb.on = e && e[0] == '1';
        if (hb.on) {
            hb.name(c->stream, "main");
            hb.name(c->side, "side");
            hb.name(c->side_hi, "side_hi");
            hb.name(c->lo, "lo");
            hb.name(c->mid, "mid");
            hb.name(c->aux, "aux");
            hb.name(c->zq, "zq");
            hb.name(c->tailq, "tailq");
            hb.name(nullptr, "legacy");
        }
        fpath = std::getenv("CPDB_FINGERPRINT");
        fp_light = std::getenv("CPDB_FINGERPRINT_LIGHT") != nullptr;
        if (fpath) {
            fplog.ensure(1u << 20);
            CPDB_CK(cudaMemset(fplog.p, 0, fplog.n * sizeof(double)));
        }
    }
    // SolverConfig::validate (solvers.hpp:41-49) and run_qr guards (:217-224)
    if (cfg.rank == 0) fail(CPDB_INVALID_ARGUMENT, "SolverConfig: rank must be >= 1");
    if (cfg.max_iterations == 0)
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: need at least one iteration");
    if (!(cfg.fitness_threshold >= 0.0 && cfg.fitness_threshold <= 1.0))
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: fitness threshold must be in [0,1]");
    if (!std::isfinite(cfg.alpha) || !std::isfinite(cfg.activation_gap))
        fail(CPDB_INVALID_ARGUMENT, "SolverConfig: alpha and activation gap must be finite");
    if (cfg.strategy < 0 || cfg.strategy > 2) fail(CPDB_INVALID_ARGUMENT, "unknown strategy");
    require_tensor(c);
    order = static_cast<uint32_t>(c->dims.size());
    if (order < 2) fail(CPDB_INVALID_ARGUMENT, "cp_als_qr: tensor order must be >= 2");
    if (order > CPDB_MAX_ORDER) fail(CPDB_INVALID_ARGUMENT, "cp_als_qr: order above 8");
    // The reference's initial factors (host Rng, solvers.hpp:116-122) are drawn
    // before the first synchronisation: after cpdb_tensor_set_async the
    // upload of X is still running, and this is host time under it.  (Only
    // when the guards below will pass; nothing here can fail.)
    std::vector<double> init_pre;
    {
        bool sane = !(state && state->factors) && cfg.rank <= 1024;
        uint64_t nf = 0;
        for (uint32_t k = 0; k < order; ++k) {
            sane = sane && cfg.rank <= c->dims[k];
            nf += c->dims[k] * cfg.rank;
        }
        if (sane) {
            init_pre.resize(nf);
            cpd::Rng rng(cfg.seed);
            for (double& v : init_pre) v = rng.normal();
        }
    }
    nx2 = ctx_norm_sq(c);
    if (nx2 == 0.0) fail(CPDB_INVALID_ARGUMENT, "cp_als_qr: zero-norm tensor");
    for (uint32_t k = 0; k < order; ++k)
        if (cfg.rank > c->dims[k])
            fail(CPDB_INVALID_ARGUMENT,
                 "cp_als_qr: rank must not exceed any mode extent (compact QR)");
    if (cfg.rank > 1024)
        fail(CPDB_INVALID_ARGUMENT, "cp_als_qr: ranks above 1024 are not supported on the device");
    R = static_cast<uint32_t>(cfg.rank);
    Rp = ttm_rpad(R);
    {
        const char* hh = std::getenv("CPDB_HOUSEHOLDER");
        if (hh && hh[0] == '1') robust = true;
    }
    extrap = cfg.extrapolate != 0;
    const Strategy strategy =
        extrap ? Strategy::branch_reuse : static_cast<Strategy>(cfg.strategy);
    done = state ? state->sweeps_done : 0;
    first_sweep = done;
    try {
        plan = build_plan(order, strategy, done + cfg.max_iterations);
    } catch (const SchedError& e) {
        fail(e.code, e.what);
    }
    sharded = c->world > 1;
    if (sharded) {
        // layouts, reductions and V collectives of every step (shard.cpp)
        splan = plan_shards(plan, c->dims, R, c->world,
                            static_cast<ShardPolicy>(c->shard_policy), c->shard_cost);
        need_local.assign(order, false);
        qp_local.resize(order);
        for (const auto& sw : splan.steps)
            for (const auto& up : sw)
                for (const StepShard& st : up)
                    if (st.src.kind == kLayShard) need_local[uint32_t(st.src.mode)] = true;
        for (uint32_t m = 0; m < order; ++m)
            if (need_local[m] && c->dims[m] % uint64_t(c->world) != 0)
                fail(CPDB_LOGIC_ERROR, "shard plan splits a mode that does not divide");
    }
    s = c->stream;
    side = c->side;
    zrows = 1;
    for (uint32_t k = 1; k < order; ++k) zrows *= R;
    if (!zqr_cluster_fits(zrows, R, order - 1)) side = c->side_hi;  // tall Z (api.cpp)
    maxI = 0;
    nfac = 0;
    for (uint64_t d : c->dims) {
        maxI = std::max(maxI, d);
        nfac += d * R;
    }
    {
        const uint64_t restarts = c->prof.qr_householder;
        c->prof = cpdb_profile{};
        if (robust) c->prof.qr_householder = restarts;  // (solve()'s second attempt)
    }
    launches0 = c->launches;
    CPDB_CK(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
    CPDB_CK(cudaEventCreateWithFlags(&ev_zqr, cudaEventDisableTiming));
    CPDB_CK(cudaEventCreateWithFlags(&ev_fin, cudaEventDisableTiming));
    CPDB_CK(cudaEventCreateWithFlags(&pf.ev, cudaEventDisableTiming));
    timeline = std::getenv("CPDB_TIMELINE");
    {
        const char* e = std::getenv("CPDB_ROOT_PREFETCH");
        // not for TTM-dominated runs (C5: the root is 95% of the sweep, so the
        // one-tile-per-CTA grid only costs)
        // Sharded runs keep the overlaps (CPDB_SHARD_OVERLAP=0: the simple
        // stream-ordered form): every collective stays on the main stream,
        // bracketed by events to the stream that produced / consumes its
        // data (ttm_step, mode_update_back), so the NCCL operations of the
        // communicator are issued and executed in one order on every rank.
        const char* so = std::getenv("CPDB_SHARD_OVERLAP");
        const bool shard_ok = !sharded || !(so && so[0] == '0');
        prefetch_enabled = c->overlap && shard_ok && !(e && e[0] == '0') &&
                           numel(c->ldims) < (1ull << 32);
        const char* cs = std::getenv("CPDB_CHAIN_SIDE");
        chain_side = c->overlap && shard_ok && !(cs && cs[0] == '0');
        // An update that runs beside the prefetched root TTM is off the
        // critical path (the root is): its branch TTMs and V-GEMM take a few
        // SMs for longer instead of every SM briefly, so the root keeps more.
        // Event-driven fronts: an update's Z-QR waits only for the finishers
        // of the modes it reads (R_k, k != n) and its TTM chain only for the
        // Q_c it contracts, not for everything before it on the stream.  At a
        // sweep boundary the next update has the SAME mode as the last one
        // (branch reuse: orders 1 3 2 | 2 3 1 ..., Appendix A), so its Z-QR
        // and chain run under the previous update's V-GEMM and finisher.
        // Pays together with the speculative next-sweep update (Session::run:
        // no host round trip at the sweep boundary left to hide the front
        // under).  Measured (B200, 100 sweeps): C1 6040 -> 6860 sweeps/s, C2
        // 1911 -> 2003, C3 1258 -> 1310, C4 4626 -> 5259.  CPDB_EARLY_FRONT=0: off.
        const char* ef = std::getenv("CPDB_EARLY_FRONT");
        dep_events = chain_side && !(ef && ef[0] == '0');
        const char* ce = std::getenv("CPDB_CHAIN_EVENTS");
        chain_events = dep_events && !(ce && ce[0] == '0');
        const char* lt = std::getenv("CPDB_LOW_TAIL");
        low_tail = !(lt && lt[0] == '0');
        // the low tail's TTM chain and V-GEMM take this many SMs (stream
        // priority alone does not keep its grids, launched first, from
        // interleaving with the next sweep's first update)
        const char* tsm = std::getenv("CPDB_TAIL_SMS");
        tail_sms = tsm ? std::atoi(tsm) : 80;
        {
            const double xe = double(numel(c->ldims));
            long_root = std::max(2.0 * xe * R / 31.5e12, 8.0 * xe / 6.0e12) >= 150e-6;
        }
        const char* sh = std::getenv("CPDB_SELF_HIST");
        self_hist = !(sh && sh[0] == '0');
        // the repeated update at the sweep boundary takes the previous one's
        // Y_(n) / Q0 / R0 (mode_update_front).  Measured on the B200: C1
        // +2.7%, C4 +2%, C2 flat, C5 +3.5% (a tall Z-QR and a TTM less per
        // sweep); C3 -2% (fourth order, small Z: the repeated chain ran early
        // beside the previous update for free), so fourth order only with a
        // tall Z.  CPDB_REUSE_BOUNDARY=0/1 overrides.
        // slabs of a reduced TTM step whose collectives overlap the next
        // slab's kernel (ttm_step); steps below ~0.2 GFLOP are launch-bound
        // (measured: the 6-7 pre-activation sweeps at C2 run 0.48 -> 0.45 ms,
        // but the steady state that follows the one misprediction settles
        // 1% (C2) to 3% (C1) slower -- the streams' phase alignment differs
        // -- so it is off unless CPDB_PREDICT_GATE=1)
        const char* pg = std::getenv("CPDB_PREDICT_GATE");
        predict_gate = pg && pg[0] == '1';
        const char* rc = std::getenv("CPDB_RS_CHUNKS");
        rs_chunks = rc ? uint32_t(std::max(1, std::atoi(rc))) : 4u;
        const char* rf = std::getenv("CPDB_RS_MIN_FLOPS");
        rs_min_flops = rf ? std::atof(rf) : 2e8;
        const char* rb = std::getenv("CPDB_REUSE_BOUNDARY");
        reuse_ok = rb ? rb[0] != '0' : (order == 3 || !zqr_cluster_fits(zrows, R, order - 1));
        const char* sp = std::getenv("CPDB_SPECULATE");
        speculate = !(sp && sp[0] == '0');
        const char* zy = std::getenv("CPDB_ZQR_YIELD");
        zqr_yield = chain_side && zy && zy[0] == '1' && !zqr_cluster_fits(zrows, R, order - 1);
        const char* os = std::getenv("CPDB_OVERLAP_SMS");
        overlap_sms = os ? std::atoi(os) : -1;
        if (overlap_sms >= c->sms) overlap_sms = 0;
    }

    // ---- factor state (factor_state.hpp:28-34) -----------------------------
    fb.resize(order);
    for (uint32_t k = 0; k < order; ++k) {
        const uint64_t I = c->dims[k];
        fb[k].a.ensure(I * R);
        fb[k].q.ensure(I * R);
        fb[k].qp.ensure(uint64_t(ttm_kpad(I)) * Rp);
        fb[k].r.ensure(uint64_t(R) * R);
    }
    fb_alt.resize(order);
    for (uint32_t k = 0; k < order; ++k) {
        const uint64_t I = c->dims[k];
        fb_alt[k].a.ensure(I * R);
        fb_alt[k].q.ensure(I * R);
        fb_alt[k].qp.ensure(uint64_t(ttm_kpad(I)) * Rp);
        fb_alt[k].r.ensure(uint64_t(R) * R);
    }
    lam.ensure(R);
    lam_alt.ensure(R);
    {
        std::vector<double> init;
        const bool given = state && state->factors;
        if (given) {
            init.assign(state->factors, state->factors + nfac);
        } else if (init_pre.size() == nfac) {
            init.swap(init_pre);  // drawn above, under the upload of X
        } else {
            init.resize(nfac);
            cpd::Rng rng(cfg.seed);  // initial_factors, solvers.hpp:116-122
            for (double& v : init) v = rng.normal();
        }
        uint64_t off = 0;
        for (uint32_t k = 0; k < order; ++k) {
            const uint64_t I = c->dims[k];
            CPDB_CK(cudaMemcpyAsync(fb[k].a.p, init.data() + off, I * R * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
            acc(s, "init_h2d", {}, {rg(fb[k].a.p, I * R)});
            if (!given) {
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
    // (wide ranks: A_hat, the Householder working copy and its partials)
    for (DevBuf& b : fscratch)
        b.ensure(wide_rank(R) || robust ? finish_wide_scratch_doubles(maxI, R) : maxI * (R + 1));
    vout.ensure(maxI * R);
    fitbuf.ensure(8);
    for (ZBuf& z : zb) {
        z.q0.ensure(zrows * R);
        z.q1.ensure(zrows * R);
        z.r0.ensure(uint64_t(R) * R);
        z.work.ensure(zqr_work_doubles(R) + uint64_t(4 * c->sms) * R * R);
    }
    for (DevBuf& b : vfull) b.ensure(maxI * R);
    for (DevBuf& b : vfitfull) b.ensure(maxI * R);
    // V-GEMM partials up front (the dual ones are first needed when the beta
    // gate opens, mid-run: no allocation inside the sweeps)
    for (DevBuf& b : vpart) b.ensure(size_t(vgemm_max_split()) * maxI * R);
    if (extrap)
        for (DevBuf& b : vfitpart) b.ensure(size_t(vgemm_max_split()) * maxI * R);
    versions.assign(order, 1);
    CPDB_CK(cudaMemsetAsync(c->dstatus, 0, 5 * sizeof(int), s));
    {
        const char* fe = std::getenv("CPDB_FAULT_SWEEP");
        fault_sweep = fe ? std::strtoull(fe, nullptr, 10) : 0;
        // (CPDB_FAULT_ONCE=1: only on the CholeskyQR kernels, so the
        // Householder restart of solve() goes through)
        const char* fo = std::getenv("CPDB_FAULT_ONCE");
        if (fo && fo[0] == '1' && robust) fault_sweep = 0;
    }
    for (uint32_t k = 0; k < order; ++k) qr_factor(k);
    for (uint32_t k = 0; k < order; ++k) pack_local(k);
    CPDB_CK(cudaEventCreateWithFlags(&ev_zq, cudaEventDisableTiming));
    CPDB_CK(cudaEventCreateWithFlags(&ev_aux, cudaEventDisableTiming));
    CPDB_CK(cudaEventCreateWithFlags(&ev_tail, cudaEventDisableTiming));
    for (uint32_t k = 0; k < order; ++k) {
        CPDB_CK(cudaEventCreateWithFlags(&ev_fac[k], cudaEventDisableTiming));
        CPDB_CK(cudaEventRecord(ev_fac[k], s));
    }
    for (uint32_t k = 0; k < 2 * order; ++k) {
        CPDB_CK(cudaEventCreateWithFlags(&ev_v[k], cudaEventDisableTiming));
        CPDB_CK(cudaEventRecord(ev_v[k], s));
    }
    for (uint32_t k = 0; k < order; ++k) {
        CPDB_CK(cudaEventCreateWithFlags(&ev_hist[k], cudaEventDisableTiming));
        CPDB_CK(cudaEventRecord(ev_hist[k], s));
    }
    CPDB_CK(cudaEventCreateWithFlags(&ev_zq_pending, cudaEventDisableTiming));
    CPDB_CK(cudaEventRecord(ev_zq_pending, s));
    for (cudaEvent_t& e : ev_zread) {
        CPDB_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CPDB_CK(cudaEventRecord(e, s));
    }
    for (cudaEvent_t& e : ev_zread_b) {
        CPDB_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CPDB_CK(cudaEventRecord(e, s));
    }
    for (uint32_t k = 0; k < 2 * order; ++k) {
        CPDB_CK(cudaEventCreateWithFlags(&ev_v_b[k], cudaEventDisableTiming));
        CPDB_CK(cudaEventRecord(ev_v_b[k], s));
    }

    // ---- Q0 history (reference row order on the host side) -----------------
    perm = natural_to_reference(order, R);
    hist.resize(order);
    has_hist.assign(order, false);
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
    if (extrap && cfg.has_beta_override) {
        has_beta = true;
        beta = cfg.beta_override;
    }
    if (extrap && state && state->has_active_beta && !has_beta) {
        has_beta = true;
        beta = state->active_beta;
    }
    has_prev = state && state->has_prev_fitness;
    prev_fit = has_prev ? state->prev_fitness : 0.0;
    {
        const double g[4] = {has_beta ? 1.0 : 0.0, has_beta ? beta : 0.0, has_prev ? 1.0 : 0.0,
                             prev_fit};
        gate.ensure(4);
        CPDB_CK(cudaMemcpyAsync(gate.p, g, sizeof g, cudaMemcpyHostToDevice, s));
        CPDB_CK(cudaStreamSynchronize(s));
    }

    // cost accounting continues from the sweeps already done (dim_tree.hpp:523-526)
    total = done > 0 ? measured_cost(plan, c->dims, R, done) : Cost{};

    // rebuild the retained intermediates from X and the current factors
    if (done > 0) {
        for (uint32_t key : retained_keys(plan, done - 1, order - 1)) {
            if (cache.count(key)) continue;
            // the layout the plan gave the slot when it last produced it
            ShardLayout want{};
            if (sharded) {
                bool found = false;
                for (uint64_t sw = done; sw-- > 0 && !found;)
                    for (uint32_t b = order; b-- > 0 && !found;) {
                        const Update& u = plan.sweeps[sw].updates[b];
                        for (size_t j = u.steps.size(); j-- > 0;)
                            if (u.steps[j].produces == key && u.steps[j].produces != (1u << u.mode)) {
                                want = splan.steps[sw][b][j].out;
                                found = true;
                                break;
                            }
                    }
            }
            std::vector<uint64_t> d = c->ldims;
            const double* cur = c->x;
            ModeSet cur_set = plan.root();
            ShardLayout lay = sharded ? ShardLayout{kLayShard, 0} : ShardLayout{};
            DevBuf tmp[2];
            int w = 0;
            for (uint32_t k = order; k-- > 0;) {
                if (key & (1u << k)) continue;
                const ModeSet next = cur_set & ~(1u << k);
                // X is split along mode 0, which is contracted last: partial
                // sums at the end only, then brought to the slot's layout
                StepShard sh{lay, lay, kRedNone, -1, 0};
                if (lay.kind == kLayShard && uint32_t(lay.mode) == k) {
                    sh.out = want;
                    if (want.kind == kLayRep) sh.red = kRedAllReduce;
                    if (want.kind == kLayShard) {
                        sh.red = kRedScatter;
                        sh.scatter = want.mode;
                    }
                }
                std::vector<uint64_t> nd = d;
                nd[k] = R;
                if (sh.red == kRedScatter) nd[uint32_t(sh.scatter)] /= uint64_t(c->world);
                double* out = tmp[w].ensure(numel(nd));
                ttm_step(cur, d, sharded ? &sh : nullptr, k, out, false);
                cur_set = next;
                cur = out;
                d = nd;
                lay = sh.out;
                w ^= 1;
            }
            if (sharded && lay != want)
                fail(CPDB_LOGIC_ERROR, "resume: cannot rebuild " + set_name(key, order) +
                                           " in its planned layout");
            Slot& sl = cache[key];
            sl.buf.ensure(numel(d));
            CPDB_CK(cudaMemcpyAsync(sl.buf.p, cur, numel(d) * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
            acc(s, "cache_rebuild_copy", {rg(cur, numel(d))}, {rg(sl.buf.p, numel(d))});
            sl.valid = true;
            sl.dims = d;
            sl.lay = lay;
            sl.sharded = lay.kind == kLayShard;
            sl.stamps.assign(order, 0);
            for (uint32_t k = 0; k < order; ++k)
                if (!(key & (1u << k))) sl.stamps[k] = versions[k];
            CPDB_CK(cudaStreamSynchronize(s));
        }
        events.recycle();
        timers.clear();
    }
    // Y_(n) per mode and update parity (consecutive updates of the same mode
    // -- the sweep boundary -- may be in flight together)
    ybuf.resize(2 * order);
    for (uint32_t n = 0; n < 2 * order; ++n)
        ybuf[n].ensure(numel(dims_in(1u << (n / 2), ShardLayout{})));
    // every cache slot the plan will use, allocated now: a first use inside
    // the sweeps would put a cudaMalloc (device-wide sync; C5: 8.6 GB slots)
    // in the middle of the run
    {
        const uint64_t span = std::min<uint64_t>(
            plan.sweeps.size(), plan.cycle_start + 2 * std::max<uint64_t>(plan.cycle_length, 1) + 1);
        for (uint64_t sw = 0; sw < span; ++sw)
            for (uint32_t b = 0; b < plan.sweeps[sw].updates.size(); ++b) {
                const Update& u = plan.sweeps[sw].updates[b];
                for (size_t j = 0; j < u.steps.size(); ++j) {
                    const Step& st = u.steps[j];
                    if (st.produces == (1u << u.mode)) continue;
                    // sharded: the slot's size in the layout the plan gives it
                    // (the largest over the productions in the span)
                    cache[st.produces].buf.ensure(numel(
                        sharded ? dims_in(st.produces, splan.steps[sw][b][j].out)
                                : local_dims_of(st.produces)));
                }
            }
        if (prefetch_enabled) {
            uint64_t mx = 0;
            for (uint32_t k = 0; k < order; ++k) {
                std::vector<uint64_t> od = c->ldims;
                od[k] = R;
                mx = std::max(mx, numel(od));
            }
            pre.ensure(mx);
        }
    }
    CPDB_CK(cudaEventCreate(&t_start));
    CPDB_CK(cudaEventRecord(t_start, s));
    CPDB_CK(cudaStreamSynchronize(s));
}

std::vector<uint64_t> Session::local_dims_of(uint32_t key) const {
    std::vector<uint64_t> d(order);
    for (uint32_t k = 0; k < order; ++k) d[k] = (key & (1u << k)) ? c->ldims[k] : R;
    return d;
}

void Session::qr_factor(uint32_t k) {
    FinishArgs f{};
    f.init = 1;
    f.I = c->dims[k];
    f.R = R;
    f.a_out = fb[k].a.p;
    f.q_out = fb[k].q.p;
    f.qp_out = fb[k].qp.p;
    f.r_out = fb[k].r.p;
    f.lambda = lam.p;
    f.scratch = fscratch[0].p;
    f.householder = robust ? 1 : 0;
    f.status = status_word(done + 1);  // reported with the first sweep
    f.v_out = vout.p;
    CPDB_CK(launch_finish(f, s));
    acc(s, "qr_factor", {rg(f.a_out, f.I * R)},
          {rg(f.q_out, f.I * R), rg(f.qp_out, uint64_t(ttm_kpad(f.I)) * Rp), rg(f.r_out, R * R),
           rg(f.scratch, f.I * (R + 1))});
    c->launches += 1;
}

// Sharded runs contract a split mode m with this rank's rows of Q_m only;
// they get their own packed copy (no row-alignment constraint), refreshed
// after every update of m.
void Session::pack_local(uint32_t m, cudaStream_t st) {
    if (!sharded || !need_local[m]) return;
    if (!st) st = s;
    const uint64_t rows = shard_rows_of(m);
    qp_local[m].ensure(uint64_t(ttm_kpad(rows)) * Rp);
    const double* src = fb[m].q.p + uint64_t(c->rank) * rows * R;
    CPDB_CK(pack_q(src, qp_local[m].p, uint32_t(rows), R, st));
    acc(st, "pack_local", {rg(src, rows * R)}, {rg(qp_local[m].p, uint64_t(ttm_kpad(rows)) * Rp)});
    c->launches += 1;
}

// CUDA-event pair around a mode-update kernel (Z-QR, V-GEMM, finisher):
// cpdb_profile.mode_update_ms, with CPDB_TIME_TAILS=1 only (the extra events
// break the programmatic launch overlap of the tail: C2 -5% sweeps/s).
Timer Session::tail_timer_begin(cudaStream_t st) {
    static const bool on = [] {
        const char* e = std::getenv("CPDB_TIME_TAILS");
        return e && e[0] == '1';
    }();
    Timer t;
    if (c->timing && on) {
        t.a = events.get();
        t.b = events.get();
        t.kind = 3;
        CPDB_CK(cudaEventRecord(t.a, st));
    }
    return t;
}

void Session::tail_timer_end(Timer& t, cudaStream_t st) {
    if (!t.a) return;
    CPDB_CK(cudaEventRecord(t.b, st));
    timers.push_back(t);
}

uint64_t Session::shard_rows_of(uint32_t m) const { return c->dims[m] / uint64_t(c->world); }

// Extents a tensor over free set `key` has on this rank in layout L (free
// modes I_k, or I_k / world for the split one; contracted modes R).
std::vector<uint64_t> Session::dims_in(uint32_t key, const ShardLayout& L) const {
    std::vector<uint64_t> d(order);
    for (uint32_t k = 0; k < order; ++k)
        d[k] = !(key & (1u << k))                            ? uint64_t(R)
               : (L.kind == kLayShard && uint32_t(L.mode) == k) ? shard_rows_of(k)
                                                                 : c->dims[k];
    return d;
}

void Session::ttm_step(const double* src, const std::vector<uint64_t>& sd, const StepShard* sh,
                       uint32_t k, double* dst, bool is_root, cudaStream_t st, bool prefetch,
                       bool no_pdl, int sms) {
    if (!st) st = s;
    const double* q = fb[k].q.p;
    const double* qp = fb[k].qp.p;
    if (sh && sh->src.kind == kLayShard && uint32_t(sh->src.mode) == k) {
        // contracting the split mode: this rank's rows of Q_k -> a partial sum
        q += uint64_t(c->rank) * shard_rows_of(k) * R;
        qp = qp_local[k].p;
    }
    // a reduce-scatter needs the whole partial first
    double* raw = dst;
    if (sh && sh->red == kRedScatter) raw = rs_tmp[st].ensure(numel(sd) / sd[k] * R);
    std::vector<uint64_t> od = sd;
    od[k] = R;
    // Reduced steps run in slabs of the outermost mode: the collective of slab
    // p (main stream) overlaps the TTM of slab p + 1 (producing stream), so
    // only the last slab's reduction is exposed.  Slabs are whole outer
    // slices of both the source and the result (k != 0), and for a
    // reduce-scatter the scattered mode lies inside them (scatter != 0), so
    // each slab's collective is the same call on a sub-range.  Every output
    // element is accumulated in the same order as in one launch.
    // CPDB_RS_CHUNKS=<n> (default 4; 1: one launch, one collective).
    const uint32_t want_chunks = rs_chunks;
    const double min_flops = rs_min_flops;
    uint32_t chunks = 1;
    // contracting the leading mode (the split one): the result is [R][rest],
    // so the slabs are column halves of Q (rows of the result) -- two 32-column
    // TTMs stay tensor-bound (C2's root shape), narrower ones would not
    const bool by_cols = k == 0;
    const bool big = sh && sh->red != kRedNone &&
                     2.0 * double(numel(od)) * double(sd[k]) >= min_flops;
    // (tensor-core TTM layouts only: the plain kernel reads the unpacked Q)
    if (big && by_cols && want_chunks > 1 && R % 2 == 0 && R / 2 >= 32 && R <= 64 &&
        (numel(sd) / sd[0]) % 8 == 0) {
        chunks = 2;
    } else if (big && !by_cols && !(sh->red == kRedScatter && sh->scatter == 0)) {
        for (uint32_t cnum = want_chunks; cnum > 1; --cnum)
            if (sd[0] % cnum == 0) {
                chunks = cnum;
                break;
            }
    }
    const bool cols = by_cols && chunks > 1;
    const uint32_t Rc = cols ? R / chunks : R;
    const uint64_t in_slab = cols ? numel(sd) : numel(sd) / chunks;
    const uint64_t out_slab = numel(od) / chunks;
    std::vector<uint64_t> sdp = sd, odp = od;
    if (!cols) sdp[0] /= chunks;
    odp[0] /= chunks;
    double* qcols = cols ? qcol_tmp[st].ensure(uint64_t(chunks) * ttm_kpad(sd[k]) * ttm_rpad(Rc))
                         : nullptr;
    Timer tc;
    bool comm_timed = false;
    for (uint32_t p = 0; p < chunks; ++p) {
        const double* srcp = cols ? src : src + uint64_t(p) * in_slab;
        double* rawp = raw + uint64_t(p) * out_slab;
        const double* qpp = qp;
        if (cols) {  // this half's columns of (this rank's rows of) Q_k, packed
            double* dstq = qcols + uint64_t(p) * ttm_kpad(sd[k]) * ttm_rpad(Rc);
            CPDB_CK(pack_q_cols(q, R, p * Rc, Rc, dstq, uint32_t(sd[k]), st));
            acc(st, "pack_cols", {rg(q, sd[k] * R)},
                {rg(dstq, uint64_t(ttm_kpad(sd[k])) * ttm_rpad(Rc))});
            c->launches += 1;
            qpp = dstq;
        }
        Timer t;
        if (c->timing) {
            t.a = events.get();
            t.b = events.get();
            t.kind = is_root ? 0 : 1;
            CPDB_CK(cudaEventRecord(t.a, st));
        }
        cudaEvent_t tla = tl_begin(st);
        fp(st, prefetch ? "root_prefetch" : is_root ? "root_ttm" : "branch_ttm", "in_before",
           {rg(srcp, in_slab), rg(qp, uint64_t(ttm_kpad(sd[k])) * Rp)});
        run_ttm(c, srcp, sdp, k, q, qpp, Rc, rawp, st, prefetch || yield_now, no_pdl || p > 0, sms,
                prefetch ? pf.tpc : 0);
        acc(st, prefetch ? "root_prefetch" : is_root ? "root_ttm" : "branch_ttm",
              {rg(srcp, in_slab), rg(qp, uint64_t(ttm_kpad(sd[k])) * Rp)}, {rg(rawp, out_slab)});
        tl_end(tla, st, prefetch ? "root_prefetch" : is_root ? "root" : "branch");
        if (c->timing) {
            CPDB_CK(cudaEventRecord(t.b, st));
            t.flops = 2.0 * double(out_slab) * double(sd[k]);
            t.bytes = 8.0 * (double(in_slab) + double(out_slab) + double(sd[k]) * R);
            timers.push_back(t);
        }
        if (!sh || sh->red == kRedNone) continue;
        // the collective runs on the main stream, after this slab's kernel
        if (st != s) {
            cudaEvent_t e0 = events.get();
            CPDB_CK(cudaEventRecord(e0, st));
            CPDB_CK(cudaStreamWaitEvent(s, e0, 0));
        }
        if (c->timing && !comm_timed) {
            tc.a = events.get();
            tc.b = events.get();
            tc.kind = 2;
            CPDB_CK(cudaEventRecord(tc.a, s));
            comm_timed = true;
        }
        if (sh->red == kRedAllReduce) {
            allreduce_sum(c, dst + uint64_t(p) * out_slab, out_slab);
        } else {
            // blocks: everything from the scattered mode inward (contiguous,
            // that mode outermost), one per index of the modes before it
            const uint32_t m = uint32_t(sh->scatter);
            uint64_t outer = 1;
            for (uint32_t j = 0; j < m; ++j) outer *= odp[j];
            const uint64_t block = out_slab / outer;
            reduce_scatter(c, rawp, outer, block,
                           dst + uint64_t(p) * outer * (block / uint64_t(c->world)));
        }
    }
    if (sh && sh->red != kRedNone) {
        if (comm_timed) {
            CPDB_CK(cudaEventRecord(tc.b, s));
            timers.push_back(tc);
        }
        if (st != s) {  // the producing stream goes on with the reduced data
            cudaEvent_t e1 = events.get();
            CPDB_CK(cudaEventRecord(e1, s));
            CPDB_CK(cudaStreamWaitEvent(st, e1, 0));
        }
    }
}

// Root-TTM prefetch.  In a branch-reuse sweep the single root TTM sits in a
// later update and contracts a mode whose Q was final one or more updates
// earlier ("Dependencies and overlap").  Right after update b,
// if update b2 > b+1 starts with a root step contracting c and no update in
// (b, b2) changes Q_c, the root TTM is issued on the low-priority stream into
// a spare buffer: its CTAs (one tile each) fill the SMs the latency-bound
// updates in between leave idle, and update b2 adopts the buffer.
void Session::prefetch_root(uint64_t sweep, uint32_t b, cudaStream_t after) {
    if (!prefetch_enabled || pf.active) return;
    const Sweep& sw = plan.sweeps[sweep - 1];
    for (uint32_t b2 = b + 2; b2 < order; ++b2) {
        const Update& u = sw.updates[b2];
        if (u.steps.empty() || u.steps[0].source != plan.root()) continue;
        const uint32_t cm = u.steps[0].contract;
        if (u.steps[0].produces == (1u << u.mode)) continue;  // (order 2: nothing to gain)
        bool fresh = true;
        for (uint32_t bm = b + 1; bm < b2; ++bm) fresh = fresh && sw.updates[bm].mode != cm;
        if (!fresh) continue;
        // sharded: a root whose partial sums are reduced stays in order (its
        // collective on the main stream would wait for the whole prefetch)
        if (sharded && splan.steps[sweep - 1][b2][0].red != kRedNone) continue;
        std::vector<uint64_t> od = c->ldims;
        od[cm] = R;
        pre.ensure(numel(od));
        CPDB_CK(cudaEventRecord(ev_fin, after));  // update b's finisher: Q_cm final
        pf.cm = cm;
        pf.launched = false;
        // SM budget of the updates in between: they are off the critical
        // path when the root is long (it, not they, gates update b2), so their
        // TTMs get just enough SMs to finish well within the root's time
        // and the root keeps the rest.  Short roots (C4: ~30 us) are not
        // worth it (the updates become the critical path).
        pf.sms = overlap_sms >= 0 ? overlap_sms : 0;
        const double xb = 8.0 * double(numel(c->ldims));
        const double root_s = std::max(2.0 * double(numel(c->ldims)) * R / 31.5e12, xb / 6.0e12);
        // CTAs of two tiles for a long root (half the per-CTA prologues; C2
        // 2204 -> 2248 sweeps/s), of one tile for a short one, whose CTAs must
        // make way for the critical Z-QR quickly (C4 5700 -> 6080)
        pf.tpc = root_s >= 150e-6 ? 2 : 1;
        if (overlap_sms < 0) {
            double upd = 0.0;
            for (uint32_t bm = b + 1; bm < b2; ++bm)
                for (const Step& st : sw.updates[bm].steps) upd += step_flops(st);
            const double per_sm = 0.15e12;  // FP64 FLOP/s per SM on a small grid
            // finish in ~0.5 of the root's time (measured on the final
            // schedule, C2: 0.3 2474, 0.38 2482, 0.5 2507, 0.75 2507, 1.0 2514
            // sweeps/s; C3 flat)
            static const double frac = [] {
                const char* e = std::getenv("CPDB_OVERLAP_FRAC");
                return e ? std::atof(e) : 0.5;
            }();
            const int need = int(std::ceil(upd / (frac * root_s * per_sm)));
            if (root_s >= 150e-6 && need < c->sms / 2) pf.sms = std::max(need, 16);
        }
        pf.active = true;
        pf.sweep = sweep;
        pf.block = b2;
        return;
    }
}

// The planned root prefetch goes on the low-priority stream right behind the
// next update's Z-QR launch: the Z-QR's 8-CTA cluster (on the critical path
// when the root is short, C4) gets its SMs before the root's CTAs fill them.
void Session::launch_prefetch() {
    if (!pf.active || pf.launched) return;
    CPDB_CK(cudaStreamWaitEvent(c->lo, ev_fin, 0));
    // (sharded: the planned step -- contracting the split mode takes this
    // rank's rows of Q; prefetched roots are never reduced, prefetch_root)
    ttm_step(c->x, c->ldims, sharded ? &splan.steps[pf.sweep - 1][pf.block][0] : nullptr, pf.cm,
             pre.p, true, c->lo, true, true);
    CPDB_CK(cudaEventRecord(pf.ev, c->lo));
    pf.launched = true;
}

void Session::fp(cudaStream_t st, const char* what, const char* phase,
                 std::initializer_list<HbCheck::Rg> regions) {
    if (!fpath || st == nullptr) return;
    // light: outputs of the TTMs, Z-QR, V-GEMM and finisher, and the V-GEMM's
    // inputs just before and after it
    if (fp_light && phase[0] != 'o' && what[0] != 'v') return;
    if (fp_light && phase[0] == 'o' && !(what[0] == 'f' || what[0] == 'z' || what[0] == 'v' ||
                                        what[0] == 'r' || what[0] == 'b'))
        return;
    int k = 0;
    for (const HbCheck::Rg& g : regions) {
        ++k;
        if (!g.p || !g.bytes) continue;
        const size_t idx = fplabels.size();
        if (idx >= fplog.n) return;
        char lab[160];
        std::snprintf(lab, sizeof lab, "%llu %u %s %s %d", (unsigned long long)hb.cur_sweep,
                      hb.cur_mode, what, phase, k);
        fplabels.push_back(lab);
        CPDB_CK(fingerprint(static_cast<const double*>(g.p), g.bytes / sizeof(double),
                            reinterpret_cast<unsigned long long*>(fplog.p) + idx, st));
    }
}

void Session::fp_flush() {
    if (!fpath || fplabels.empty()) return;
    CPDB_CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(fplabels.size());
    CPDB_CK(cudaMemcpy(h.data(), fplog.p, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost));
    FILE* f = std::fopen(fpath, "a");
    if (f) {
        std::fprintf(f, "=== session\n");
        for (size_t i = 0; i < h.size(); ++i)
            std::fprintf(f, "%zu %s %016llx\n", i, fplabels[i].c_str(), h[i]);
        std::fclose(f);
    }
    fplabels.clear();
    CPDB_CK(cudaMemset(fplog.p, 0, fplog.n * sizeof(double)));
}

cudaEvent_t Session::ready_event(uint32_t key) {
    auto it = slot_ready.find(key);
    if (it != slot_ready.end()) return it->second;
    cudaEvent_t e;
    CPDB_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CPDB_CK(cudaEventRecord(e, s));  // (first use: everything issued so far)
    slot_ready[key] = e;
    return e;
}

double Session::step_flops(const Step& st) const {
    uint64_t out = 1;
    for (uint32_t k = 0; k < order; ++k)
        out *= (st.produces & (1u << k)) ? c->ldims[k] : uint64_t(R);
    return 2.0 * double(out) * double(st.source == plan.root() || (st.source & (1u << st.contract))
                                          ? c->ldims[st.contract]
                                          : R);
}

// ---------------------------------------------------------------- one mode update
void Session::mode_update(uint64_t sweep, uint32_t b, cpdb_q0_observer observer, void* user,
                          double& beta_used) {
    mode_update_front(sweep, b, observer, user);
    mode_update_back(sweep, b, beta_used);
}

// Steps 1-2 and 4: Z-QR (side stream) and the TTM chain.  Neither depends on
// the beta decision, so the first update of the next sweep can be issued
// before the host reads this sweep's fitness (Session::run).
void Session::mode_update_front(uint64_t sweep, uint32_t b, cpdb_q0_observer observer,
                                void* user) {
    const Sweep& sw = plan.sweeps[sweep - 1];
    const uint32_t n = sw.updates[b].mode;
    const uint32_t root = plan.root();

    // The sweep boundary repeats a mode: the permuted orders end one sweep
    // and begin the next with the same mode n, and nothing this update's
    // Z-QR and TTM chain read (R_k and Q_k of the other modes, the cached
    // source) has changed since the previous update's -- its Q0, R0 and
    // Y_(n) are what the kernels would produce again, bit for bit (they are
    // deterministic).  The repeated launches are elided and the back takes
    // the previous update's buffers (the other parity's Y_(n) and R0, and Q0
    // where the previous back left it).  The cost report still counts the
    // step, as the reference does (it executes it).  Checked, not assumed:
    // same mode, same single step on the same source buffer and stamps, same
    // factor versions of every other mode.
    zb[zpar].reuse = false;
    if (reuse_ok && self_hist && dep_events && !sharded && observer == nullptr &&
        tail_override == nullptr && last_mode == int(n) && prev_front.valid &&
        prev_front.mode == n && sw.updates[b].steps.size() == 1) {
        const Step& st = sw.updates[b].steps[0];
        auto it = st.source == root ? cache.end() : cache.find(st.source);
        bool same = it != cache.end() && it->second.valid && st.produces == (1u << n) &&
                    prev_front.source == st.source && prev_front.contract == st.contract &&
                    prev_front.src_buf == it->second.buf.p &&
                    prev_front.src_stamps == it->second.stamps && (!extrap || has_hist[n]);
        for (uint32_t k = 0; same && k < order; ++k)
            same = k == n || prev_front.versions[k] == versions[k];
        if (same) {
            for (uint32_t m = 0; m < order; ++m)
                if (it->second.stamps[m] && it->second.stamps[m] != versions[m])
                    fail(CPDB_STALE_INTERMEDIATE,
                         "execute: stale intermediate " + set_name(st.source, order));
            uint64_t gout = 1;
            for (uint32_t k = 0; k < order; ++k)
                gout *= (st.produces & (1u << k)) ? c->dims[k] : uint64_t(R);
            total.flops += 2ull * gout * c->dims[st.contract];
            const std::vector<ModeSet> keep = retained_keys(plan, sweep - 1, b);
            for (auto& kv : cache)
                if (std::find(keep.begin(), keep.end(), kv.first) == keep.end())
                    kv.second.valid = false;
            zb[zpar].reuse = true;
            zb[zpar].hist_is_self = true;
            early = true;
            tl_sweep = sweep;
            tl_mode = n;
            hb.cur_sweep = sweep;
            hb.cur_mode = n;
            launch_prefetch();
            return;
        }
    }

    // 1-2. Khatri-Rao + QR of the other R_k -> Q0, R0 (solvers.hpp:250-255)
    ZqrArgs z{};
    uint32_t t = 0;
    for (uint32_t k = 0; k < order; ++k)
        if (k != n) z.rmats[t++] = fb[k].r.p;
    z.nm = order - 1;
    z.R = R;
    z.zrows = zrows;
    ZBuf& zcur = zb[zpar];
    z.q1 = zcur.q1.p;
    z.q0 = zcur.q0.p;
    z.r0 = zcur.r0.p;
    z.work = zcur.work.p;
    z.status = status_word(sweep);
    z.householder = robust ? 1 : 0;
    // Z-QR depends only on R_k (k != n), final since the previous update's
    // finisher, and overlaps the TTM chain on a second stream.  Unsharded, the
    // Z-QR follows the finisher on the main stream (programmatic launch: its
    // 8-CTA cluster is resident before the chain's CTAs arrive, which would
    // otherwise leave no GPC with 8 free SMs) and the chain runs on the side
    // stream; sharded runs keep the chain (and its collectives) on the main one.
    // Event-driven when the previous update had the same mode (the sweep
    // boundary): Z-QR on the side stream, chain on the mid one, both free of
    // the previous update's V-GEMM and finisher.  Otherwise the stream-ordered
    // form below (its Z-QR launches programmatically right behind the
    // finisher, measured faster when it has to wait for that finisher anyway).
    early = dep_events && last_mode == int(n);
    // same deterministic kernel on the same R_k (k != n) as the previous
    // update of mode n: its Q0 (the history, solvers.hpp:265) is this Q0
    zb[zpar].hist_is_self = last_mode == int(n) && has_hist[n] && self_hist;
    // (the sweep-boundary Z-QR on its own stream, not behind the previous
    // chain on `side`)
    cudaStream_t zs = early ? c->zq : chain_side ? s : side;
    if (!early && zqr_stream_override) {
        // right behind the speculative update's finisher on its own stream,
        // so its cluster is resident before the root prefetch and the chain
        // fill the GPU; the Z-QR buffer set's last readers ran elsewhere
        zs = zqr_stream_override;
        CPDB_CK(cudaStreamWaitEvent(zs, ev_zread[zpar], 0));
        CPDB_CK(cudaStreamWaitEvent(zs, ev_zread_b[zpar], 0));
    }
    static const bool trace_phases = std::getenv("CPDB_PHASE_TRACE") != nullptr;
    if (trace_phases) {
        z.ts = reinterpret_cast<unsigned long long*>(zts.ensure(32));
        CPDB_CK(cudaMemsetAsync(z.ts, 0, 32 * sizeof(double), zs));
    }
    const cudaStream_t ts = tail_override ? tail_override
                            : early       ? c->mid
                            : chain_side  ? (zqr_yield ? c->mid : side)
                                          : s;
    if (early) {
        for (uint32_t k = 0; k < order; ++k)
            if (k != n) CPDB_CK(cudaStreamWaitEvent(zs, ev_fac[k], 0));
        CPDB_CK(cudaStreamWaitEvent(zs, ev_zread[zpar], 0));
        CPDB_CK(cudaStreamWaitEvent(zs, ev_zread_b[zpar], 0));
        uint32_t waited = 0;
        for (const Step& st : sw.updates[b].steps)
            if (!(waited & (1u << st.contract))) {
                CPDB_CK(cudaStreamWaitEvent(ts, ev_fac[st.contract], 0));
                waited |= 1u << st.contract;
            }
        // the producer of its cached source (the previous update's adopted
        // root, typically) and the older V-GEMM that last read this parity's
        // ybuf -- not the previous chain or V-GEMM: this chain (the same
        // contraction as the previous update's last step) runs beside them.
        // A chain that also writes cache slots waits for the previous one.
        CPDB_CK(cudaStreamWaitEvent(ts, ev_v[2 * n + zpar], 0));
        CPDB_CK(cudaStreamWaitEvent(ts, ev_v_b[2 * n + zpar], 0));
        const Step& s0 = sw.updates[b].steps.front();
        if (s0.source != root) CPDB_CK(cudaStreamWaitEvent(ts, ready_event(s0.source), 0));
        bool writes_slots = false;
        for (const Step& st : sw.updates[b].steps) writes_slots |= st.produces != (1u << n);
        // (measured: C2 2278 -> 2363 sweeps/s; CPDB_EARLY_CHAIN_RELAXED=0 off)
        static const bool relaxed = [] {
            const char* e = std::getenv("CPDB_EARLY_CHAIN_RELAXED");
            return !(e && e[0] == '0');
        }();
        if (!relaxed || writes_slots || s0.source == root)
            CPDB_CK(cudaStreamWaitEvent(ts, ev_zqr, 0));
    } else if (chain_events) {
        // Event-driven chain: not behind the previous update's finisher but
        // behind the previous chain (cached sources, slot reuse) and the
        // V-GEMM that last read ybuf[n]; each step then waits for the update
        // that last changed the Q it contracts (below).  A fourth-order
        // update's first step usually contracts a mode the previous update
        // did not touch, so it runs under that update's V-GEMM and finisher.
        CPDB_CK(cudaStreamWaitEvent(ts, ev_zqr, 0));
        CPDB_CK(cudaStreamWaitEvent(ts, ev_v[2 * n + zpar], 0));
        CPDB_CK(cudaStreamWaitEvent(ts, ev_v_b[2 * n + zpar], 0));
    } else {
        CPDB_CK(cudaEventRecord(ev_ready, s));
        CPDB_CK(cudaStreamWaitEvent(chain_side ? ts : side, ev_ready, 0));
    }
    z.pdl = chain_side && !early && !trace_phases ? 1 : 0;
    tl_sweep = sweep;
    tl_mode = n;
    hb.cur_sweep = sweep;
    hb.cur_mode = n;
    cudaEvent_t tla = tl_begin(zs);
    fp(zs, "zqr", "in_before",
       {rg(z.rmats[0], R * R), rg(z.rmats[1], order > 2 ? R * R : 0),
        rg(z.rmats[2], order > 3 ? R * R : 0), rg(z.rmats[3], order > 4 ? R * R : 0)});
    {
        Timer tt = tail_timer_begin(zs);
        CPDB_CK(launch_zqr(z, zs, c->sms));
        tail_timer_end(tt, zs);
    }
    acc(zs, "zqr",
          {rg(z.rmats[0], R * R), rg(z.rmats[1], order > 2 ? R * R : 0),
           rg(z.rmats[2], order > 3 ? R * R : 0), rg(z.rmats[3], order > 4 ? R * R : 0)},
          {rg(z.q1, zrows * R), rg(z.q0, zrows * R), rg(z.r0, R * R), rg(z.work, zcur.work.n)});
    tl_end(tla, zs, "zqr");
    launch_prefetch();
    if (!chain_side) CPDB_CK(cudaEventRecord(ev_zqr, side));
    // (the V-GEMM may run on another stream than the Z-QR: the speculative
    // next-sweep update goes on its own stream, Session::run)
    if (dep_events) CPDB_CK(cudaEventRecord(ev_zq, zs));
    CPDB_CK(cudaEventRecord(ev_zq_pending, zs));  // becomes ev_hist[n] at the back
    if (trace_phases) {
        unsigned long long ts[32];
        CPDB_CK(cudaMemcpyAsync(ts, z.ts, sizeof ts, cudaMemcpyDeviceToHost, zs));
        CPDB_CK(cudaStreamSynchronize(zs));
        std::fprintf(stderr, "zqr mode %u phases(us):", n);
        for (int k = 1; k < 13; ++k)
            std::fprintf(stderr, " %d:%.2f", k, ts[k] ? (ts[k] - ts[0]) * 1e-3 : -1.0);
        std::fprintf(stderr, "\n");
    }
    c->launches += 5;
    if (observer) {
        std::vector<double> nat(zrows * R), ref(zrows * R);
        CPDB_CK(cudaMemcpyAsync(nat.data(), zcur.q0.p, zrows * R * sizeof(double),
                                cudaMemcpyDeviceToHost, zs));
        acc(zs, "observer_d2h", {rg(zcur.q0.p, zrows * R)}, {});
        CPDB_CK(cudaStreamSynchronize(zs));
        for (uint64_t i = 0; i < zrows; ++i)
            std::memcpy(&ref[perm[i] * R], &nat[i * R], R * sizeof(double));
        observer(user, sweep, n, ref.data(), zrows, R);
    }
    // 4. the scheduled TTM chain (execute, dim_tree.hpp:496-541)
    yield_now = zqr_yield;
    bool after_wait = chain_side;  // the side stream's first kernel follows an event wait
    uint32_t chain_waited = 0;     // (chain_events) modes whose finisher this chain waited for
    for (size_t si = 0; si < sw.updates[b].steps.size(); ++si) {
        const Step& st = sw.updates[b].steps[si];
        const double* src;
        std::vector<uint64_t> sd;
        std::vector<uint64_t> stamp(order, 0);
        const StepShard* sh = sharded ? &splan.steps[sweep - 1][b][si] : nullptr;
        if (st.source == root) {
            src = c->x;
            sd = c->ldims;
        } else {
            auto it = cache.find(st.source);
            if (it == cache.end() || !it->second.valid)
                fail(CPDB_LOGIC_ERROR, "execute: scheduled source " + set_name(st.source, order) +
                                           " missing from cache");
            for (uint32_t m = 0; m < order; ++m)
                if (it->second.stamps[m] && it->second.stamps[m] != versions[m])
                    fail(CPDB_STALE_INTERMEDIATE,
                         "execute: stale intermediate " + set_name(st.source, order));
            src = it->second.buf.p;
            sd = it->second.dims;
            stamp = it->second.stamps;
            if (sh && it->second.lay != sh->src)
                fail(CPDB_LOGIC_ERROR, "execute: shard layout of " + set_name(st.source, order));
        }
        std::vector<uint64_t> od = sd;
        od[st.contract] = R;
        if (sh && sh->red == kRedScatter) od[uint32_t(sh->scatter)] /= uint64_t(c->world);
        if (si == 0 && pf.active && pf.sweep == sweep && pf.block == b) {
            // issued early by prefetch_root: adopt its buffer as the slot
            launch_prefetch();
            cudaEvent_t tlw = tl_begin(ts);
            CPDB_CK(cudaStreamWaitEvent(ts, pf.ev, 0));
            tl_end(tlw, ts, "adopt_wait");
            cache[st.produces].buf.swap(pre);
            pf.active = false;
            after_wait = true;
            // ready when the root kernel on the low-priority stream is: a
            // later chain on this source (the next sweep's first update)
            // then waits for the root itself, like this chain, instead of
            // for this stream -- both become runnable together and the
            // stream priorities decide which gets the SMs first
            if (dep_events) CPDB_CK(cudaEventRecord(ready_event(st.produces), c->lo));
        } else {
            double* dst = (st.produces == (1u << n)) ? ybuf[2 * n + zpar].p
                                                    : cache[st.produces].buf.ensure(numel(od));
            if (chain_events && !early && !(chain_waited & (1u << st.contract))) {
                CPDB_CK(cudaStreamWaitEvent(ts, ev_fac[st.contract], 0));
                chain_waited |= 1u << st.contract;
                after_wait = true;
            }
            ttm_step(src, sd, sh, st.contract, dst, st.source == root, ts, false,
                     after_wait, tail_override ? tail_sms : budget(sweep, b));
            after_wait = false;
            if (dep_events && st.produces != (1u << n))
                CPDB_CK(cudaEventRecord(ready_event(st.produces), ts));
        }
        // global-extent flop count, exactly as the reference counts it
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
            sl.lay = sh ? sh->out : ShardLayout{};
            sl.sharded = sl.lay.kind == kLayShard;
        }
    }
    const std::vector<ModeSet> keep = retained_keys(plan, sweep - 1, b);
    for (auto& kv : cache)
        if (std::find(keep.begin(), keep.end(), kv.first) == keep.end()) kv.second.valid = false;
    yield_now = false;
    if (chain_side) CPDB_CK(cudaEventRecord(ev_zqr, ts));  // join: V needs Y_(n)
    // what this front computed (a repetition at the sweep boundary reuses it)
    prev_front.valid = false;
    if (!sw.updates[b].steps.empty() && sw.updates[b].steps.back().source != root &&
        sw.updates[b].steps.back().produces == (1u << n)) {
        const Step& st = sw.updates[b].steps.back();  // Y_(n) from a cached source
        auto it = cache.find(st.source);
        if (it != cache.end()) {
            prev_front.valid = true;
            prev_front.mode = n;
            prev_front.source = st.source;
            prev_front.contract = st.contract;
            prev_front.src_buf = it->second.buf.p;
            prev_front.src_stamps = it->second.stamps;
            prev_front.versions = versions;
        }
    }

}

// Steps 3 and 5-9: extrapolation gate, V, and the mode-update tail.
void Session::mode_update_back(uint64_t sweep, uint32_t b, double& beta_used, cudaStream_t bs,
                               bool host_beta) {
    if (!bs) bs = s;
    const Sweep& sw = plan.sweeps[sweep - 1];
    const uint32_t n = sw.updates[b].mode;
    const bool last = (b == order - 1);
    // 3. extrapolation gate (solvers.hpp:260-265).  The V-GEMM takes the beta
    // decision from the device copy of the state (gate), which is already
    // current when this update was issued before the host read the previous
    // sweep's fitness (speculation, Session::run); the host mirror below is
    // current otherwise and only feeds the trace.
    const bool maybe_ex = extrap && has_hist[n];
    const bool use_ex = maybe_ex && has_beta && beta != 0.0;
    if (use_ex) beta_used = beta;

    // 5. V = Y_(n) Q0_hat (+ the unextrapolated V for the fitness, :277-284)
    const UpdateShard* ush = sharded ? &splan.updates[sweep - 1][b] : nullptr;
    const std::vector<uint64_t> yd =
        sharded ? dims_in(1u << n, ush->yn) : local_dims_of(1u << n);
    VgemmArgs v{};
    ZBuf& zcur = zb[zpar];
    // (a repeated update reads the previous update's outputs: the other
    // parity's Y_(n) and R0; its Q0 was moved into the history by that back
    // when extrapolation is on)
    const bool reuse = zcur.reuse;
    const int ypar = reuse ? (zpar ^ 1) : zpar;
    const double* q0_src = !reuse ? zcur.q0.p : extrap ? hist[n].p : zb[ypar].q0.p;
    v.y = ybuf[2 * n + ypar].p;
    v.q0 = q0_src;
    // (at the sweep boundary the history is this update's own Q0, bit for
    // bit: the V-GEMM need not wait for the previous update's Z-QR)
    v.hist = maybe_ex ? (zcur.hist_is_self ? q0_src : hist[n].p) : nullptr;
    v.beta = beta;
    v.alpha = cfg.alpha;
    v.extrap = maybe_ex ? 1 : 0;
    v.gate = (maybe_ex && !host_beta) ? gate.p : nullptr;
    if (host_beta && !use_ex) v.extrap = 0;
    // (dual with the gate closed: V and Vfit come out bit-identical)
    v.dual = (last && maybe_ex) ? 1 : 0;
    v.I = yd[n];
    v.O = 1;
    for (uint32_t k = 0; k < n; ++k) v.O *= R;
    v.J = 1;
    for (uint32_t k = n + 1; k < order; ++k) v.J *= R;
    v.R = R;
    const size_t part = size_t(vgemm_max_split()) * v.I * R;
    // (split partials, V, scratch: one set per update parity -- consecutive
    // updates may run concurrently, Session::run)
    DevBuf& vf = vfull[zpar];
    DevBuf& vff = vfitfull[zpar];
    v.vpart = vpart[zpar].ensure(part);
    v.vfitpart = v.dual ? vfitpart[zpar].ensure(part) : nullptr;
    // split-K partials -> V (this rank's rows; sharded mode-0 updates gather
    // the full V on every rank)
    // V's collective: this rank's rows of a split Y(n) are gathered, the
    // partial V of a partial Y(n) is all-reduced
    const bool gather = ush && ush->vop == kVGather;
    const bool vsum = ush && ush->vop == kVAllReduce;
    const uint64_t off = gather ? uint64_t(c->rank) * yd[n] * R : 0;
    v.v_out = vf.p + off;
    v.vfit_out = v.dual ? vff.p + off : nullptr;
    CPDB_CK(cudaStreamWaitEvent(bs, ev_zqr, 0));
    if (dep_events) CPDB_CK(cudaStreamWaitEvent(bs, ev_zq, 0));  // Q0, R0 ready
    // the history Q0 comes from the previous update of this mode's Z-QR, which
    // nothing else orders before this V-GEMM once the fronts are event-driven
    if (maybe_ex && !zcur.hist_is_self) CPDB_CK(cudaStreamWaitEvent(bs, ev_hist[n], 0));
    tl_sweep = sweep;
    tl_mode = n;
    hb.cur_sweep = sweep;
    hb.cur_mode = n;
    cudaEvent_t tla = tl_begin(bs);
    // partials summed by the finisher: few enough that its 8 CTAs read them
    // quickly (env CPDB_VSPLIT_MAX, default 16)
    static const uint32_t vsplit_max = [] {
        const char* e = std::getenv("CPDB_VSPLIT_MAX");
        return e ? uint32_t(std::atoi(e)) : 16u;
    }();
    v.max_split = (vsplit_max > 0 && !gather && !vsum && !robust && finish_sums_splits(v.I, R)) ? vsplit_max
                                                                                        : 0;
    const int vsms = bs == c->tailq && tail_sms > 0 ? tail_sms : budget(sweep, b);
    fp(bs, "vgemm", "in_before",
       {rg(v.y, numel(yd)), rg(v.q0, zrows * R), rg(v.hist, v.extrap ? zrows * R : 0),
        rg(v.gate, v.gate ? 4 : 0)});
    {
        Timer tt = tail_timer_begin(bs);
        CPDB_CK(launch_vgemm(v, bs, vsms > 0 ? vsms : c->sms));
        tail_timer_end(tt, bs);
    }
    acc(bs, "vgemm",
          {rg(v.y, numel(yd)), rg(v.q0, zrows * R), rg(v.hist, v.extrap ? zrows * R : 0),
           rg(v.gate, v.gate ? 4 : 0)},
          {rg(v.vpart, v.reduced ? 0 : uint64_t(v.nsplit) * v.I * R),
           rg(v.vfitpart, v.dual && !v.reduced ? uint64_t(v.nsplit) * v.I * R : 0),
           rg(v.v_out, v.reduced ? v.I * R : 0), rg(v.vfit_out, v.reduced && v.dual ? v.I * R : 0)});
    tl_end(tla, bs, "vgemm");
    c->launches += 1;
    if (dep_events) CPDB_CK(cudaEventRecord(ev_v[2 * n + zpar], bs));  // ybuf consumed
    if (dep_events && reuse) CPDB_CK(cudaEventRecord(ev_v_b[2 * n + ypar], bs));
    // the cluster finisher sums the split-K partials itself (no reduction
    // launch on the chain); gathered (sharded mode-0) V needs them reduced
    const bool fused = vsplit_max > 0 && !v.reduced && !gather && !vsum && v.nsplit <= 64 &&
                       !robust && finish_sums_splits(v.I, R);
    if (!v.reduced && !fused) {
        tla = tl_begin(bs);
        CPDB_CK(reduce_splits(v.vpart, v.nsplit, v.I * R, vf.p + off, bs));
        acc(bs, "reduce", {rg(v.vpart, uint64_t(v.nsplit) * v.I * R)}, {rg(vf.p + off, v.I * R)});
        if (v.dual) {
            CPDB_CK(reduce_splits(v.vfitpart, v.nsplit, v.I * R, vff.p + off, bs));
            acc(bs, "reduce", {rg(v.vfitpart, uint64_t(v.nsplit) * v.I * R)},
                  {rg(vff.p + off, v.I * R)});
        }
        tl_end(tla, bs, "reduce");
        c->launches += v.dual ? 2 : 1;
    }
    if ((gather || vsum) && bs != s) {  // collectives on the main stream
        cudaEvent_t e0 = events.get();
        CPDB_CK(cudaEventRecord(e0, bs));
        CPDB_CK(cudaStreamWaitEvent(s, e0, 0));
    }
    if (gather) {
        allgather(c, vf.p, v.I * R);
        if (v.dual) allgather(c, vff.p, v.I * R);
    }
    if (vsum) {
        allreduce_sum(c, vf.p, v.I * R);
        if (v.dual) allreduce_sum(c, vff.p, v.I * R);
    }
    if ((gather || vsum) && bs != s) {
        cudaEvent_t e1 = events.get();
        CPDB_CK(cudaEventRecord(e1, s));
        CPDB_CK(cudaStreamWaitEvent(bs, e1, 0));
    }
    // 6-9. A_hat, lambda, factor QR, fitness (solvers.hpp:272-292)
    FinishArgs f{};
    f.init = 0;
    f.vpart = fused ? v.vpart : vf.p;
    f.vfitpart = v.dual ? (fused ? v.vfitpart : vff.p) : nullptr;
    f.nsplit = fused ? v.nsplit : 1;
    f.dual = v.dual;
    f.r0 = zb[ypar].r0.p;
    f.I = c->dims[n];
    f.R = R;
    f.v_out = vout.p;
    f.a_out = fb_alt[n].a.p;
    f.q_out = fb_alt[n].q.p;
    f.qp_out = fb_alt[n].qp.p;
    f.r_out = fb_alt[n].r.p;
    f.lambda = lam_alt.p;
    f.scratch = fscratch[zpar].p;
    f.householder = robust ? 1 : 0;
    f.fitness = last ? 1 : 0;
    f.norm_x_sq = nx2;
    f.fit_out = fitbuf.p;
    f.status = status_word(sweep);
    static const bool trace_phases = std::getenv("CPDB_PHASE_TRACE") != nullptr;
    if (trace_phases) {
        f.ts = reinterpret_cast<unsigned long long*>(tsbuf.ensure(32));
        CPDB_CK(cudaMemsetAsync(f.ts, 0, 32 * sizeof(double), bs));
    }
    tla = tl_begin(bs);
    {
        const uint64_t vin = uint64_t(f.nsplit) * f.I * R;
        fp(bs, "finish", "in_before",
           {rg(f.vpart, vin), rg(f.vfitpart, f.dual ? vin : 0), rg(f.r0, R * R)});
    }
    {
        Timer tt = tail_timer_begin(bs);
        CPDB_CK(launch_finish(f, bs));
        tail_timer_end(tt, bs);
    }
    {
        const uint64_t vin = uint64_t(f.nsplit) * f.I * R;
        acc(bs, "finish", {rg(f.vpart, vin), rg(f.vfitpart, f.dual ? vin : 0), rg(f.r0, R * R)},
              {rg(f.a_out, f.I * R), rg(f.q_out, f.I * R),
               rg(f.qp_out, uint64_t(ttm_kpad(f.I)) * Rp), rg(f.r_out, R * R), rg(f.lambda, R),
               rg(f.scratch, f.I * (R + 1)), rg(f.fit_out, f.fitness ? 2 : 0)});
    }
    tl_end(tla, bs, "finish");
    c->launches += 1;
    if (fault_sweep == sweep && b == 0)  // test hook: a breakdown in this update
        CPDB_CK(cudaMemsetAsync(status_word(sweep), 2, 1, bs));
    fb[n].swap(fb_alt[n]);  // the new factor state (the old one stays for undo)
    lam.swap(lam_alt);
    if (trace_phases) {
        unsigned long long ts[32];
        CPDB_CK(cudaMemcpyAsync(ts, f.ts, sizeof ts, cudaMemcpyDeviceToHost, bs));
        CPDB_CK(cudaStreamSynchronize(bs));
        std::fprintf(stderr, "finish mode %u phases(us):", n);
        for (int k = 1; k < 21; ++k)
            std::fprintf(stderr, " %d:%.2f", k, ts[k] ? (ts[k] - ts[0]) * 1e-3 : -1.0);
        std::fprintf(stderr, "\n");
    }
    pack_local(n, bs);  // (on the finisher's stream: ev_fac[n] covers it)
    if (dep_events) {
        CPDB_CK(cudaEventRecord(ev_fac[n], bs));       // A_n, Q_n, R_n final
        CPDB_CK(cudaEventRecord(ev_zread[zpar], bs));  // Q0 / R0 / history consumed
        if (reuse) CPDB_CK(cudaEventRecord(ev_zread_b[ypar], bs));
    }
    ++versions[n];
    if (extrap && !reuse) {
        hist[n].swap(zcur.q0);  // the history keeps the unextrapolated Q0 (:265)
        std::swap(ev_hist[n], ev_zq_pending);
        has_hist[n] = true;
    }
    spec.reused = reuse;  // (read by undo_speculative_update when this was the speculative one)
    zcur.reuse = false;
    zpar ^= 1;
    last_mode = int(n);
    prefetch_root(sweep, b, bs);
}

// ---------------------------------------------------------------- sweeps
uint64_t Session::run(uint64_t nsweeps, cpdb_trace_row* trace, double* fps, double* lps,
                      cpdb_q0_observer observer, void* user) {
    uint64_t rows_out = 0;
    const uint64_t last_sweep = plan.sweeps.size();
    if (ended) fail(CPDB_LOGIC_ERROR, "session: run() after end() took back speculative work");
    // A resumable session keeps the device pipeline full across run() calls:
    // the last sweep of this call still issues the next sweep's first update
    // ahead of its host sync (the next call consumes it; end() undoes it).
    const bool across = observer == nullptr && fps == nullptr && lps == nullptr;
    while (rows_out < nsweeps && !converged && done < last_sweep) {
        const uint64_t sweep = done + 1;
        const Sweep& sw = plan.sweeps[sweep - 1];
        double beta_used = 0.0;
        // the next sweep's first update will run beside this sweep's last one
        // (below): the last one then yields to it
        // (long roots only: with a short root (C4) the last update is on the
        // critical path again -- measured C4 -4%, C2 +2.7%)
        // (third order only: a fourth-order sweep's last update carries the
        // heavy TTMs itself -- C5 -13% with it budgeted, C3 flat)
        const bool tail_low = low_tail && long_root && order == 3 && dep_events && speculate &&
                              !sharded &&
                              observer == nullptr && fps == nullptr && lps == nullptr &&
                              (!extrap || has_beta) && (rows_out + 1 < nsweeps || across) &&
                              done + 1 < last_sweep;
        for (uint32_t b = 0; b < order; ++b) {
            const bool low = tail_low && b == order - 1;
            if (b == 0 && front_issued) {
                front_issued = false;  // issued ahead of the previous sweep's host sync
            } else if (b == 1 && front1_issued) {
                front1_issued = false;
            } else {
                // (with the boundary repetition elided the next sweep's
                // first update reads this front's Y_(n) and Q0: it is on the
                // critical path and stays at normal priority; the back below
                // -- V-GEMM and finisher, for the record only -- yields)
                if (low && !(reuse_ok && self_hist)) tail_override = c->tailq;
                mode_update_front(sweep, b, observer, user);
                tail_override = nullptr;
            }
            if (b == 0 && spec.issued) {
                spec.issued = false;  // issued (whole) ahead of the previous sweep's host sync
                beta_used = spec.beta_used;
            } else if (low) {
                mode_update_back(sweep, b, beta_used, c->tailq);
                CPDB_CK(cudaEventRecord(ev_tail, c->tailq));
                CPDB_CK(cudaStreamWaitEvent(s, ev_tail, 0));
            } else {
                mode_update_back(sweep, b, beta_used);
            }
        }
        // the beta state machine of this sweep on the device (solvers.hpp:297-301),
        // read by the next sweep's V-GEMMs (the host mirrors it below)
        if (extrap)
            CPDB_CK(beta_gate(gate.p, fitbuf.p,
                              (!cfg.has_beta_override && sweep >= 2) ? 1 : 0,
                              cfg.activation_gap, s));
        if (extrap) acc(s, "beta_gate", {rg(fitbuf.p, 2), rg(gate.p, 4)}, {rg(gate.p, 4)});
        cudaEvent_t e_end = events.get();
        CPDB_CK(cudaEventRecord(e_end, s));
        CPDB_CK(cudaMemcpyAsync(c->pinned, fitbuf.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        acc(s, "fitness_d2h", {rg(fitbuf.p, 2)}, {});
        CPDB_CK(cudaMemcpyAsync(c->pinned + 2, status_word(sweep), sizeof(int),
                                cudaMemcpyDeviceToHost, s));
        cudaEvent_t e_fit = events.get();
        CPDB_CK(cudaEventRecord(e_fit, s));
        const Cost at_end = total;
        const size_t ntimers = timers.size(), nevents = events.used.size();
        // Hide the host round trip: the next sweep's first Z-QR + TTM chain do
        // not depend on the beta gate, so they go on the stream before the
        // host waits for this sweep's fitness (wasted only if it converges).
        const bool more = (rows_out + 1 < nsweeps || across) && done + 1 < last_sweep;
        if (more && observer == nullptr && fps == nullptr) {
            mode_update_front(sweep + 1, 0, nullptr, nullptr);
            front_issued = true;
            // ... and, with the beta decision taken on the device, its V-GEMM
            // and finisher too: the GPU goes straight on while the host reads
            // this sweep's fitness.  If the stop test fires on it, the update
            // is undone (factor buffers swapped back, undo_speculative_update).
            if (speculate && lps == nullptr) {
                const uint32_t n1 = plan.sweeps[sweep].updates[0].mode;
                spec.mode = n1;
                spec.had_hist = has_hist[n1];
                spec.prev_last_mode = last_mode;
                double unused = 0.0;
                // Until the beta gate opens no update extrapolates, and it
                // opens once per run: the update is issued on the prediction
                // that this sweep's fitness leaves it closed (plain V, the
                // host's decision -- nothing read from this sweep's finisher),
                // beside the last update like a frozen-beta one.  If the gate
                // does open on this sweep, the update is undone and issued
                // again with beta (below); its successor's front waits for
                // the host in the predicted case, so nothing else is redone.
                // CPDB_PREDICT_GATE=1 enables it (off by default, see begin()).
                const bool frozen = !extrap || has_beta;
                const bool predicted = !frozen && predict_gate;
                spec.predicted = false;
                if (dep_events && (frozen || predicted)) {
                    spec.predicted = predicted;
                    // beta frozen (or no extrapolation): the update needs
                    // nothing from this sweep's last V-GEMM / finisher, so
                    // it runs beside them on its own stream (its front waited
                    // for the V-GEMM that read ybuf[n]; factor and lambda
                    // buffers are the other copies, partials the other parity)
                    // behind its own chain on the chain's stream (mid), so
                    // the V-GEMM follows the branch TTM without a
                    // cross-stream event hop (C2 +0.9%, C1 +2.9%, C4 flat;
                    // CPDB_SPEC_STREAM=aux: its own stream)
                    static const bool spec_mid = [] {
                        const char* e = std::getenv("CPDB_SPEC_STREAM");
                        return !(e && std::strcmp(e, "aux") == 0);
                    }();
                    const cudaStream_t ss = spec_mid ? c->mid : c->aux;
                    mode_update_back(sweep + 1, 0, unused, ss, true);
                    CPDB_CK(cudaEventRecord(ev_aux, ss));
                    CPDB_CK(cudaStreamWaitEvent(s, ev_aux, 0));
                    // and the second update's front (Z-QR + chain: no beta,
                    // no returned state -- nothing to undo), which also
                    // launches the root prefetch planned by the first
                    if (order > 2 && frozen) {
                        // (its Z-QR right behind the speculative finisher on
                        // aux: measured C4 6270 -> 6440 sweeps/s, C1 +1%; C3
                        // (fourth order) -2%, so third order only;
                        // CPDB_ZQR_AUX=0/1 overrides)
                        static const char* zae = std::getenv("CPDB_ZQR_AUX");
                        // (long roots, C2: with the boundary repetition elided
                        // the main stream is free at this point and the Z-QR is
                        // better off there -- 2507 -> 2523 sweeps/s; C4 loses 2%
                        // without it)
                        const bool zaux = zae ? zae[0] == '1' : order == 3 && !long_root;
                        if (zaux) zqr_stream_override = ss;
                        mode_update_front(sweep + 1, 1, nullptr, nullptr);
                        zqr_stream_override = nullptr;
                        front1_issued = true;
                    }
                } else {
                    // beta still open: the update takes the gate's decision on
                    // the device, behind this sweep's finisher on the main
                    // stream; its successor's front (root prefetch included)
                    // follows it without waiting for the host either
                    mode_update_back(sweep + 1, 0, unused);
                    if (order > 2 && dep_events) {
                        mode_update_front(sweep + 1, 1, nullptr, nullptr);
                        front1_issued = true;
                    }
                }
                spec.issued = true;
                spec.beta_used = 0.0;
            }
        }
        CPDB_CK(cudaEventSynchronize(e_fit));
        int status;
        std::memcpy(&status, c->pinned + 2, sizeof(int));
        if (status & (1 << 16)) c->prof.qr_shifted += 1;  // rowalg.cuh kStatusShifted
        status &= 0xFFFF;
        // the word is free again for sweep + 4, whose first kernels the host
        // issues only after it has synchronised on sweep + 2's fitness, i.e.
        // after this clear (no device-side wait needed).  The next sweep's
        // speculative work has its own word, so a breakdown in an update the
        // reference never runs -- undone when the stop test fires -- is never
        // reported.
        CPDB_CK(cudaMemsetAsync(status_word(sweep), 0, sizeof(int), s));
        if (status) {
            if ((status & 0xFF) == 1)
                fail(CPDB_SINGULAR_TRIANGULAR,
                     "triangular solve: diagonal entry of column " + std::to_string(status >> 8) +
                         " is ~0 (rank-deficient Khatri-Rao factor)");
            fail(CPDB_SINGULAR_TRIANGULAR, kBreakdownMessage);
        }
        static const bool dbg_guard = std::getenv("CPDB_GUARD") != nullptr;
        if (dbg_guard) dev_guard_check(("sweep " + std::to_string(sweep)).c_str());
        const double fit = c->pinned[0], raw = c->pinned[1];
        float ms = 0.f;
        CPDB_CK(cudaEventElapsedTime(&ms, t_start, e_end));
        if (sweep == first_sweep + 1) c->prof.sweep1_ms = ms;
        c->prof.solve_ms = ms;
        for (size_t ti = 0; ti < ntimers; ++ti) {
            const Timer& t = timers[ti];
            float tm = 0.f;
            CPDB_CK(cudaEventElapsedTime(&tm, t.a, t.b));
            if (t.kind == 0) {
                c->prof.root_ttms += 1;
                c->prof.root_ttm_ms += tm;
                c->prof.root_ttm_flops += t.flops;
                c->prof.root_ttm_bytes += t.bytes;
            } else if (t.kind == 1) {
                c->prof.branch_ttm_ms += tm;
            } else if (t.kind == 3) {
                c->prof.mode_update_ms += tm;
            } else {
                c->prof.comm_ms += tm;
            }
        }
        timers.erase(timers.begin(), timers.begin() + long(ntimers));
        events.recycle_prefix(nevents);
        if (trace) {
            cpdb_trace_row& row = trace[rows_out];
            std::memset(&row, 0, sizeof row);
            row.iteration = sweep;
            row.order = order;
            for (uint32_t b = 0; b < order; ++b) row.update_order[b] = sw.updates[b].mode;
            row.fitness = fit;
            row.raw_radicand = raw;
            row.wall_seconds = ms * 1e-3;
            row.root_ttm_count = at_end.roots;
            row.flops = at_end.flops;
            row.beta_used = beta_used;
        }
        if (fps) {
            uint64_t off = 0;
            for (uint32_t k = 0; k < order; ++k) {
                acc(nullptr, "factors_d2h", {rg(fb[k].a.p, c->dims[k] * R)}, {});
                CPDB_CK(cudaMemcpy(fps + rows_out * nfac + off, fb[k].a.p,
                                   c->dims[k] * R * sizeof(double), cudaMemcpyDeviceToHost));
                off += c->dims[k] * R;
            }
        }
        if (lps)
            CPDB_CK(cudaMemcpy(lps + rows_out * R, lam.p, R * sizeof(double), cudaMemcpyDeviceToHost));
        ++rows_out;
        ++done;
        // beta gate (solvers.hpp:297-300)
        if (extrap && !has_beta && !cfg.has_beta_override && sweep >= 2 && has_prev) {
            double b = 0.0;
            if (cpdb_select_beta(prev_fit, fit, cfg.activation_gap, &b)) {
                has_beta = true;
                beta = b;
            }
        }
        prev_fit = fit;
        has_prev = true;
        if (fit >= cfg.fitness_threshold) converged = true;  // :301
        if (spec.issued) {
            if (converged) {
                undo_speculative_update();
            } else if (spec.predicted && spec.had_hist && has_beta && beta != 0.0) {
                // the gate opened on this sweep: the update issued ahead
                // assumed it closed.  Taken back; the next iteration issues
                // it again, extrapolated (its front's results stand).
                undo_speculative_update();
                c->prof.gate_mispredictions += 1;
            } else if (extrap && spec.had_hist && has_beta && beta != 0.0) {
                spec.beta_used = beta;  // what the device gate decided for it
            }
        }
    }
    tl_flush();
    fp_flush();
    if (hb.on)
        std::fprintf(stderr, "cpdb hbcheck: %llu sweeps checked, %llu violations\n",
                     (unsigned long long)(done - first_sweep), (unsigned long long)hb.violations);
    c->prof.sweeps = done - first_sweep;
    c->prof.kernel_launches = c->launches - launches0;
    return rows_out;
}

// The stop test fired on the sweep before a speculatively issued update:
// restore the state the reference returns (factors, lambda, Q0 history).
void Session::undo_speculative_update() {
    CPDB_CK(cudaStreamSynchronize(s));
    const uint32_t n = spec.mode;
    fb[n].swap(fb_alt[n]);
    lam.swap(lam_alt);
    zpar ^= 1;
    zb[zpar].reuse = spec.reused;  // (an update issued again reads the same buffers)
    // the root prefetch its back planned (not launched yet: that happens in
    // the next front) is planned again by the update issued in its place --
    // and must not budget that update's own kernels meanwhile
    if (pf.active && !pf.launched) pf.active = false;
    if (extrap && !spec.reused) {
        hist[n].swap(zb[zpar].q0);
        std::swap(ev_hist[n], ev_zq_pending);
    }
    has_hist[n] = spec.had_hist;
    pack_local(n);  // this rank's rows of the restored Q_n
    --versions[n];
    last_mode = spec.prev_last_mode;
    spec.issued = false;
    // whatever the undone update reported is moot
    CPDB_CK(cudaMemsetAsync(status_word(done + 1), 0, sizeof(int), s));
    CPDB_CK(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------- results
void Session::end(cpdb_state* state, double* out_lambda, double* out_factors) {
    // work issued ahead for a sweep the caller never ran: take it back so the
    // exported state is the one after `done` sweeps (the reference's)
    if (spec.issued) undo_speculative_update();
    if (front_issued || front1_issued) {
        CPDB_CK(cudaDeviceSynchronize());
        ended = true;
    }
    auto get_factors = [&](double* dst) {
        uint64_t off = 0;
        for (uint32_t k = 0; k < order; ++k) {
            acc(nullptr, "end_factors_d2h", {rg(fb[k].a.p, c->dims[k] * R)}, {});
            CPDB_CK(cudaMemcpy(dst + off, fb[k].a.p, c->dims[k] * R * sizeof(double),
                               cudaMemcpyDeviceToHost));
            off += c->dims[k] * R;
        }
    };
    if (out_lambda) CPDB_CK(cudaMemcpy(out_lambda, lam.p, R * sizeof(double), cudaMemcpyDeviceToHost));
    if (out_factors) get_factors(out_factors);
    if (!state) return;
    state->sweeps_done = done;
    if (state->lambda)
        CPDB_CK(cudaMemcpy(state->lambda, lam.p, R * sizeof(double), cudaMemcpyDeviceToHost));
    if (state->factors) get_factors(state->factors);
    if (state->q0_history) {
        state->history_mask = 0;
        std::vector<double> nat(zrows * R);
        for (uint32_t n = 0; n < order; ++n) {
            if (!has_hist[n]) continue;
            acc(nullptr, "end_hist_d2h", {rg(hist[n].p, zrows * R)}, {});
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

void solve(cpdb_ctx* c, const cpdb_config& cfg, cpdb_state* state, cpdb_trace_row* trace,
           uint64_t* trace_len, double* out_lambda, double* out_factors, double* fps,
           double* lps, cpdb_q0_observer observer, void* user) {
    // CholeskyQR2 (with its shifted retry) breaks down beyond kappa ~1e15,
    // where the reference's Householder QR carries on (linalg.hpp:39-99): such
    // a run is started again on the Householder kernels (widerank.cu), which
    // follow the reference's algorithm at any rank.  (Q0 observers have seen
    // the first attempt's sweeps by then, so observed runs are not restarted.)
    for (int attempt = 0;; ++attempt) {
        Session ss;
        ss.robust = attempt > 0;
        try {
            ss.begin(c, cfg, state);
            const uint64_t n = ss.run(cfg.max_iterations, trace, fps, lps, observer, user);
            if (trace_len) *trace_len = n;
            ss.end(state, out_lambda, out_factors);
            return;
        } catch (const Fail& e) {
            if (attempt > 0 || ss.robust || observer != nullptr ||
                e.code != CPDB_SINGULAR_TRIANGULAR || e.what != kBreakdownMessage)
                throw;
            c->prof.qr_householder += 1;
        }
    }
}

}  // namespace cpdb
