// Solver session: the device-resident run_qr state between calls.
#pragma once

#include <cstdint>
#include <map>
#include <vector>

#include "hb.hpp"
#include "runtime.hpp"

namespace cpdb {

struct EventPool {
    std::vector<cudaEvent_t> free_, used;
    cudaEvent_t get();
    void recycle();
    void recycle_prefix(size_t n);  // the first n events handed out since the last recycle
    ~EventPool();
};

struct FactorBufs {
    DevBuf a, q, qp, r;  // A_n, Q_n, packed Q_n, R_n
    void swap(FactorBufs& o) noexcept {
        a.swap(o.a);
        q.swap(o.q);
        qp.swap(o.qp);
        r.swap(o.r);
    }
};

struct Session {
    cpdb_ctx* c = nullptr;
    cpdb_config cfg{};
    Plan plan;
    uint32_t order = 0, R = 0, Rp = 0;
    bool extrap = false, sharded = false;
    uint64_t done = 0, first_sweep = 0;
    uint64_t zrows = 1, maxI = 0, nfac = 0;
    double nx2 = 0.0;
    cudaStream_t s = nullptr;
    uint64_t launches0 = 0;

    std::vector<FactorBufs> fb;
    // A mode update writes the OTHER copy of its factor buffers and of lambda
    // and swaps them in after the launch, so a speculatively issued update
    // (the next sweep's first, before the host has read this sweep's fitness)
    // can be undone by swapping back when the stop test fires.
    std::vector<FactorBufs> fb_alt;
    DevBuf lam, lam_alt, tsbuf, zts;
    // sharded runs: the layout / reduction plan of every step
    // (shard.cpp), this rank's packed rows of each split Q_m, and the whole
    // partial of a step whose output is reduce-scattered
    ShardPlan splan;
    std::vector<bool> need_local;
    std::vector<DevBuf> qp_local;
    std::map<cudaStream_t, DevBuf> rs_tmp;  // per producing stream
    uint32_t rs_chunks = 4;      // CPDB_RS_CHUNKS
    double rs_min_flops = 2e8;   // CPDB_RS_MIN_FLOPS
    std::map<cudaStream_t, DevBuf> qcol_tmp;  // packed column halves of Q (ttm_step)
    DevBuf gate;  // {has_beta, beta, has_prev, prev_fitness} on the device (beta_gate)
    // the next sweep's first update issued before the host read this sweep's
    // fitness (Session::run); what undoing it needs
    struct Spec {
        bool issued = false;
        uint32_t mode = 0;
        bool had_hist = false;  // has_hist[mode] before it (extrapolation possible)
        int prev_last_mode = -1;
        double beta_used = 0.0;  // its trace contribution, once the host knows the gate
        bool reused = false;     // it took the previous update's Y_(n) / Q0 (no history swap)
        bool predicted = false;  // issued on the prediction that the beta gate stays closed
    } spec;
    bool speculate = false;  // CPDB_SPECULATE=0 turns it off
    bool self_hist = true;   // CPDB_SELF_HIST=0: always wait for the history's own Z-QR
    // The sweep's last update while the next sweep's first update runs beside
    // it (beta frozen): off the critical path (it only yields this sweep's
    // fitness), so its chain, V-GEMM and finisher go on c->tailq, below the
    // next update's kernels (CPDB_LOW_TAIL=0: off)
    bool low_tail = true;
    bool long_root = false;  // the root TTM takes >= 150 us (estimate)
    int tail_sms = 80;       // CPDB_TAIL_SMS: SM budget of the low tail's TTMs / V-GEMM
    cudaStream_t tail_override = nullptr;
    // Device status words (Cholesky breakdown / singular R0), a ring of four:
    // a sweep's kernels write word 1 + (sweep & 3), the host reads it when it
    // consumes that sweep and then clears it (Session::run)
    int* status_word(uint64_t sweep) const { return c->dstatus + 1 + (sweep & 3); }
    uint64_t fault_sweep = 0;  // CPDB_FAULT_SWEEP=k: test hook, a breakdown in sweep k's first update
    cudaEvent_t ev_tail = nullptr;
    DevBuf fscratch[2], vpart[2], vfitpart[2], vfull[2], vfitfull[2], vout, fitbuf;
    // Z-QR outputs, double-buffered so the next update's Z-QR can run while
    // this update's V-GEMM / finisher still read Q0 and R0
    struct ZBuf {
        DevBuf q0, q1, r0, work;
        // the previous update was of the same mode (sweep boundary): no R_k
        // it reads changed since that update's Z-QR, so its Q0 -- this
        // mode's extrapolation history -- equals this Z-QR's Q0 bit for bit
        bool hist_is_self = false;
        // this update takes the previous update's Y_(n), Q0 and R0 (the
        // other parity's buffers): the sweep boundary repeats the mode with
        // unchanged inputs, see mode_update_front
        bool reuse = false;
    } zb[2];
    // What the last front computed, to recognise a repetition: mode, the
    // single chain step that produced Y_(n) straight from a cached source
    // (key, contracted mode, the source's buffer and stamps) and the factor
    // versions its Z-QR and chain read
    struct LastFront {
        bool valid = false;
        uint32_t mode = 0, source = 0, contract = 0;
        const double* src_buf = nullptr;
        std::vector<uint64_t> src_stamps, versions;
    } prev_front;
    bool reuse_ok = true;  // CPDB_REUSE_BOUNDARY=0: recompute (A/B testing)
    bool predict_gate = false;  // CPDB_PREDICT_GATE=1: pre-activation updates issued on "the gate stays closed"
    int zpar = 0;  // parity of the update in flight (set by the front, used by the back)
    // Dependency events of the event-driven schedule (dep_events): the
    // finisher that last updated each mode, the V-GEMM that last read ybuf[n],
    // the last readers of each Z-QR buffer set, and the front's joins
    bool dep_events = false;
    // ev_v[2n + parity]: the V-GEMM that last read ybuf[2n + parity]
    cudaEvent_t ev_fac[CPDB_MAX_ORDER] = {}, ev_v[2 * CPDB_MAX_ORDER] = {}, ev_zread[2] = {};
    // second readers of the same buffers: an update that repeats the previous
    // one reads its Y_(n) / Q0 / R0 from another stream (zb[].reuse)
    cudaEvent_t ev_v_b[2 * CPDB_MAX_ORDER] = {}, ev_zread_b[2] = {};
    std::map<uint32_t, cudaEvent_t> slot_ready;  // cache slot -> its producer done
    // ev_hist[n]: the Z-QR that produced hist[n] (the Q0 history of mode n);
    // ev_zq_pending: this update's Z-QR, swapped into ev_hist[n] by its back
    cudaEvent_t ev_hist[CPDB_MAX_ORDER] = {}, ev_zq_pending = nullptr;
    cudaEvent_t ready_event(uint32_t key);
    cudaEvent_t ev_zq = nullptr, ev_aux = nullptr;
    int last_mode = -1;   // mode of the last update issued (back)
    cudaStream_t zqr_stream_override = nullptr;  // (run: the speculative second front)
    bool early = false;   // this update's front runs event-driven (set by the front)
    bool chain_events = false;  // CPDB_CHAIN_EVENTS: every chain step waits only for its Q_c
    cudaStream_t side = nullptr;  // c->side, or c->side_hi for a tall Z
    std::vector<DevBuf> hist, ybuf;
    std::vector<bool> has_hist;
    std::vector<uint64_t> versions;
    std::vector<uint64_t> perm;
    std::map<uint32_t, Slot> cache;

    bool has_beta = false, has_prev = false, converged = false;
    double beta = 0.0, prev_fit = 0.0;
    Cost total;

    EventPool events;
    HbCheck hb;  // CPDB_HBCHECK=1: happens-before check of every declared access
    // CPDB_FINGERPRINT=<file>: hash every declared input before and after each
    // launch and every output after it, appended to <file> at the end of run()
    const char* fpath = nullptr;
    bool fp_light = false;  // CPDB_FINGERPRINT_LIGHT=1: outputs of zqr / vgemm / finish only
    DevBuf fplog;
    std::vector<std::string> fplabels;
    void fp(cudaStream_t st, const char* what, const char* phase,
            std::initializer_list<HbCheck::Rg> regions);
    // hb.op + fingerprints of the inputs and outputs after the launch
    void acc(cudaStream_t st, const char* what, std::initializer_list<HbCheck::Rg> rd,
             std::initializer_list<HbCheck::Rg> wr) {
        hb.op(st, what, rd, wr);
        // (legacy-stream accesses are blocking cudaMemcpy calls: the host has
        // synchronised with them when they return)
        if (st == nullptr) hb.sync_stream(nullptr);
        if (fpath) {
            if (!fp_light || what[0] == 'v') fp(st, what, "in_after", rd);
            fp(st, what, "out", wr);
        }
    }
    void fp_flush();
    bool front_issued = false;  // next sweep's first Z-QR + TTM chain already on the stream
    // root TTM of a later update of the sweep issued early on the low-priority
    // stream, overlapped with the updates in between (prefetch_root)
    struct Prefetch {
        bool active = false;
        uint64_t sweep = 0;
        uint32_t block = 0;
        int sms = 0;  // SM budget of the updates it overlaps (0: all SMs)
        uint32_t cm = 0;        // contracted mode
        uint32_t tpc = 2;       // tiles per CTA of its non-persistent grid
        bool launched = false;  // planned at update b's end, launched behind the
                                // next update's Z-QR (launch_prefetch)
        cudaEvent_t ev = nullptr;
    } pf;
    void launch_prefetch();
    // CholeskyQR kernels replaced by the Householder ones (widerank.cu) at any
    // rank: set by solve() when a run broke down, or CPDB_HOUSEHOLDER=1
    bool robust = false;
    bool ended = false;          // end() took back work issued ahead: no further run()
    bool front1_issued = false;  // next sweep's second front issued ahead (Session::run)
    DevBuf pre;
    cudaEvent_t ev_fin = nullptr;
    bool prefetch_enabled = false;
    bool chain_side = false;  // TTM chain on the side stream, Z-QR on the main one
    // SM budget of the branch TTMs and the V-GEMM of an update that runs
    // while a prefetched root TTM is in flight (0: all SMs)
    int overlap_sms = -1;  // CPDB_OVERLAP_SMS: fixed budget (-1: per root, see prefetch_root)
    int budget(uint64_t sweep, uint32_t b) const {
        return (pf.active && pf.sweep == sweep && pf.block > b) ? pf.sms : 0;
    }
    double step_flops(const Step& st) const;
    // tall Z (multi-kernel Z-QR, C5): the TTM chain runs one tile per CTA on
    // the mid-priority stream so the Z-QR's CTAs take SMs as tiles retire
    // instead of waiting for a persistent grid to drain (CPDB_ZQR_YIELD=1; off by
    // default: measured at C5 the one-tile TTMs lose more than the Z-QR gains)
    bool zqr_yield = false;
    bool yield_now = false;
    std::vector<Timer> timers;
    cudaEvent_t t_start = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_zqr = nullptr;  // main -> side -> main fork/join
    // CPDB_TIMELINE=<csv>: an event pair around every launch site, written
    // at the end of run() (diagnostic: the events cost PDL overlap)
    struct Mark {
        const char* label;
        int stream;  // 0 main, 1 side, 2 low priority
        uint64_t sweep;
        uint32_t mode;
        cudaEvent_t a, b;
    };
    const char* timeline = nullptr;
    std::vector<Mark> marks;
    uint64_t tl_sweep = 0;
    uint32_t tl_mode = 0;
    cudaEvent_t tl_begin(cudaStream_t st);
    void tl_end(cudaEvent_t a, cudaStream_t st, const char* label);
    void tl_flush();

    ~Session();
    void begin(cpdb_ctx* ctx, const cpdb_config& cfg, const cpdb_state* state);
    // Runs up to n sweeps (stops early on convergence or at max_iterations);
    // returns the number of trace rows written.
    uint64_t run(uint64_t n, cpdb_trace_row* trace, double* fps, double* lps,
                 cpdb_q0_observer observer, void* user);
    void end(cpdb_state* state, double* out_lambda, double* out_factors);

private:
    std::vector<uint64_t> local_dims_of(uint32_t key) const;
    void qr_factor(uint32_t k);
    void pack_local(uint32_t m, cudaStream_t st = nullptr);
    uint64_t shard_rows_of(uint32_t m) const;
    std::vector<uint64_t> dims_in(uint32_t key, const ShardLayout& L) const;
    void ttm_step(const double* src, const std::vector<uint64_t>& sd, const StepShard* sh,
                  uint32_t k, double* dst, bool is_root, cudaStream_t st = nullptr,
                  bool prefetch = false, bool no_pdl = false, int sms = 0);
    void prefetch_root(uint64_t sweep, uint32_t b, cudaStream_t after);
    void mode_update(uint64_t sweep, uint32_t b, cpdb_q0_observer observer, void* user,
                     double& beta_used);
    void mode_update_front(uint64_t sweep, uint32_t b, cpdb_q0_observer observer, void* user);
    // bs: the stream of the V-GEMM and finisher (default: the main one);
    // host_beta: the host's beta decision is final (frozen gate), no device gate read
    void mode_update_back(uint64_t sweep, uint32_t b, double& beta_used, cudaStream_t bs = nullptr,
                          bool host_beta = false);
    void undo_speculative_update();
    Timer tail_timer_begin(cudaStream_t st);
    void tail_timer_end(Timer& t, cudaStream_t st);
};

}  // namespace cpdb

struct cpdb_session {
    cpdb::Session s;
};
