// Sharding planner for mode-0 sharded runs (the reference is
// single-process, so this has no reference counterpart).
//
// X is split into equal slabs of mode-0 rows.  Every intermediate Y(S) of
// the plan gets a layout: replicated, sharded along one of its free modes, or
// a per-rank PARTIAL SUM (TTMs are linear, so contracting the sharded mode
// yields partial sums that may travel further before being reduced).  A TTM
// on a sharded source keeps the shard unless it contracts the shard mode;
// that step's output is partial and one of three things happens to it:
//   all-reduce       -> replicated (eager: every later step runs full-size
//                       on every rank),
//   reduce-scatter   -> sharded along another free mode (later steps stay
//                       divided; the scattered mode's own contraction makes
//                       a smaller partial later),
//   nothing (lazy)   -> partial; later TTMs run full-size on the partials
//                       and the reduction happens further down -- at the
//                       latest on V = Y_(n) Q0 (I_n x R), the smallest point.
// V of a sharded Y(n) holds this rank's rows and is all-gathered; V of a
// partial Y(n) is all-reduced.
//
// Policy kAuto chooses per step by a cost model (per-rank seconds: FP64
// flops at `tflops`, collective bytes at `bus_gbs` NCCL bus bandwidth plus a
// per-call latency) over the step's whole consumer tree in the plan (a slot
// produced once is read by every later step until it is produced again), by
// memoised recursion.  The other policies fix the choice (kScatter falls back
// to an all-reduce when no free mode divides by the world size).
#include <cmath>
#include <map>

#include "schedule.hpp"

namespace cpdb {
namespace {

struct Ctx {
    const Plan& p;
    const std::vector<uint64_t>& dims;
    uint64_t R;
    int P;
    ShardPolicy pol;
    ShardCost cp;
    // flattened steps
    struct FS {
        uint64_t sweep;
        uint32_t block, mode;
        size_t idx;  // step within the update
        Step st;
        bool last;   // the update's last step (produces Y(n))
    };
    std::vector<FS> fs;
    std::map<std::pair<size_t, int>, double> memo;

    // global extents of a mode set's tensor: free modes keep I_k, others R
    uint64_t words(ModeSet s) const {
        uint64_t w = 1;
        for (uint32_t k = 0; k < p.order; ++k) w *= (s & (1u << k)) ? dims[k] : R;
        return w;
    }
    double ttm_flops(const Step& st) const {
        return 2.0 * double(words(st.produces)) *
               double((st.source & (1u << st.contract)) ? dims[st.contract] : R);
    }
    double t_flops(double f) const { return f / (cp.tflops * 1e12); }
    double t_allreduce(double w) const {
        return P > 1 ? cp.latency_s + 2.0 * (P - 1) / P * 8.0 * w / (cp.bus_gbs * 1e9) : 0.0;
    }
    double t_scatter(double w) const {
        return P > 1 ? cp.latency_s + double(P - 1) / P * 8.0 * w / (cp.bus_gbs * 1e9) : 0.0;
    }
    double t_gather(double w) const { return t_scatter(w); }
    bool divisible(uint32_t m) const { return dims[m] % uint64_t(P) == 0; }
    static int key(const ShardLayout& l) { return l.kind * 16 + (l.mode + 1); }

    // raw output layout of a step on a source of layout L
    ShardLayout raw(const ShardLayout& L, uint32_t c) const {
        if (L.kind == kLayShard && uint32_t(L.mode) == c) return {kLayPartial, -1};
        return L;
    }
    // the free mode a reduce-scatter of a partial over set s goes onto: the
    // divisible free mode with the fewest outer slices (one collective each)
    int scatter_mode(ModeSet s) const {
        for (uint32_t k = 0; k < p.order; ++k)
            if ((s & (1u << k)) && divisible(k)) return int(k);
        return -1;
    }
    // V-GEMM (2 I_n R^(N-1) R flops) and its collective for Y(n) of layout L
    double v_cost(uint32_t n, const ShardLayout& L, bool dual) const {
        double f = 2.0 * double(dims[n]) * double(words(0)) * (dual ? 2.0 : 1.0);
        const double vw = double(dims[n]) * R * (dual ? 2.0 : 1.0);
        if (L.kind == kLayShard) return t_flops(f / P) + t_gather(vw);
        if (L.kind == kLayPartial) return t_flops(f) + t_allreduce(vw);
        return t_flops(f);
    }
    // consumers of step i's output (until the set is produced again)
    std::vector<size_t> consumers(size_t i) const {
        std::vector<size_t> out;
        const ModeSet s = fs[i].st.produces;
        if (fs[i].last) return out;
        for (size_t j = i + 1; j < fs.size(); ++j) {
            if (fs[j].st.source == s) out.push_back(j);
            if (fs[j].st.produces == s && !fs[j].last) break;
        }
        return out;
    }
    // seconds per rank of everything downstream of step i whose stored
    // output has layout L (its consumers' TTMs, their reductions, V)
    double downstream(size_t i, const ShardLayout& L) {
        const auto k = std::make_pair(i, key(L));
        auto it = memo.find(k);
        if (it != memo.end()) return it->second;
        double t = 0.0;
        if (fs[i].last) {
            t = v_cost(fs[i].mode, L, false);
        } else {
            for (size_t j : consumers(i)) t += step_cost(j, L, nullptr);
        }
        memo[k] = t;
        return t;
    }
    // cost of step j (source layout L) plus its downstream, with the best
    // (or policy-fixed) reduction; fills `choice` when given
    double step_cost(size_t j, const ShardLayout& L, StepShard* choice) {
        const Step& st = fs[j].st;
        const ShardLayout r = raw(L, st.contract);
        const double comp = t_flops(ttm_flops(st) / (L.kind == kLayShard ? P : 1));
        StepShard best{L, r, kRedNone, -1, 0};
        double best_t = 0.0;
        if (r.kind != kLayPartial) {
            best_t = comp + downstream(j, r);
        } else {
            const double w = double(words(st.produces));
            const bool fresh = L.kind != kLayPartial;  // the partial is created here
            // candidates
            struct Cand { int red; ShardLayout out; double comm; };
            std::vector<Cand> cand;
            const int sm = scatter_mode(st.produces);
            switch (pol) {
                case kPolicyEager:
                    cand.push_back({kRedAllReduce, {kLayRep, -1}, t_allreduce(w)});
                    break;
                case kPolicyScatter:
                    if (sm >= 0)
                        cand.push_back({kRedScatter, {kLayShard, sm}, t_scatter(w)});
                    else
                        cand.push_back({kRedAllReduce, {kLayRep, -1}, t_allreduce(w)});
                    break;
                case kPolicyLazy:
                    cand.push_back({kRedNone, r, 0.0});
                    break;
                default:
                    cand.push_back({kRedAllReduce, {kLayRep, -1}, t_allreduce(w)});
                    if (sm >= 0) cand.push_back({kRedScatter, {kLayShard, sm}, t_scatter(w)});
                    cand.push_back({kRedNone, r, 0.0});
                    break;
            }
            (void)fresh;
            best_t = -1.0;
            for (const Cand& c : cand) {
                const double t = comp + c.comm + downstream(j, c.out);
                if (best_t < 0.0 || t < best_t - 1e-12) {
                    best_t = t;
                    best = StepShard{L, c.out, c.red, c.red == kRedScatter ? c.out.mode : -1,
                                     c.red == kRedNone ? 0 : uint64_t(w)};
                }
            }
        }
        if (choice) *choice = best;
        return best_t;
    }
};

}  // namespace

ShardPlan plan_shards(const Plan& p, const std::vector<uint64_t>& dims, uint64_t R, int world,
                      ShardPolicy pol, const ShardCost& cp) {
    Ctx c{p, dims, R, world < 1 ? 1 : world, pol, cp, {}, {}};
    for (uint64_t i = 0; i < p.sweeps.size(); ++i)
        for (uint32_t b = 0; b < p.sweeps[i].updates.size(); ++b) {
            const Update& u = p.sweeps[i].updates[b];
            for (size_t j = 0; j < u.steps.size(); ++j)
                c.fs.push_back({i, b, u.mode, j, u.steps[j], j + 1 == u.steps.size()});
        }
    ShardPlan out;
    out.steps.resize(p.sweeps.size());
    out.updates.resize(p.sweeps.size());
    for (uint64_t i = 0; i < p.sweeps.size(); ++i) {
        out.steps[i].resize(p.sweeps[i].updates.size());
        out.updates[i].resize(p.sweeps[i].updates.size());
    }
    // forward pass: the layout of every stored slot follows from the choices
    std::map<ModeSet, ShardLayout> slot;
    const ModeSet root = p.root();
    const ShardLayout xl = world > 1 ? ShardLayout{kLayShard, 0} : ShardLayout{kLayRep, -1};
    for (size_t i = 0; i < c.fs.size(); ++i) {
        const auto& f = c.fs[i];
        ShardLayout L = f.st.source == root ? xl : slot.at(f.st.source);
        StepShard ch{};
        if (world > 1) {
            c.step_cost(i, L, &ch);
        } else {
            ch = StepShard{L, L, kRedNone, -1, 0};
        }
        const double fl = c.ttm_flops(f.st) / (L.kind == kLayShard ? c.P : 1);
        out.est_compute_s += c.t_flops(fl);
        if (ch.red == kRedAllReduce) out.est_comm_s += c.t_allreduce(double(ch.words));
        if (ch.red == kRedScatter) out.est_comm_s += c.t_scatter(double(ch.words));
        out.steps[f.sweep][f.block].push_back(ch);
        if (f.last) {
            UpdateShard& us = out.updates[f.sweep][f.block];
            us.yn = ch.out;
            const double vw = double(dims[f.mode]) * R;
            us.vop = ch.out.kind == kLayShard ? kVGather
                     : ch.out.kind == kLayPartial ? kVAllReduce : kVNone;
            us.vwords = us.vop == kVNone ? 0 : uint64_t(vw);
            if (us.vop == kVGather) out.est_comm_s += c.t_gather(vw);
            if (us.vop == kVAllReduce) out.est_comm_s += c.t_allreduce(vw);
            out.est_compute_s += c.t_flops(2.0 * double(dims[f.mode]) * double(c.words(0)) /
                                           (ch.out.kind == kLayShard ? c.P : 1));
        } else {
            slot[f.st.produces] = ch.out;
        }
    }
    return out;
}

}  // namespace cpdb
