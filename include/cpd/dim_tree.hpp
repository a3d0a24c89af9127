// Drop-in for /root/reference/proj/include/cpd/dim_tree.hpp on libcpdb.
//
// Schedule data types and the cache keep the reference's API (dim_tree.hpp:
// 25-178).  The plans themselves, their validation and the eviction
// look-ahead come from the library's native scheduler (csrc/schedule.cpp via
// cpdb_schedule_build / _validate / cpdb_retained_keys), so the device solver
// and this header can never disagree about a plan.  execute() (dim_tree.hpp:
// 473-544) is the host-typed "test path" of SURVEY.md 8b: every scheduled TTM
// runs on the device (cpdb_ttm) while the freshness stamps, cost accounting
// and eviction stay on the host exactly as in the reference.  Production
// sweeps never come through here: cp_als_qr / als_qr_bre keep X and the cache
// resident in HBM (solvers.hpp drop-in).
#pragma once

#include <bit>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "cpd/abi.hpp"
#include "cpd/factor_state.hpp"
#include "cpd/tensor.hpp"

namespace cpd {

enum class Strategy { naive, dim_tree, branch_reuse };

inline const char* strategy_name(Strategy s) {
    if (s == Strategy::naive) return "naive";
    if (s == Strategy::dim_tree) return "dim-tree";
    if (s == Strategy::branch_reuse) return "branch-reuse";
    return "?";
}

// Bit m set = mode m is still free (not yet contracted).
using ModeSet = std::uint32_t;

inline ModeSet mode_bit(std::size_t mode) { return ModeSet(1u) << mode; }
inline ModeSet full_set(std::size_t order) { return ModeSet((1u << order) - 1u); }

// "Y(1,3)": 1-based free modes, as the reference prints them.
inline std::string mode_set_name(ModeSet set, std::size_t order) {
    std::string name;
    for (std::size_t m = 0; m < order; ++m)
        if (set & mode_bit(m)) name += (name.empty() ? "" : ",") + std::to_string(m + 1);
    return "Y(" + name + ")";
}

struct ContractionStep {
    ModeSet source;
    std::size_t contract_mode;
    ModeSet produces;
};

struct ModeUpdate {
    std::size_t mode;
    std::vector<ContractionStep> steps;
};

struct ScheduleIteration {
    std::vector<ModeUpdate> updates;
};

class Schedule {
public:
    Schedule(std::size_t order, Strategy strategy, std::vector<ScheduleIteration> iterations,
             std::size_t cycle_start, std::size_t cycle_length)
        : order_(order),
          strategy_(strategy),
          its_(std::move(iterations)),
          cycle_start_(cycle_start),
          cycle_length_(cycle_length) {}

    std::size_t order() const { return order_; }
    Strategy strategy() const { return strategy_; }
    std::size_t num_iterations() const { return its_.size(); }
    std::size_t cycle_start() const { return cycle_start_; }
    std::size_t cycle_length() const { return cycle_length_; }
    const ScheduleIteration& iteration(std::size_t i) const { return its_.at(i); }
    std::vector<std::size_t> update_order(std::size_t i) const {
        std::vector<std::size_t> modes;
        for (const ModeUpdate& u : iteration(i).updates) modes.push_back(u.mode);
        return modes;
    }

private:
    std::size_t order_;
    Strategy strategy_;
    std::vector<ScheduleIteration> its_;
    std::size_t cycle_start_, cycle_length_;
};

class IntermediateCache {
public:
    struct Entry {
        DenseTensor tensor;
        std::map<std::size_t, std::uint64_t> stamps;  // contracted mode -> version absorbed
    };

    const Entry* find(ModeSet key) const {
        const auto it = map_.find(key);
        return it == map_.end() ? nullptr : &it->second;
    }
    void put(ModeSet key, Entry entry) { map_[key] = std::move(entry); }
    template <typename Pred>
    void evict_unless(Pred keep) {
        std::erase_if(map_, [&](const auto& kv) { return !keep(kv.first); });
    }
    void clear() { map_.clear(); }
    std::size_t size() const { return map_.size(); }

private:
    std::unordered_map<ModeSet, Entry> map_;
};

struct CostReport {
    struct Bucket {
        std::uint64_t count = 0;
        std::uint64_t flops = 0;
    };
    // key: (power of R in the step's flop count, free modes of the source)
    std::map<std::pair<std::size_t, ModeSet>, Bucket> categories;
    std::uint64_t root_ttm_count = 0;
    std::uint64_t total_flops = 0;

    void add(ModeSet i_modes, std::size_t r_power, std::uint64_t flops, bool root) {
        Bucket& b = categories[{r_power, i_modes}];
        ++b.count;
        b.flops += flops;
        total_flops += flops;
        root_ttm_count += root ? 1 : 0;
    }
    void merge(const CostReport& other) {
        for (const auto& [key, b] : other.categories) {
            Bucket& mine = categories[key];
            mine.count += b.count;
            mine.flops += b.flops;
        }
        root_ttm_count += other.root_ttm_count;
        total_flops += other.total_flops;
    }
    // "2*I1*I2*R^2"
    static std::string category_label(std::pair<std::size_t, ModeSet> key, std::size_t order) {
        std::string label = "2";
        for (std::size_t m = 0; m < order; ++m)
            if (key.second & mode_bit(m)) label += "*I" + std::to_string(m + 1);
        return label + (key.first == 1 ? std::string("*R") : "*R^" + std::to_string(key.first));
    }
};

namespace detail {

inline ContractionStep step(ModeSet source, std::size_t contract) {
    return {source, contract, ModeSet(source & ~mode_bit(contract))};
}

inline ModeSet bits(std::initializer_list<std::size_t> modes) {
    ModeSet s = 0;
    for (const std::size_t m : modes) s |= mode_bit(m);
    return s;
}

inline ModeUpdate make_update(std::size_t mode, std::initializer_list<ContractionStep> steps) {
    return {mode, std::vector<ContractionStep>(steps)};
}

// {iteration, block, mode, source, contract, produces} rows for the C ABI.
inline std::vector<int64_t> flatten(const Schedule& s) {
    std::vector<int64_t> rows;
    for (std::size_t i = 0; i < s.num_iterations(); ++i) {
        const auto& ups = s.iteration(i).updates;
        for (std::size_t b = 0; b < ups.size(); ++b)
            for (const ContractionStep& st : ups[b].steps)
                rows.insert(rows.end(), {int64_t(i), int64_t(b), int64_t(ups[b].mode),
                                         int64_t(st.source), int64_t(st.contract_mode),
                                         int64_t(st.produces)});
    }
    return rows;
}

// Structure + version simulation (dim_tree.hpp:335-379); throws
// stale_intermediate_error / std::logic_error / std::invalid_argument.
inline void validate_schedule(const Schedule& s) {
    for (std::size_t i = 0; i < s.num_iterations(); ++i)
        for (const ModeUpdate& u : s.iteration(i).updates)
            if (u.steps.empty())  // (not representable in the ABI's step rows)
                throw std::logic_error("schedule: update must end in its final tensor");
    const std::vector<int64_t> rows = flatten(s);
    abi::check(cpdb_schedule_validate(uint32_t(s.order()), rows.data(), rows.size() / 6,
                                      s.num_iterations()));
}

// Cache keys still read after `block` of iteration `iter` (dim_tree.hpp:433-465).
inline std::vector<ModeSet> retained_keys(const Schedule& s, std::size_t iter, std::size_t block) {
    const std::vector<int64_t> rows = flatten(s);
    uint32_t keys[256];
    uint64_t n = 0;
    abi::check(cpdb_retained_keys(uint32_t(s.order()), rows.data(), rows.size() / 6,
                                  s.num_iterations(), s.cycle_start(), s.cycle_length(), iter,
                                  block, keys, 256, &n));
    return std::vector<ModeSet>(keys, keys + (n < 256 ? n : 256));
}

}  // namespace detail

inline Schedule build_schedule(std::size_t order, Strategy strategy, std::size_t num_iterations) {
    uint64_t n = 0, cycle[2] = {0, 1};
    const int32_t st = int32_t(strategy);
    abi::check(cpdb_schedule_build(uint32_t(order), st, num_iterations, nullptr, 0, &n, cycle));
    std::vector<int64_t> rows(6 * n);
    abi::check(cpdb_schedule_build(uint32_t(order), st, num_iterations, rows.data(), n, &n, cycle));
    std::vector<ScheduleIteration> its(num_iterations);
    for (uint64_t k = 0; k < n; ++k) {
        const int64_t* r = &rows[6 * k];
        auto& ups = its[std::size_t(r[0])].updates;
        if (ups.size() <= std::size_t(r[1])) ups.resize(std::size_t(r[1]) + 1);
        ModeUpdate& u = ups[std::size_t(r[1])];
        u.mode = std::size_t(r[2]);
        u.steps.push_back({ModeSet(r[3]), std::size_t(r[4]), ModeSet(r[5])});
    }
    return Schedule(order, strategy, std::move(its), cycle[0], cycle[1]);
}

// One ModeUpdate of the schedule: returns Y for `mode` and the step costs.
inline std::pair<DenseTensor, CostReport> execute(const Schedule& schedule, const DenseTensor& x,
                                                  const FactorState& state,
                                                  IntermediateCache& cache,
                                                  std::size_t iteration, std::size_t mode) {
    const std::size_t order = schedule.order();
    if (x.order() != order || state.order() != order)
        throw std::invalid_argument("execute: order mismatch");
    const auto& ups = schedule.iteration(iteration).updates;
    std::size_t block = ups.size();
    for (std::size_t b = 0; b < ups.size() && block == ups.size(); ++b)
        if (ups[b].mode == mode) block = b;
    if (block == ups.size()) throw std::invalid_argument("execute: mode not in iteration");

    const ModeSet root = full_set(order);
    CostReport cost;
    std::optional<DenseTensor> y;
    for (const ContractionStep& s : ups[block].steps) {
        const DenseTensor* src = &x;
        std::map<std::size_t, std::uint64_t> stamps;
        if (s.source != root) {
            const IntermediateCache::Entry* e = cache.find(s.source);
            if (e == nullptr)
                throw std::logic_error("execute: scheduled source " +
                                       mode_set_name(s.source, order) + " missing from cache");
            for (const auto& [m, v] : e->stamps)
                if (v != state.version(m))
                    throw stale_intermediate_error(
                        "execute: stale intermediate " + mode_set_name(s.source, order) +
                        " (mode " + std::to_string(m + 1) + " stamped v" + std::to_string(v) +
                        ", current v" + std::to_string(state.version(m)) + ") at iteration " +
                        std::to_string(iteration + 1) + ", update of mode " +
                        std::to_string(mode + 1));
            src = &e->tensor;
            stamps = e->stamps;
        }
        const std::size_t c = s.contract_mode;
        const std::uint64_t ic = src->shape().extent(c);
        DenseTensor out = ttm(*src, transpose(state.q(c)), c);  // device TTM
        const std::size_t r_power = order - std::size_t(std::popcount(s.source)) + 1;
        cost.add(s.source, r_power, 2ull * std::uint64_t(out.size()) * ic, s.source == root);
        stamps[c] = state.version(c);
        if (s.produces == mode_bit(mode))
            y = std::move(out);
        else
            cache.put(s.produces, {std::move(out), std::move(stamps)});
    }
    const std::vector<ModeSet> keep = detail::retained_keys(schedule, iteration, block);
    cache.evict_unless([&](ModeSet k) {
        for (const ModeSet n : keep)
            if (n == k) return true;
        return false;
    });
    if (!y) throw std::logic_error("execute: update produced no result");
    return {std::move(*y), std::move(cost)};
}

// Dry-run accounting over the first `iterations` sweeps (dim_tree.hpp:549-570).
inline CostReport measured_cost(const Schedule& schedule, const std::vector<std::size_t>& dims,
                                std::size_t rank, std::size_t iterations = 3) {
    const std::size_t order = schedule.order();
    if (dims.size() != order)
        throw std::invalid_argument("measured_cost: dims do not match schedule order");
    CostReport cost;
    const std::size_t n = iterations < schedule.num_iterations() ? iterations
                                                                 : schedule.num_iterations();
    for (std::size_t i = 0; i < n; ++i)
        for (const ModeUpdate& u : schedule.iteration(i).updates)
            for (const ContractionStep& s : u.steps) {
                const std::size_t r_power = order - std::size_t(std::popcount(s.source)) + 1;
                std::uint64_t f = 2;
                for (std::size_t m = 0; m < order; ++m)
                    if (s.source & mode_bit(m)) f *= dims[m];
                for (std::size_t p = 0; p < r_power; ++p) f *= rank;
                cost.add(s.source, r_power, f, s.source == full_set(order));
            }
    return cost;
}

inline std::uint64_t closed_form_cost(std::size_t order, Strategy strategy,
                                      const std::vector<std::size_t>& dims, std::size_t rank) {
    if (dims.size() != order && (order == 3 || order == 4))
        throw std::invalid_argument("closed_form_cost: dims do not match order");
    const std::vector<uint64_t> d = abi::u64(dims);
    uint64_t total = 0;
    abi::check(cpdb_closed_form_cost(uint32_t(order), int32_t(strategy),
                                     d.empty() ? nullptr : d.data(), rank, &total));
    return total;
}

inline std::uint64_t leading_flop_coefficient(std::size_t order, Strategy strategy) {
    uint64_t c = 0;
    abi::check(cpdb_leading_flop_coefficient(uint32_t(order), int32_t(strategy), &c));
    return c;
}

}  // namespace cpd
