// Dimension-tree contraction scheduler (host metadata, native C++).
//
// B200-side restatement of the reference scheduler
// (/root/reference/proj/include/cpd/dim_tree.hpp):
//   plans            dim_tree.hpp:191-331 (naive / dim-tree / branch-reuse 3 & 4)
//   build            dim_tree.hpp:386-426
//   validate         dim_tree.hpp:335-379 (structure + version simulation)
//   retained_keys    dim_tree.hpp:433-465 (cache eviction look-ahead)
//   measured_cost    dim_tree.hpp:549-570
//   closed_form_cost dim_tree.hpp:579-621
// The plans are the same fixed data; the code is organised around the device
// runtime's needs: every step also carries whether it is a root TTM and the
// distinct sweep "patterns" a CUDA graph can be captured for.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace cpdb {

using ModeSet = uint32_t;

enum class Strategy : int32_t { naive = 0, dim_tree = 1, branch_reuse = 2 };

struct Step {
    ModeSet source;
    uint32_t contract;
    ModeSet produces;
};

struct Update {
    uint32_t mode;
    std::vector<Step> steps;
};

struct Sweep {
    std::vector<Update> updates;
};

struct Plan {
    uint32_t order = 0;
    Strategy strategy = Strategy::naive;
    std::vector<Sweep> sweeps;
    uint64_t cycle_start = 0;
    uint64_t cycle_length = 1;

    ModeSet root() const { return (1u << order) - 1u; }
    std::vector<uint32_t> update_order(uint64_t i) const;
    // Index of the first sweep with the same step structure as sweep i
    // (sweeps of one pattern can share a captured CUDA graph).
    uint64_t pattern_of(uint64_t i) const;
};

// Error classes surfaced through the C ABI (status codes in include/cpdb.h).
struct SchedError {
    int code;  // CPDB_INVALID_ARGUMENT / CPDB_LOGIC_ERROR / CPDB_STALE_INTERMEDIATE
    std::string what;
};

// Throws SchedError.
Plan build_plan(uint32_t order, Strategy strategy, uint64_t sweeps);
void validate_plan(const Plan& p);
std::vector<ModeSet> retained_keys(const Plan& p, uint64_t sweep, uint32_t block);

struct Cost {
    uint64_t flops = 0;
    uint64_t roots = 0;
};
Cost measured_cost(const Plan& p, const std::vector<uint64_t>& dims, uint64_t rank,
                   uint64_t sweeps);
uint64_t closed_form_cost(uint32_t order, Strategy s, const std::vector<uint64_t>& dims,
                          uint64_t rank);
uint64_t leading_flop_coefficient(uint32_t order, Strategy s);

inline uint32_t popcount(ModeSet s) { return static_cast<uint32_t>(__builtin_popcount(s)); }

// ---- mode-0 sharding ---------------------------------------
// X is split into contiguous slabs of mode-0 rows.  An intermediate Y(S) is
// sharded exactly when mode 0 is still free (0 in S): contracting mode 0 of a
// sharded source yields a partial sum that is all-reduced (the path's only
// data exchange); every other TTM is local.  The mode-0 update's Y(0) keeps
// local rows, so its V (I_0 x R) is all-gathered before the replicated tail.
enum ShardFlag : int32_t {
    kSrcSharded = 1,   // the step reads a sharded source
    kAllReduce = 2,    // the step's output is a partial sum -> ncclAllReduce
    kOutSharded = 4,   // the step's output stays sharded
    kGatherV = 8,      // last step of the mode-0 update: all-gather V afterwards
};
inline bool set_sharded(ModeSet s, bool distributed) { return distributed && (s & 1u); }
inline int32_t shard_flags(ModeSet source, uint32_t contract, ModeSet produces, uint32_t mode,
                           bool distributed) {
    int32_t f = 0;
    if (set_sharded(source, distributed)) f |= kSrcSharded;
    if ((f & kSrcSharded) && contract == 0) f |= kAllReduce;
    if (set_sharded(produces, distributed)) f |= kOutSharded;
    if (distributed && mode == 0 && produces == 1u) f |= kGatherV;
    return f;
}

// ---- sharding planner (shard.cpp): layouts, reductions, cost model ---------
enum ShardLayKind : int32_t { kLayRep = 0, kLayShard = 1, kLayPartial = 2 };
struct ShardLayout {
    int32_t kind = kLayRep;
    int32_t mode = -1;  // kLayShard: the split free mode
    bool operator==(const ShardLayout& o) const { return kind == o.kind && mode == o.mode; }
    bool operator!=(const ShardLayout& o) const { return !(*this == o); }
};
enum ShardRed : int32_t { kRedNone = 0, kRedAllReduce = 1, kRedScatter = 2 };
enum ShardVOp : int32_t { kVNone = 0, kVGather = 1, kVAllReduce = 2 };
enum ShardPolicy : int32_t { kPolicyEager = 0, kPolicyScatter = 1, kPolicyLazy = 2, kPolicyAuto = 3 };
struct StepShard {
    ShardLayout src;      // layout of the step's source (X: sharded along mode 0)
    ShardLayout out;      // layout of the stored output (after the reduction)
    int32_t red = kRedNone;
    int32_t scatter = -1;  // kRedScatter: the free mode the partial is scattered onto
    uint64_t words = 0;    // doubles of the reduced partial (global size)
};
struct UpdateShard {
    ShardLayout yn;        // layout of Y(n) at the V-GEMM
    int32_t vop = kVNone;  // V's collective
    uint64_t vwords = 0;   // I_n x R
};
struct ShardCost {
    double tflops = 30.0;      // FP64 DMMA rate of the TTMs / V-GEMM (per GPU)
    double bus_gbs = 700.0;    // NCCL bus bandwidth over NVLink 5 / NVSwitch
    double latency_s = 20e-6;  // per collective
};
struct ShardPlan {
    std::vector<std::vector<std::vector<StepShard>>> steps;  // [sweep][update][step]
    std::vector<std::vector<UpdateShard>> updates;           // [sweep][update]
    double est_compute_s = 0.0, est_comm_s = 0.0;            // per rank, whole plan
};
ShardPlan plan_shards(const Plan& p, const std::vector<uint64_t>& dims, uint64_t R, int world,
                      ShardPolicy pol, const ShardCost& cp);

}  // namespace cpdb
