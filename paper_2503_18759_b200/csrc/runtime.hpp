// Device runtime of libcpdb: the context behind the C ABI (include/cpdb.h).
//
// A context owns one B200, one stream and every device buffer of a solve:
// the tensor X (whole, or this rank's slab of the leading mode), the
// branch-reuse intermediate cache (one persistent buffer per free-mode set,
// dim_tree.hpp:112-139 semantics: valid flag + per-mode version stamps), the
// factor state (A_n, Q_n, packed Q_n, R_n, lambda; factor_state.hpp:18-48),
// the per-mode Q0 history and the scratch of the mode-update kernels.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <utility>
#include <string>
#include <vector>

#include "cpdb.h"
#include "kernels.hpp"
#include "schedule.hpp"

namespace cpdb {

struct Fail {
    int code;
    std::string what;
};

[[noreturn]] void fail(int code, const std::string& what);
void check_cuda(cudaError_t e, const char* where);
#define CPDB_CK(expr) ::cpdb::check_cuda((expr), #expr)

// Device memory cache: released blocks are kept per device and handed out
// again (best fit within 2x), so a new session / context on the same GPU does
// not pay cudaMalloc/cudaFree of GB-sized buffers (page mapping costs ms and
// made the host-buffer e2e runs jitter).  release() synchronises the device
// first, so a block is never handed out while a kernel may still touch it.
// On allocation failure the cache of that device is returned to the driver
// and the allocation retried once.
void* dev_alloc(size_t bytes, int* device, size_t* got);
void dev_release(void* p, size_t bytes, int device);
void dev_trim(int device);  // give every cached block of `device` back
void dev_guard_check(const char* where);  // CPDB_GUARD debug: verify guard zones

// Growable device allocation (never shrinks; released with its owner).
struct DevBuf {
    double* p = nullptr;
    size_t n = 0;  // doubles
    int dev = -1;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), dev(o.dev) {
        o.p = nullptr;
        o.n = 0;
    }
    ~DevBuf();
    double* ensure(size_t doubles);
    void swap(DevBuf& o) noexcept {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(dev, o.dev);
    }
};

struct Slot {
    DevBuf buf;
    bool valid = false;
    std::vector<uint64_t> dims;    // local extents
    std::vector<uint64_t> stamps;  // 0 = mode not absorbed
    bool sharded = false;          // split across ranks along a free mode (lay.mode)
    ShardLayout lay;               // replicated / split / partial sums (shard.cpp)
};

struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    int kind = 0;  // 0 root ttm, 1 branch ttm, 2 comm, 3 mode-update kernel
    double flops = 0, bytes = 0;
};

}  // namespace cpdb

namespace cpdb {
// Ranks of one process on one device, each driven by its own host thread:
// the collectives of the sharded path (all-reduce of partial sums, all-gather
// of V) run through a shared device buffer and host barriers instead of
// NCCL.  Exists so the sharded session is exercised on a single GPU
// (cpdb_create_local_group); production multi-GPU runs use NCCL.
struct LocalGroup {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    double* slots = nullptr;  // world x cap doubles on the group's device
    size_t cap = 0;
    // every rank blocks until all arrived; the last one runs `last` first
    void barrier(const std::function<void()>& last = {});
    ~LocalGroup();
};
}  // namespace cpdb

struct cpdb_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // Z-QR overlapped with the TTM chain
    cudaStream_t side_hi = nullptr;  // the same at top priority (tall-Z runs)
    cudaStream_t lo = nullptr;    // low priority: root TTM prefetched under the previous update
    cudaStream_t mid = nullptr;   // below stream/side: TTM chain beside a multi-kernel Z-QR
    cudaStream_t aux = nullptr;   // speculative next-sweep update beside the last one
    cudaStream_t zq = nullptr;    // the sweep-boundary Z-QR (not behind any chain)
    cudaStream_t tailq = nullptr;  // a sweep's last update beside the next sweep's first

    // sharding: leading mode split in contiguous slabs
    int rank = 0, world = 1;
    void* comm = nullptr;  // ncclComm_t
    std::shared_ptr<cpdb::LocalGroup> group;  // in-process ranks (tests)
    uint64_t row_begin = 0, rows = 0;
    int32_t shard_policy = 3;          // CPDB_SHARD_* (shard.cpp), default auto
    cpdb::ShardCost shard_cost;

    // X
    const double* x = nullptr;
    cpdb::DevBuf xown;
    std::vector<uint64_t> dims;   // global extents
    std::vector<uint64_t> ldims;  // local extents (ldims[0] = rows)
    bool norm_valid = false;
    double norm_x_sq = 0.0;
    // last cpdb_tensor_synth: global ||X_clean||^2 and ||E||^2 (E unscaled)
    double synth_norms[2] = {0.0, 0.0};

    // cache slots for the device execute() API (dim_tree.hpp:473-544)
    std::map<uint32_t, cpdb::Slot> slots;

    // scratch
    cpdb::DevBuf scratch_a, scratch_b, scratch_c, scratch_d, partials;
    int* dstatus = nullptr;
    double* pinned = nullptr;  // 64 doubles of pinned host memory

    cpdb_profile prof{};
    bool timing = true;
    bool overlap = true;  // root-TTM prefetch (Session::prefetch_root)
    uint64_t launches = 0;

    ~cpdb_ctx();
};

namespace cpdb {

// X-side helpers
uint64_t numel(const std::vector<uint64_t>& d);
void require_tensor(cpdb_ctx* c);
double ctx_norm_sq(cpdb_ctx* c);
void allreduce_sum(cpdb_ctx* c, double* dev, size_t n);
void allgather(cpdb_ctx* c, double* dev_full, size_t per_rank);
// src: `outer` contiguous blocks of `block` doubles, each the full extent of
// the scattered mode (outermost within the block); dst: this rank's
// block/world-sized chunk of every block, summed over the ranks
void reduce_scatter(cpdb_ctx* c, const double* src, uint64_t outer, uint64_t block, double* dst);

// The device-resident run_qr (solvers.hpp:215-336).
void solve(cpdb_ctx* c, const cpdb_config& cfg, cpdb_state* state, cpdb_trace_row* trace,
           uint64_t* trace_len, double* out_lambda, double* out_factors, double* fps,
           double* lps, cpdb_q0_observer observer, void* user);

// Natural (Y row-major) <-> reference (Khatri-Rao, descending fold) row order
// of Z / Q0 for mode n: digit reversal over the N-1 other modes.
// CP-ALS through the normal equations (als.cpp, solvers.hpp:149-208)
void als_solve(cpdb_ctx* c, const cpdb_config& cfg, const double* init_lambda,
               const double* init_factors, cpdb_trace_row* trace, uint64_t* trace_len,
               double* out_lambda, double* out_factors);
void mttkrp_primitive(cpdb_ctx* c, const double* x, const std::vector<uint64_t>& dims,
                      const std::vector<const double*>& fac_dev, uint32_t R, uint32_t n,
                      double* m_out);

std::vector<uint64_t> natural_to_reference(uint32_t order, uint64_t R);

// One TTM of the execute() chain on device buffers: contracts `c` of a
// tensor with local extents `sd` using factor Q (I_c x R) / packed Qp.
void run_ttm(cpdb_ctx* ctx, const double* src, const std::vector<uint64_t>& sd, uint32_t c,
             const double* q, const double* qp, uint32_t R, double* dst,
             cudaStream_t stream = nullptr, bool one_tile_per_cta = false, bool no_pdl = false,
             int sms = 0, uint32_t tiles_per_cta = 0);

}  // namespace cpdb
