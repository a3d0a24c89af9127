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
#include <cstdio>
#include <cstring>
#include <mutex>
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

namespace {

struct Block {
    int dev;
    size_t bytes;
    void* p;
};
std::mutex g_pool_mu;
std::vector<Block> g_pool;
std::vector<Block> g_guarded;  // CPDB_GUARD debug registry

}  // namespace

void* dev_alloc(size_t bytes, int* device, size_t* got) {
    int dev = 0;
    CPDB_CK(cudaGetDevice(&dev));
    *device = dev;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        size_t best = g_pool.size();
        for (size_t i = 0; i < g_pool.size(); ++i) {
            const Block& b = g_pool[i];
            if (b.dev != dev || b.bytes < bytes || b.bytes > 2 * bytes + (1u << 20)) continue;
            if (best == g_pool.size() || b.bytes < g_pool[best].bytes) best = i;
        }
        if (best != g_pool.size()) {
            void* p = g_pool[best].p;
            *got = g_pool[best].bytes;
            g_pool.erase(g_pool.begin() + long(best));
            return p;
        }
    }
    void* p = nullptr;
    static const bool guard = std::getenv("CPDB_GUARD") != nullptr;
    const size_t gb = guard ? (size_t(1) << 20) : 0;  // debug: 1 MiB guard after the block
    cudaError_t e = cudaMalloc(&p, bytes + gb);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        dev_trim(dev);
        e = cudaMalloc(&p, bytes + gb);
    }
    CPDB_CK(e);
    if (guard) {
        CPDB_CK(cudaMemset(static_cast<char*>(p) + bytes, 0xA5, gb));
        std::lock_guard<std::mutex> lk(g_pool_mu);
        g_guarded.push_back({dev, bytes, p});
    }
    *got = bytes;
    return p;
}

void dev_guard_check(const char* where) {
    std::vector<Block> blocks;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        blocks = g_guarded;
    }
    CPDB_CK(cudaDeviceSynchronize());
    std::vector<unsigned char> h(size_t(1) << 20);
    for (const Block& b : blocks) {
        CPDB_CK(cudaMemcpy(h.data(), static_cast<char*>(b.p) + b.bytes, h.size(),
                           cudaMemcpyDeviceToHost));
        size_t bad = 0, first = h.size();
        for (size_t i = 0; i < h.size(); ++i)
            if (h[i] != 0xA5) {
                ++bad;
                if (first == h.size()) first = i;
            }
        if (bad)
            std::fprintf(stderr, "GUARD %s: block %p (%zu B) guard overwritten: %zu bytes, first +%zu\n",
                         where, b.p, b.bytes, bad, first);
    }
}

void dev_release(void* p, size_t bytes, int device) {
    if (!p) return;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    cudaDeviceSynchronize();  // no kernel may still use the block
    if (cur != device) cudaSetDevice(cur);
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back({device, bytes, p});
}

void dev_trim(int device) {
    std::vector<void*> drop;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t i = 0; i < g_pool.size();) {
            if (g_pool[i].dev == device) {
                drop.push_back(g_pool[i].p);
                g_pool.erase(g_pool.begin() + long(i));
            } else {
                ++i;
            }
        }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    for (void* p : drop) cudaFree(p);
    if (cur != device) cudaSetDevice(cur);
    if (!drop.empty()) {  // (CPDB_GUARD: freed blocks leave the registry)
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t i = 0; i < g_guarded.size();) {
            if (std::find(drop.begin(), drop.end(), g_guarded[i].p) != drop.end())
                g_guarded.erase(g_guarded.begin() + long(i));
            else
                ++i;
        }
    }
}

DevBuf::~DevBuf() { dev_release(p, n * sizeof(double), dev); }

double* DevBuf::ensure(size_t d) {
    if (p && d <= n) return p;
    dev_release(p, n * sizeof(double), dev);
    p = nullptr;
    n = 0;
    size_t got = 0;
    p = static_cast<double*>(dev_alloc(std::max<size_t>(d, 1) * sizeof(double), &dev, &got));
    n = got / sizeof(double);
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

void LocalGroup::barrier(const std::function<void()>& last) {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == world) {
        if (last) last();
        arrived = 0;
        ++generation;
        cv.notify_all();
    } else {
        cv.wait(lk, [&] { return generation != gen; });
    }
}

LocalGroup::~LocalGroup() {
    if (slots) cudaFree(slots);
}

namespace {

// rank r's n values -> slot r, then every rank reads all slots in rank order
void group_publish(cpdb_ctx* c, const double* src, size_t n) {
    LocalGroup& g = *c->group;
    g.barrier([&] {  // grow the shared buffer while nobody uses it
        if (g.cap < n) {
            if (g.slots) cudaFree(g.slots);
            g.slots = nullptr;
            CPDB_CK(cudaMalloc(&g.slots, sizeof(double) * n * size_t(g.world)));
            g.cap = n;
        }
    });
    CPDB_CK(cudaMemcpyAsync(g.slots + size_t(c->rank) * g.cap, src, n * sizeof(double),
                            cudaMemcpyDeviceToDevice, c->stream));
    CPDB_CK(cudaStreamSynchronize(c->stream));
    g.barrier();
}

}  // namespace

void allreduce_sum(cpdb_ctx* c, double* dev, size_t n) {
    if (c->world <= 1) return;
    if (c->group) {
        LocalGroup& g = *c->group;
        group_publish(c, dev, n);
        CPDB_CK(sum_slots(g.slots, g.cap, uint32_t(g.world), n, dev, c->stream));
        CPDB_CK(cudaStreamSynchronize(c->stream));
        g.barrier();  // slots are reused by the next collective
        return;
    }
    const Nccl& N = nccl();
    const ncclResult_t r =
        N.AllReduce(dev, dev, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->comm), c->stream);
    if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, std::string("ncclAllReduce: ") + N.GetErrorString(r));
}

void allgather(cpdb_ctx* c, double* dev_full, size_t per_rank) {
    if (c->world <= 1) return;
    if (c->group) {
        LocalGroup& g = *c->group;
        group_publish(c, dev_full + per_rank * size_t(c->rank), per_rank);
        for (int r = 0; r < g.world; ++r)
            CPDB_CK(cudaMemcpyAsync(dev_full + per_rank * size_t(r), g.slots + size_t(r) * g.cap,
                                    per_rank * sizeof(double), cudaMemcpyDeviceToDevice,
                                    c->stream));
        CPDB_CK(cudaStreamSynchronize(c->stream));
        g.barrier();
        return;
    }
    const Nccl& N = nccl();
    const ncclResult_t r = N.AllGather(dev_full + per_rank * c->rank, dev_full, per_rank,
                                       ncclDouble, static_cast<ncclComm_t>(c->comm), c->stream);
    if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, std::string("ncclAllGather: ") + N.GetErrorString(r));
}

void reduce_scatter(cpdb_ctx* c, const double* src, uint64_t outer, uint64_t block,
                    double* dst) {
    const uint64_t chunk = block / uint64_t(c->world);
    if (c->world <= 1) {
        CPDB_CK(cudaMemcpyAsync(dst, src, outer * block * sizeof(double),
                                cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    if (c->group) {
        LocalGroup& g = *c->group;
        group_publish(c, src, outer * block);
        CPDB_CK(sum_slots_scatter(g.slots, g.cap, uint32_t(g.world), outer, block, chunk,
                                  uint32_t(c->rank), dst, c->stream));
        CPDB_CK(cudaStreamSynchronize(c->stream));
        g.barrier();
        return;
    }
    // one reduce-scatter per outer slice (each slice is contiguous with the
    // scattered mode outermost), batched into one NCCL group
    const Nccl& N = nccl();
    ncclResult_t r = N.GroupStart();
    for (uint64_t o = 0; o < outer && r == ncclSuccess; ++o)
        r = N.ReduceScatter(src + o * block, dst + o * chunk, chunk, ncclDouble, ncclSum,
                            static_cast<ncclComm_t>(c->comm), c->stream);
    const ncclResult_t r2 = N.GroupEnd();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess)
        fail(CPDB_NCCL_ERROR, std::string("ncclReduceScatter: ") + N.GetErrorString(r));
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
             const double* q, const double* qp, uint32_t R, double* dst, cudaStream_t stream,
             bool one_tile_per_cta, bool no_pdl, int sms, uint32_t tiles_per_cta) {
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
    a.one_tile_per_cta = one_tile_per_cta ? 1 : 0;
    a.tiles_per_cta = tiles_per_cta;
    a.no_pdl = (no_pdl || one_tile_per_cta) ? 1 : 0;
    a.no_tma = 0;
    CPDB_CK(launch_ttm(a, stream ? stream : ctx->stream, sms > 0 ? sms : ctx->sms));
    ctx->launches += 1;
}

}  // namespace cpdb

cpdb_ctx::~cpdb_ctx() {
    if (stream) cudaStreamSynchronize(stream);
    if (lo) cudaStreamSynchronize(lo);
    if (mid) cudaStreamSynchronize(mid);
    if (aux) cudaStreamSynchronize(aux);
    if (zq) cudaStreamSynchronize(zq);
    if (side) cudaStreamSynchronize(side);
    if (side_hi) cudaStreamSynchronize(side_hi);
    if (comm) {
        const cpdb::Nccl& N = cpdb::nccl();
        if (N.ok) N.CommDestroy(static_cast<ncclComm_t>(comm));
    }
    if (dstatus) cudaFree(dstatus);
    if (pinned) cudaFreeHost(pinned);
    if (stream) cudaStreamDestroy(stream);
    if (side) cudaStreamDestroy(side);
    if (side_hi) cudaStreamDestroy(side_hi);
    if (lo) cudaStreamDestroy(lo);
    if (mid) cudaStreamDestroy(mid);
    if (aux) cudaStreamDestroy(aux);
    if (zq) cudaStreamDestroy(zq);
    if (tailq) cudaStreamDestroy(tailq);
}
