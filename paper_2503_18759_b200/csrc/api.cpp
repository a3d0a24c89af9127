// The C ABI of libcpdb (declarations and reference map in include/cpdb.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "comm.hpp"
#include "cpdt.hpp"
#include "cpdb.h"
#include "kernels.hpp"
#include "prims.hpp"
#include "runtime.hpp"
#include "schedule.hpp"
#include "session.hpp"

using cpdb::Fail;
using cpdb::fail;

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& body) {
    try {
        body();
        return CPDB_OK;
    } catch (const Fail& e) {
        g_error = e.what;
        return e.code;
    } catch (const cpdb::SchedError& e) {
        g_error = e.what;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return CPDB_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_error = e.what();
        return CPDB_LOGIC_ERROR;
    }
}

void use_device(cpdb_ctx* c) {
    if (!c) fail(CPDB_INVALID_ARGUMENT, "null context");
    CPDB_CK(cudaSetDevice(c->device));
}

std::vector<uint64_t> dims_of(const uint64_t* dims, uint32_t order) {
    if (!dims || order == 0) fail(CPDB_INVALID_ARGUMENT, "Shape: order must be >= 1");
    if (order > CPDB_MAX_ORDER) fail(CPDB_INVALID_ARGUMENT, "Shape: order above 8");
    std::vector<uint64_t> d(dims, dims + order);
    for (uint64_t v : d)
        if (v == 0) fail(CPDB_INVALID_ARGUMENT, "Shape: every extent must be >= 1");
    return d;
}

void upload(cpdb_ctx* c, double* dst, const double* src, size_t n) {
    CPDB_CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
}
void download(cpdb_ctx* c, double* dst, const double* src, size_t n) {
    CPDB_CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CPDB_CK(cudaStreamSynchronize(c->stream));
}

void init_ctx(cpdb_ctx* c, int device) {
    int count = 0;
    CPDB_CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) fail(CPDB_CUDA_ERROR, "no such CUDA device");
    cudaDeviceProp p{};
    CPDB_CK(cudaGetDeviceProperties(&p, device));
    if (p.major != 10)
        fail(CPDB_CUDA_ERROR, std::string("libcpdb is built for sm_100a (B200); device is ") +
                                  p.name + " sm_" + std::to_string(p.major) +
                                  std::to_string(p.minor));
    c->device = device;
    CPDB_CK(cudaSetDevice(device));
    c->sms = p.multiProcessorCount;
    // the solve's critical path (stream, side) at high priority; the root-TTM
    // prefetch (lo) yields to it CTA by CTA (Session::prefetch_root).  With a
    // small Z the chains (side) sit one level below the latency-bound Z-QR /
    // V-GEMM / finisher kernels so those get SMs first when both are ready
    // (measured: C3 1447 -> 1506 sweeps/s, C1 C2 C4 flat); a tall-Z run (C5,
    // TTM-dominated) keeps them on side_hi (low priority there: 25.1 -> 24.3)
    int least = 0, greatest = 0;
    CPDB_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    const int below = greatest < least ? greatest + 1 : greatest;
    CPDB_CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, greatest));
    CPDB_CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, below));
    CPDB_CK(cudaStreamCreateWithPriority(&c->side_hi, cudaStreamNonBlocking, greatest));
    CPDB_CK(cudaStreamCreateWithPriority(&c->lo, cudaStreamNonBlocking, least));
    // the next sweep's first V-GEMM + finisher beside this sweep's last ones
    CPDB_CK(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, greatest));
    CPDB_CK(cudaStreamCreateWithPriority(&c->zq, cudaStreamNonBlocking, greatest));
    // a TTM chain that must yield SMs to a concurrent multi-kernel Z-QR
    CPDB_CK(cudaStreamCreateWithPriority(&c->mid, cudaStreamNonBlocking, below));
    // the last update of a sweep while the next sweep's first update runs
    // beside it (Session::run): below that update's chain, above the root
    const int below2 = below < least ? (below + 1 < least ? below + 1 : below) : below;
    CPDB_CK(cudaStreamCreateWithPriority(&c->tailq, cudaStreamNonBlocking, below2));
    if (const char* sp = std::getenv("CPDB_SHARD_POLICY")) {
        const std::string v(sp);
        c->shard_policy = v == "eager" ? 0 : v == "scatter" ? 1 : v == "lazy" ? 2 : 3;
    }
    CPDB_CK(cudaMalloc(&c->dstatus, 64));
    CPDB_CK(cudaMemset(c->dstatus, 0, 64));
    CPDB_CK(cudaMallocHost(&c->pinned, 64 * sizeof(double)));
}

void set_local_geometry(cpdb_ctx* c, const std::vector<uint64_t>& d) {
    c->dims = d;
    c->ldims = d;
    if (c->world > 1) {
        if (d[0] % c->world != 0)
            fail(CPDB_INVALID_ARGUMENT, "sharded tensor: leading extent must divide by the world size");
        c->rows = d[0] / c->world;
        c->row_begin = c->rows * c->rank;
        c->ldims[0] = c->rows;
    } else {
        c->rows = d[0];
        c->row_begin = 0;
    }
    c->norm_valid = false;
    c->slots.clear();
}

int live_contexts(int device, int delta) {
    static std::mutex mu;
    static std::map<int, int> live;
    std::lock_guard<std::mutex> lk(mu);
    return live[device] += delta;
}

cpdb::Plan plan_from_steps(uint32_t order, const int64_t* steps, uint64_t n, uint64_t iterations) {
    cpdb::Plan p;
    p.order = order;
    p.sweeps.resize(iterations);
    for (uint64_t i = 0; i < n; ++i) {
        const int64_t* r = steps + 6 * i;
        if (r[0] < 0 || uint64_t(r[0]) >= iterations)
            fail(CPDB_INVALID_ARGUMENT, "schedule: iteration index out of range");
        auto& sw = p.sweeps[r[0]];
        const uint64_t block = uint64_t(r[1]);
        if (sw.updates.size() <= block) sw.updates.resize(block + 1);
        sw.updates[block].mode = uint32_t(r[2]);
        sw.updates[block].steps.push_back(
            {uint32_t(r[3]), uint32_t(r[4]), uint32_t(r[5])});
    }
    return p;
}

}  // namespace

extern "C" {

const char* cpdb_version(void) { return "cpdb 0.1.0 (sm_100a, FP64 DMMA)"; }
const char* cpdb_last_error(void) { return g_error.c_str(); }

int cpdb_device_ok(int device) {
    cudaDeviceProp p{};
    if (cudaGetDeviceProperties(&p, device) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return p.major == 10 ? 1 : 0;
}

int cpdb_create(int device, cpdb_ctx** out) {
    if (!out) return CPDB_INVALID_ARGUMENT;
    *out = nullptr;
    cpdb_ctx* c = new (std::nothrow) cpdb_ctx();
    if (!c) return CPDB_OUT_OF_MEMORY;
    const int rc = guarded([&] { init_ctx(c, device); });
    if (rc != CPDB_OK) {
        delete c;
        return rc;
    }
    live_contexts(c->device, +1);
    *out = c;
    return CPDB_OK;
}

int cpdb_nccl_unique_id(void* out128) {
    return guarded([&] {
        const cpdb::Nccl& N = cpdb::nccl();
        if (!N.ok) fail(CPDB_NCCL_ERROR, N.why);
        ncclUniqueId id;
        const ncclResult_t r = N.GetUniqueId(&id);
        if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, N.GetErrorString(r));
        std::memcpy(out128, &id, sizeof id);
    });
}

int cpdb_create_sharded(int device, int rank, int world, const void* nccl_id, cpdb_ctx** out) {
    if (!out) return CPDB_INVALID_ARGUMENT;
    *out = nullptr;
    cpdb_ctx* c = new (std::nothrow) cpdb_ctx();
    if (!c) return CPDB_OUT_OF_MEMORY;
    const int rc = guarded([&] {
        if (world < 1 || rank < 0 || rank >= world)
            fail(CPDB_INVALID_ARGUMENT, "sharded context: bad rank/world");
        init_ctx(c, device);
        c->rank = rank;
        c->world = world;
        if (world > 1) {
            const cpdb::Nccl& N = cpdb::nccl();
            if (!N.ok) fail(CPDB_NCCL_ERROR, N.why);
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof id);
            ncclComm_t comm;
            const ncclResult_t r = N.CommInitRank(&comm, world, id, rank);
            if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, N.GetErrorString(r));
            c->comm = comm;
        }
    });
    if (rc != CPDB_OK) {
        delete c;
        return rc;
    }
    live_contexts(c->device, +1);
    *out = c;
    return CPDB_OK;
}

int cpdb_nccl_selftest(int device, double* max_err) {
    return guarded([&] {
        if (!max_err) fail(CPDB_INVALID_ARGUMENT, "nccl_selftest: null output");
        const cpdb::Nccl& N = cpdb::nccl();
        if (!N.ok) fail(CPDB_NCCL_ERROR, N.why);
        CPDB_CK(cudaSetDevice(device));
        ncclUniqueId id;
        ncclResult_t r = N.GetUniqueId(&id);
        if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, N.GetErrorString(r));
        ncclComm_t comm;
        r = N.CommInitRank(&comm, 1, id, 0);
        if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, N.GetErrorString(r));
        cudaStream_t st;
        CPDB_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        // the three call patterns of runtime.cpp on a one-rank communicator:
        // all-reduce in place, all-gather of this rank's chunk, and the
        // grouped per-slice reduce-scatter (identities for one rank)
        const size_t outer = 3, block = 40, n = outer * block;
        std::vector<double> h(n), back(n);
        for (size_t i = 0; i < n; ++i) h[i] = double(i) * 0.5 - 7.0;
        double *a, *b;
        CPDB_CK(cudaMalloc(&a, n * sizeof(double)));
        CPDB_CK(cudaMalloc(&b, n * sizeof(double)));
        CPDB_CK(cudaMemcpy(a, h.data(), n * sizeof(double), cudaMemcpyHostToDevice));
        double err = 0.0;
        auto check = [&](const double* dev) {
            CPDB_CK(cudaStreamSynchronize(st));
            CPDB_CK(cudaMemcpy(back.data(), dev, n * sizeof(double), cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < n; ++i) err = std::max(err, std::fabs(back[i] - h[i]));
        };
        r = N.AllReduce(a, a, n, ncclDouble, ncclSum, comm, st);
        if (r == ncclSuccess) check(a);
        if (r == ncclSuccess) r = N.AllGather(a, b, n, ncclDouble, comm, st);
        if (r == ncclSuccess) check(b);
        if (r == ncclSuccess) {
            CPDB_CK(cudaMemsetAsync(b, 0, n * sizeof(double), st));
            r = N.GroupStart();
            for (size_t o = 0; o < outer && r == ncclSuccess; ++o)
                r = N.ReduceScatter(a + o * block, b + o * block, block, ncclDouble, ncclSum, comm,
                                    st);
            const ncclResult_t r2 = N.GroupEnd();
            if (r == ncclSuccess) r = r2;
            if (r == ncclSuccess) check(b);
        }
        cudaFree(a);
        cudaFree(b);
        cudaStreamDestroy(st);
        N.CommDestroy(comm);
        if (r != ncclSuccess) fail(CPDB_NCCL_ERROR, N.GetErrorString(r));
        *max_err = err;
    });
}

int cpdb_create_local_group(int device, int world, cpdb_ctx** out) {
    if (!out || world < 1) return CPDB_INVALID_ARGUMENT;
    for (int r = 0; r < world; ++r) out[r] = nullptr;
    auto group = std::make_shared<cpdb::LocalGroup>();
    group->world = world;
    for (int r = 0; r < world; ++r) {
        cpdb_ctx* c = new (std::nothrow) cpdb_ctx();
        if (!c) return CPDB_OUT_OF_MEMORY;
        const int rc = guarded([&] {
            init_ctx(c, device);
            c->rank = r;
            c->world = world;
            c->group = group;
        });
        if (rc != CPDB_OK) {
            delete c;
            for (int q = 0; q < r; ++q) cpdb_destroy(out[q]);
            return rc;
        }
        live_contexts(c->device, +1);
        out[r] = c;
    }
    return CPDB_OK;
}

void cpdb_destroy(cpdb_ctx* ctx) {
    if (!ctx) return;
    const int dev = ctx->device;
    cudaSetDevice(dev);
    delete ctx;
    // the last context on a device hands the cached blocks back to the driver
    if (live_contexts(dev, -1) == 0) cpdb::dev_trim(dev);
}

int cpdb_shard_rows(uint64_t extent0, int rank, int world, uint64_t* begin, uint64_t* count) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world)
            fail(CPDB_INVALID_ARGUMENT, "shard_rows: bad rank/world");
        if (extent0 % uint64_t(world) != 0)
            fail(CPDB_INVALID_ARGUMENT, "shard_rows: leading extent must divide by the world size");
        *count = extent0 / world;
        *begin = *count * rank;
    });
}

int cpdb_tensor_set(cpdb_ctx* c, const double* host, const uint64_t* dims, uint32_t order) {
    return guarded([&] {
        use_device(c);
        if (!host) fail(CPDB_INVALID_ARGUMENT, "tensor_set: null data");
        set_local_geometry(c, dims_of(dims, order));
        const uint64_t n = cpdb::numel(c->ldims);
        double* d = c->xown.ensure(n);
        upload(c, d, host, n);
        CPDB_CK(cudaStreamSynchronize(c->stream));
        c->x = d;
    });
}

int cpdb_tensor_set_async(cpdb_ctx* c, const double* host, const uint64_t* dims,
                          uint32_t order) {
    return guarded([&] {
        use_device(c);
        if (!host) fail(CPDB_INVALID_ARGUMENT, "tensor_set: null data");
        set_local_geometry(c, dims_of(dims, order));
        const uint64_t n = cpdb::numel(c->ldims);
        double* d = c->xown.ensure(n);
        upload(c, d, host, n);  // on the context's stream: later calls are ordered behind it
        c->x = d;
    });
}

int cpdb_tensor_load_cpdt(cpdb_ctx* c, const char* path) {
    return guarded([&] {
        use_device(c);
        if (!path) fail(CPDB_INVALID_ARGUMENT, "tensor_load: null path");
        const cpdb::CpdtHeader h = cpdb::read_cpdt_header(path);
        if (h.dims.size() > CPDB_MAX_ORDER)
            fail(CPDB_INVALID_ARGUMENT, "tensor_load: order above 8 is not supported");
        set_local_geometry(c, h.dims);
        const uint64_t n = cpdb::numel(c->ldims);
        double* d = c->xown.ensure(n);
        // this rank's contiguous mode-0 slab: rows [row_begin, row_begin + rows)
        const uint64_t inner = n / c->ldims[0];
        cpdb::file_to_device(path, h.payload_offset + 8 * c->row_begin * inner, 8 * n, d,
                             c->stream);
        if (cpdb::count_nonfinite(d, n, c->stream) != 0)
            fail(CPDB_FORMAT_ERROR, "tensor payload contains a non-finite value");
        c->x = d;
    });
}

int cpdb_tensor_save_cpdt(cpdb_ctx* c, const char* path) {
    return guarded([&] {
        use_device(c);
        if (!path) fail(CPDB_INVALID_ARGUMENT, "tensor_save: null path");
        if (!c->x) fail(CPDB_LOGIC_ERROR, "tensor_save: no tensor");
        if (c->world > 1) fail(CPDB_INVALID_ARGUMENT, "tensor_save: sharded context");
        cpdb::device_to_cpdt(path, c->dims, c->x, cpdb::numel(c->dims), c->stream);
    });
}

int cpdb_cpdt_info(const char* path, uint32_t* order, uint64_t* dims) {
    return guarded([&] {
        if (!path || !order || !dims) fail(CPDB_INVALID_ARGUMENT, "cpdt_info: null argument");
        const cpdb::CpdtHeader h = cpdb::read_cpdt_header(path);
        *order = uint32_t(h.dims.size());
        for (size_t k = 0; k < h.dims.size() && k < CPDB_MAX_ORDER; ++k) dims[k] = h.dims[k];
    });
}

int cpdb_tensor_set_device(cpdb_ctx* c, const double* dptr, const uint64_t* dims, uint32_t order) {
    return guarded([&] {
        use_device(c);
        if (!dptr) fail(CPDB_INVALID_ARGUMENT, "tensor_set_device: null pointer");
        set_local_geometry(c, dims_of(dims, order));
        c->x = dptr;
    });
}

int cpdb_tensor_synth(cpdb_ctx* c, int32_t kind, const uint64_t* dims, uint32_t order,
                      uint64_t rank, double rho, uint64_t seed) {
    return guarded([&] {
        use_device(c);
        if (kind != 0 && kind != 1) fail(CPDB_INVALID_ARGUMENT, "synth: unknown kind");
        if (rank == 0) fail(CPDB_INVALID_ARGUMENT, "synth: rank must be >= 1");
        set_local_geometry(c, dims_of(dims, order));
        const uint64_t n = cpdb::numel(c->ldims);
        double* x = c->xown.ensure(n);
        uint64_t nf = 0;
        for (uint64_t d : c->dims) nf += d * rank;
        double* f = c->scratch_a.ensure(nf);
        double* part = c->partials.ensure(cpdb::synth_partials_doubles() + 8);
        double* scal = part + cpdb::synth_partials_doubles();
        cpdb::DevBuf ddims;
        double* dd = ddims.ensure(order);
        CPDB_CK(cudaMemcpyAsync(dd, c->dims.data(), order * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, c->stream));
        CPDB_CK(cpdb::synth_pass1(x, c->dims.data(), reinterpret_cast<const uint64_t*>(dd), order,
                                  rank, kind, seed, c->row_begin, c->rows, f, part, scal,
                                  c->stream));
        cpdb::allreduce_sum(c, scal, 2);
        CPDB_CK(cpdb::synth_pass2(x, c->dims.data(), order, rank, seed, c->row_begin, c->rows,
                                  scal, rho, c->stream));
        c->launches += 4;
        CPDB_CK(cudaMemcpyAsync(c->synth_norms, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                c->stream));
        CPDB_CK(cudaStreamSynchronize(c->stream));
        if (rho <= 0.0) c->synth_norms[1] = 0.0;
        c->x = x;
    });
}

int cpdb_tensor_synth_truth(cpdb_ctx* c, int32_t kind, const uint64_t* dims, uint32_t order,
                            uint64_t rank, uint64_t seed, double* factors) {
    return guarded([&] {
        use_device(c);
        if (kind != 0 && kind != 1) fail(CPDB_INVALID_ARGUMENT, "synth: unknown kind");
        if (rank == 0) fail(CPDB_INVALID_ARGUMENT, "synth: rank must be >= 1");
        if (!factors) fail(CPDB_INVALID_ARGUMENT, "synth_truth: null output");
        const std::vector<uint64_t> d = dims_of(dims, order);
        uint64_t nf = 0;
        for (uint64_t e : d) nf += e * rank;
        cpdb::DevBuf fb, ddims;
        double* f = fb.ensure(nf);
        double* dd = ddims.ensure(order);
        CPDB_CK(cudaMemcpyAsync(dd, d.data(), order * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                c->stream));
        CPDB_CK(cpdb::synth_factors(f, reinterpret_cast<const uint64_t*>(dd), order, rank, kind,
                                    seed, c->stream));
        c->launches += 1;
        download(c, factors, f, nf);
    });
}

int cpdb_tensor_synth_norms(cpdb_ctx* c, double* out) {
    return guarded([&] {
        if (!out) fail(CPDB_INVALID_ARGUMENT, "synth_norms: null output");
        out[0] = c->synth_norms[0];
        out[1] = c->synth_norms[1];
    });
}

int cpdb_tensor_get(cpdb_ctx* c, double* host) {
    return guarded([&] {
        use_device(c);
        cpdb::require_tensor(c);
        download(c, host, c->x, cpdb::numel(c->ldims));
    });
}

int cpdb_tensor_norm_sq(cpdb_ctx* c, double* out) {
    return guarded([&] {
        use_device(c);
        *out = cpdb::ctx_norm_sq(c);
    });
}

int cpdb_solve(cpdb_ctx* c, const cpdb_config* cfg, cpdb_state* state, cpdb_trace_row* trace,
               uint64_t* trace_len, double* out_lambda, double* out_factors,
               double* factors_per_sweep, double* lambda_per_sweep, cpdb_q0_observer observer,
               void* observer_user) {
    return guarded([&] {
        use_device(c);
        if (!cfg) fail(CPDB_INVALID_ARGUMENT, "null config");
        cpdb::solve(c, *cfg, state, trace, trace_len, out_lambda, out_factors, factors_per_sweep,
                    lambda_per_sweep, observer, observer_user);
    });
}

int cpdb_session_begin(cpdb_ctx* c, const cpdb_config* cfg, const cpdb_state* state,
                       cpdb_session** out) {
    if (!out) return CPDB_INVALID_ARGUMENT;
    *out = nullptr;
    cpdb_session* ss = new (std::nothrow) cpdb_session();
    if (!ss) return CPDB_OUT_OF_MEMORY;
    const int rc = guarded([&] {
        use_device(c);
        if (!cfg) fail(CPDB_INVALID_ARGUMENT, "null config");
        ss->s.begin(c, *cfg, state);
    });
    if (rc != CPDB_OK) {
        delete ss;
        return rc;
    }
    *out = ss;
    return CPDB_OK;
}

int cpdb_session_run(cpdb_session* ss, uint64_t sweeps, cpdb_trace_row* trace, uint64_t* rows,
                     int32_t* finished) {
    return guarded([&] {
        if (!ss) fail(CPDB_INVALID_ARGUMENT, "null session");
        use_device(ss->s.c);
        const uint64_t n = ss->s.run(sweeps, trace, nullptr, nullptr, nullptr, nullptr);
        if (rows) *rows = n;
        if (finished)
            *finished = (ss->s.converged || ss->s.done >= ss->s.plan.sweeps.size()) ? 1 : 0;
    });
}

int cpdb_session_end(cpdb_session* ss, cpdb_state* state, double* out_lambda,
                     double* out_factors) {
    return guarded([&] {
        if (!ss) fail(CPDB_INVALID_ARGUMENT, "null session");
        use_device(ss->s.c);
        ss->s.end(state, out_lambda, out_factors);
    });
}

void cpdb_session_destroy(cpdb_session* ss) {
    if (!ss) return;
    if (ss->s.c) cudaSetDevice(ss->s.c->device);
    delete ss;
}

int cpdb_profile_get(cpdb_ctx* c, cpdb_profile* out) {
    if (!c || !out) return CPDB_INVALID_ARGUMENT;
    *out = c->prof;
    return CPDB_OK;
}

int cpdb_set_options(cpdb_ctx* c, int32_t timing, int32_t overlap) {
    if (!c) return CPDB_INVALID_ARGUMENT;
    c->timing = timing != 0;
    c->overlap = overlap != 0;
    return CPDB_OK;
}

// ---------------------------------------------------------------- primitives
int cpdb_ttm(cpdb_ctx* c, const double* t, const uint64_t* dims, uint32_t order, const double* b,
             uint64_t b_rows, uint32_t mode, double* out) {
    return guarded([&] {
        use_device(c);
        const auto d = dims_of(dims, order);
        if (mode >= order) fail(CPDB_INVALID_ARGUMENT, "ttm: mode out of range");
        if (b_rows == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
        const uint64_t K = d[mode], n = cpdb::numel(d);
        const uint64_t nout = n / K * b_rows;
        double* dx = c->scratch_a.ensure(n);
        double* db = c->scratch_b.ensure(b_rows * K);
        double* dq = c->scratch_c.ensure(b_rows * K);
        double* dy = c->scratch_d.ensure(nout);
        upload(c, dx, t, n);
        upload(c, db, b, b_rows * K);
        CPDB_CK(cpdb::transpose_dev(db, b_rows, K, dq, c->stream));
        double* qp = nullptr;
        cpdb::DevBuf packed;
        qp = packed.ensure(uint64_t(cpdb::ttm_kpad(K)) * cpdb::ttm_rpad(uint32_t(b_rows)));
        CPDB_CK(cpdb::pack_q(dq, qp, uint32_t(K), uint32_t(b_rows), c->stream));
        cpdb::run_ttm(c, dx, d, mode, dq, qp, uint32_t(b_rows), dy);
        download(c, out, dy, nout);
    });
}

int cpdb_unfold(cpdb_ctx* c, const double* t, const uint64_t* dims, uint32_t order, uint32_t mode,
                double* out) {
    return guarded([&] {
        use_device(c);
        const auto d = dims_of(dims, order);
        if (mode >= order) fail(CPDB_INVALID_ARGUMENT, "unfold: mode out of range");
        const uint64_t n = cpdb::numel(d);
        double* dx = c->scratch_a.ensure(n);
        double* dy = c->scratch_b.ensure(n);
        upload(c, dx, t, n);
        cpdb::Dims8 g{};
        g.order = order;
        for (uint32_t k = 0; k < order; ++k) g.v[k] = d[k];
        CPDB_CK(cpdb::unfold_dev(dx, g, mode, dy, c->stream));
        download(c, out, dy, n);
    });
}

int cpdb_khatri_rao(cpdb_ctx* c, const double* const* mats, const uint64_t* rows, uint32_t count,
                    uint64_t cols, double* out) {
    return guarded([&] {
        use_device(c);
        if (count == 0) fail(CPDB_INVALID_ARGUMENT, "khatri_rao: empty list");
        if (count > 8) fail(CPDB_INVALID_ARGUMENT, "khatri_rao: at most 8 factors");
        if (cols == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
        uint64_t total = 0, prod = 1;
        for (uint32_t i = 0; i < count; ++i) {
            if (rows[i] == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
            total += rows[i] * cols;
            prod *= rows[i];
        }
        double* dm = c->scratch_a.ensure(total + 16);
        double* dy = c->scratch_b.ensure(prod * cols);
        std::vector<const double*> ptrs(count);
        uint64_t off = 0;
        for (uint32_t i = 0; i < count; ++i) {
            upload(c, dm + off, mats[i], rows[i] * cols);
            ptrs[i] = dm + off;
            off += rows[i] * cols;
        }
        // pointer table after the matrices (16 slots reserved)
        double* table = dm + total;
        CPDB_CK(cudaMemcpyAsync(table, ptrs.data(), count * sizeof(double*), cudaMemcpyHostToDevice,
                                c->stream));
        cpdb::Dims8 g{};
        g.order = count;
        for (uint32_t i = 0; i < count; ++i) g.v[i] = rows[i];
        CPDB_CK(cpdb::khatri_rao_dev(reinterpret_cast<const double* const*>(table), g, cols, dy,
                                     c->stream));
        download(c, out, dy, prod * cols);
    });
}

int cpdb_thin_qr(cpdb_ctx* c, const double* a, uint64_t m, uint64_t n, double* q, double* r) {
    return guarded([&] {
        use_device(c);
        if (m == 0 || n == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
        if (m < n) fail(CPDB_INVALID_ARGUMENT, "thin_qr: requires rows >= cols");
        double* da = c->scratch_a.ensure(m * n);
        // (tall inputs: the cooperative multi-CTA kernel, widerank.cu -- the
        // same reference algorithm with the rows split across the SMs)
        const bool coop = m >= 256 && n <= 1024;
        double* dw = c->scratch_b.ensure(
            coop ? m * n + cpdb::zqr_wide_work_doubles(uint32_t(n)) : 2 * m * n + n);
        double* dq = c->scratch_c.ensure(m * n);
        double* dr = c->scratch_d.ensure(n * n);
        upload(c, da, a, m * n);
        if (coop)
            CPDB_CK(cpdb::householder_qr_wide(da, m, uint32_t(n), dw, dq, dr, c->stream));
        else
            CPDB_CK(cpdb::householder_qr(da, m, uint32_t(n), dw, dq, dr, c->stream));
        download(c, q, dq, m * n);
        download(c, r, dr, n * n);
    });
}

int cpdb_solve_rows_lower(cpdb_ctx* c, const double* l, uint64_t n, const double* rhs,
                          uint64_t rows, double* out, int64_t* bad_column) {
    if (bad_column) *bad_column = -1;
    return guarded([&] {
        use_device(c);
        if (n == 0 || rows == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
        double* dl = c->scratch_a.ensure(n * n);
        double* dx = c->scratch_b.ensure(rows * n);
        upload(c, dl, l, n * n);
        upload(c, dx, rhs, rows * n);
        CPDB_CK(cpdb::solve_rows_lower_dev(dl, uint32_t(n), dx, rows, c->dstatus, c->stream));
        int bad = 0;
        CPDB_CK(cudaMemcpyAsync(c->pinned, c->dstatus, sizeof(int), cudaMemcpyDeviceToHost,
                                c->stream));
        CPDB_CK(cudaStreamSynchronize(c->stream));
        std::memcpy(&bad, c->pinned, sizeof(int));
        CPDB_CK(cudaMemsetAsync(c->dstatus, 0, sizeof(int), c->stream));
        if (bad) {
            if (bad_column) *bad_column = bad - 1;
            fail(CPDB_SINGULAR_TRIANGULAR,
                 "triangular solve: diagonal entry of column " + std::to_string(bad - 1) + " is " +
                     std::to_string(l[(bad - 1) * n + (bad - 1)]) +
                     " (rank-deficient Khatri-Rao factor)");
        }
        download(c, out, dx, rows * n);
    });
}

int cpdb_normalize_columns(cpdb_ctx* c, const double* a, uint64_t m, uint64_t n, double* out,
                           double* weights) {
    return guarded([&] {
        use_device(c);
        if (m == 0 || n == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
        double* da = c->scratch_a.ensure(m * n);
        double* dw = c->scratch_b.ensure(n);
        upload(c, da, a, m * n);
        CPDB_CK(cpdb::normalize_exact(da, m, uint32_t(n), dw, c->stream));
        download(c, out, da, m * n);
        download(c, weights, dw, n);
    });
}

int cpdb_extrapolate_q0(cpdb_ctx* c, const double* now, const double* prev, uint64_t rows,
                        uint64_t cols, double beta, double alpha, double* out) {
    return guarded([&] {
        use_device(c);
        const uint64_t n = rows * cols;
        if (n == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
        double* dn = c->scratch_a.ensure(n);
        double* dp = c->scratch_b.ensure(n);
        double* dy = c->scratch_c.ensure(n);
        upload(c, dn, now, n);
        upload(c, dp, prev, n);
        CPDB_CK(cpdb::extrapolate_dev(dn, dp, n, beta, alpha, dy, c->stream));
        download(c, out, dy, n);
    });
}

int cpdb_fitness_fast_qr(cpdb_ctx* c, double nx2, const double* v, const double* a_hat,
                         uint64_t rows, const double* r0, const double* r_n, const double* lambda,
                         uint64_t r, double* fitness, double* raw) {
    return guarded([&] {
        use_device(c);
        if (!(nx2 > 0.0)) fail(CPDB_INVALID_ARGUMENT, "fitness_fast_qr: zero-norm tensor");
        if (rows == 0 || r == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
        double* dv = c->scratch_a.ensure(2 * rows * r);
        double* dm = c->scratch_b.ensure(2 * r * r + r + 8);
        upload(c, dv, v, rows * r);
        upload(c, dv + rows * r, a_hat, rows * r);
        upload(c, dm, r0, r * r);
        upload(c, dm + r * r, r_n, r * r);
        upload(c, dm + 2 * r * r, lambda, r);
        double* o = dm + 2 * r * r + r;
        CPDB_CK(cpdb::fitness_dev(nx2, dv, dv + rows * r, rows, dm, dm + r * r, dm + 2 * r * r,
                                  uint32_t(r), o, c->stream));
        double h[4];
        download(c, h, o, 4);
        *fitness = h[2];
        *raw = h[3];
    });
}

int cpdb_als_solve(cpdb_ctx* c, const cpdb_config* cfg, const double* init_lambda,
                   const double* init_factors, cpdb_trace_row* trace, uint64_t* trace_len,
                   double* out_lambda, double* out_factors) {
    return guarded([&] {
        use_device(c);
        if (!cfg) fail(CPDB_INVALID_ARGUMENT, "null config");
        cpdb::als_solve(c, *cfg, init_lambda, init_factors, trace, trace_len, out_lambda,
                        out_factors);
    });
}

int cpdb_mttkrp(cpdb_ctx* c, const double* t, const uint64_t* dims, uint32_t order,
                const double* const* factors, const uint64_t* factor_rows,
                const uint64_t* factor_cols, uint32_t mode, double* out) {
    return guarded([&] {
        use_device(c);
        const std::vector<uint64_t> d = dims_of(dims, order);
        // check_mttkrp_args (tensor.hpp:415-431)
        if (mode >= order) fail(CPDB_INVALID_ARGUMENT, "mttkrp: mode out of range");
        if (!factors || !factor_rows || !factor_cols)
            fail(CPDB_INVALID_ARGUMENT, "mttkrp: need one factor per mode");
        uint64_t rank = 0;
        for (uint32_t k = 0; k < order; ++k) {
            if (k == mode) continue;
            if (!factors[k]) fail(CPDB_INVALID_ARGUMENT, "mttkrp: missing factor");
            if (rank == 0) rank = factor_cols[k];
            if (factor_cols[k] != rank) fail(CPDB_INVALID_ARGUMENT, "mttkrp: mismatched ranks");
            if (factor_rows[k] != d[k])
                fail(CPDB_INVALID_ARGUMENT, "mttkrp: factor rows do not match mode extent");
        }
        if (rank == 0) fail(CPDB_INVALID_ARGUMENT, "mttkrp: order must be >= 2");
        if (rank > 1024) fail(CPDB_INVALID_ARGUMENT, "mttkrp: ranks above 1024 are not supported");
        const uint32_t R = uint32_t(rank);
        const uint64_t nx = cpdb::numel(d);
        uint64_t nf = 0;
        for (uint32_t k = 0; k < order; ++k)
            if (k != mode) nf += d[k] * R;
        double* dx = c->scratch_a.ensure(nx);
        double* df = c->scratch_b.ensure(nf + d[mode] * R);
        upload(c, dx, t, nx);
        std::vector<const double*> fac(order, nullptr);
        uint64_t off = 0;
        for (uint32_t k = 0; k < order; ++k) {
            if (k == mode) continue;
            upload(c, df + off, factors[k], d[k] * R);
            fac[k] = df + off;
            off += d[k] * R;
        }
        double* dm = df + nf;
        cpdb::mttkrp_primitive(c, dx, d, fac, R, mode, dm);
        download(c, out, dm, d[mode] * R);
    });
}

int cpdb_solve_spd(cpdb_ctx* c, const double* g, uint64_t g_rows, uint64_t g_cols,
                   const double* rhs, uint64_t rows, uint64_t cols, double* x,
                   int32_t* regularized) {
    return guarded([&] {
        use_device(c);
        // linalg.hpp:133-135
        if (g_cols != g_rows) fail(CPDB_INVALID_ARGUMENT, "solve_spd: G must be square");
        if (cols != g_rows) fail(CPDB_INVALID_ARGUMENT, "solve_spd: RHS columns must match G");
        if (g_rows == 0) fail(CPDB_INVALID_ARGUMENT, "Matrix: zero dimension");
        if (g_rows > 1024)
            fail(CPDB_INVALID_ARGUMENT, "solve_spd: n above 1024 is not supported");
        const uint32_t n = uint32_t(g_rows);
        const uint64_t uw = cpdb::spd_work_doubles(n);
        double* dg = c->scratch_a.ensure(uint64_t(n) * n + uw + 8);
        double* dx = c->scratch_b.ensure(std::max<uint64_t>(rows * n, 1));
        upload(c, dg, g, uint64_t(n) * n);
        if (rows) upload(c, dx, rhs, rows * n);
        int* flags = reinterpret_cast<int*>(dg + uint64_t(n) * n + uw);
        CPDB_CK(cudaMemsetAsync(flags, 0, 2 * sizeof(int), c->stream));
        CPDB_CK(cpdb::launch_spd_solve(dg, n, dg + uint64_t(n) * n, dx, rows, flags, flags + 1,
                                       c->stream, c->sms));
        int h[2];
        CPDB_CK(cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, c->stream));
        CPDB_CK(cudaStreamSynchronize(c->stream));
        if (h[0] == 5) fail(CPDB_INVALID_ARGUMENT, "solve_spd: G is not symmetric");
        if (h[0] == 4)
            fail(CPDB_SINGULAR_SYSTEM, "solve_spd: factorization failed after ridge");
        if (rows) download(c, x, dx, rows * n);
        if (regularized) *regularized = h[1];
    });
}

int cpdb_fitness_fast_als(cpdb_ctx* c, double nx2, const double* m, const double* a_hat,
                          uint64_t rows, uint64_t cols, const double* gamma,
                          const double* lambda, uint64_t r, const double* s_last,
                          double* fitness, double* raw) {
    return guarded([&] {
        use_device(c);
        if (!(nx2 > 0.0)) fail(CPDB_INVALID_ARGUMENT, "fitness_fast_als: zero-norm tensor");
        if (r == 0) fail(CPDB_INVALID_ARGUMENT, "fitness_fast_als: dimension mismatch");
        double* dv = c->scratch_a.ensure(std::max<uint64_t>(2 * rows * cols, 1));
        double* dm = c->scratch_b.ensure(2 * r * r + r + 8);
        if (rows * cols) {
            upload(c, dv, m, rows * cols);
            upload(c, dv + rows * cols, a_hat, rows * cols);
        }
        upload(c, dm, gamma, r * r);
        upload(c, dm + r * r, s_last, r * r);
        upload(c, dm + 2 * r * r, lambda, r);
        double* o = dm + 2 * r * r + r;
        CPDB_CK(cpdb::launch_fitness_als(nx2, dv, dv + rows * cols, rows * cols, dm,
                                         dm + 2 * r * r, dm + r * r, uint32_t(r), o, c->stream));
        double h[2];
        download(c, h, o, 2);
        *fitness = h[0];
        *raw = h[1];
    });
}

int cpdb_inner(cpdb_ctx* c, const double* a, const double* b, uint64_t n, double* out) {
    return guarded([&] {
        use_device(c);
        double* da = c->scratch_a.ensure(n + 1);
        double* db = c->scratch_b.ensure(n + 1);
        double* part = c->partials.ensure(cpdb::kNormBlocks + 8);
        upload(c, da, a, n);
        upload(c, db, b, n);
        CPDB_CK(cpdb::dot_dev(da, db, n, part, part + cpdb::kNormBlocks, c->stream));
        download(c, out, part + cpdb::kNormBlocks, 1);
    });
}

int cpdb_select_beta(double prev, double now, double gap, double* beta) {
    const double p = prev < 0.0 ? 0.0 : (prev > 1.0 ? 1.0 : prev);
    const double q = now < 0.0 ? 0.0 : (now > 1.0 ? 1.0 : now);
    if (beta) *beta = 0.0;
    if (std::fabs(q - p) >= gap) return 0;
    if (beta) *beta = q > 0.90 ? 1.0 / 2000.0 : (q >= 0.70 ? 1.0 / 500.0 : 1.0 / 250.0);
    return 1;
}

// ---------------------------------------------------------------- scheduler
int cpdb_schedule_build(uint32_t order, int32_t strategy, uint64_t iterations, int64_t* steps,
                        uint64_t cap, uint64_t* n_steps, uint64_t* cycle) {
    return guarded([&] {
        if (strategy < 0 || strategy > 2) fail(CPDB_INVALID_ARGUMENT, "unknown strategy");
        const cpdb::Plan p =
            cpdb::build_plan(order, static_cast<cpdb::Strategy>(strategy), iterations);
        uint64_t n = 0;
        for (uint64_t i = 0; i < p.sweeps.size(); ++i)
            for (uint64_t b = 0; b < p.sweeps[i].updates.size(); ++b)
                for (const auto& s : p.sweeps[i].updates[b].steps) {
                    if (n < cap && steps) {
                        int64_t* r = steps + 6 * n;
                        r[0] = int64_t(i);
                        r[1] = int64_t(b);
                        r[2] = p.sweeps[i].updates[b].mode;
                        r[3] = s.source;
                        r[4] = s.contract;
                        r[5] = s.produces;
                    }
                    ++n;
                }
        if (n_steps) *n_steps = n;
        if (cycle) {
            cycle[0] = p.cycle_start;
            cycle[1] = p.cycle_length;
        }
    });
}

int cpdb_schedule_validate(uint32_t order, const int64_t* steps, uint64_t n_steps,
                           uint64_t iterations) {
    return guarded([&] { cpdb::validate_plan(plan_from_steps(order, steps, n_steps, iterations)); });
}

int cpdb_retained_keys(uint32_t order, const int64_t* steps, uint64_t n_steps,
                       uint64_t iterations, uint64_t cycle_start, uint64_t cycle_length,
                       uint64_t iteration, uint64_t block, uint32_t* keys, uint64_t cap,
                       uint64_t* n_keys) {
    return guarded([&] {
        cpdb::Plan p = plan_from_steps(order, steps, n_steps, iterations);
        p.cycle_start = cycle_start;
        p.cycle_length = std::max<uint64_t>(cycle_length, 1);
        if (iteration >= p.sweeps.size()) fail(CPDB_INVALID_ARGUMENT, "retained_keys: iteration");
        const auto k = cpdb::retained_keys(p, iteration, uint32_t(block));
        *n_keys = k.size();
        for (size_t i = 0; i < k.size() && i < cap; ++i) keys[i] = k[i];
    });
}

int cpdb_measured_cost(uint32_t order, int32_t strategy, const uint64_t* dims, uint64_t rank,
                       uint64_t iterations, uint64_t* total_flops, uint64_t* root_ttms) {
    return guarded([&] {
        if (strategy < 0 || strategy > 2) fail(CPDB_INVALID_ARGUMENT, "unknown strategy");
        const cpdb::Plan p =
            cpdb::build_plan(order, static_cast<cpdb::Strategy>(strategy), iterations);
        const cpdb::Cost cst =
            cpdb::measured_cost(p, std::vector<uint64_t>(dims, dims + order), rank, iterations);
        *total_flops = cst.flops;
        *root_ttms = cst.roots;
    });
}

int cpdb_shard_plan(uint32_t order, int32_t strategy, uint64_t iterations, const uint64_t* dims,
                    uint64_t rank, int world, int32_t* flags, uint64_t* payload, uint64_t cap,
                    uint64_t* n_steps) {
    return guarded([&] {
        if (strategy < 0 || strategy > 2) fail(CPDB_INVALID_ARGUMENT, "unknown strategy");
        if (world < 1) fail(CPDB_INVALID_ARGUMENT, "shard_plan: world must be >= 1");
        if (dims == nullptr || n_steps == nullptr) fail(CPDB_INVALID_ARGUMENT, "shard_plan: null");
        const cpdb::Plan p =
            cpdb::build_plan(order, static_cast<cpdb::Strategy>(strategy), iterations);
        const bool dist = world > 1;
        uint64_t i = 0;
        for (const auto& sw : p.sweeps)
            for (const auto& up : sw.updates)
                for (size_t j = 0; j < up.steps.size(); ++j) {
                    const cpdb::Step& st = up.steps[j];
                    int32_t f = cpdb::shard_flags(st.source, st.contract, st.produces, up.mode,
                                                  dist);
                    if (j + 1 != up.steps.size()) f &= ~cpdb::kGatherV;
                    uint64_t words = 0;
                    if (f & cpdb::kAllReduce) {
                        words = 1;
                        for (uint32_t k = 0; k < order; ++k)
                            words *= (st.produces & (1u << k)) ? dims[k] : rank;
                    }
                    if (f & cpdb::kGatherV) words += dims[0] * rank;
                    if (i < cap) {
                        if (flags) flags[i] = f;
                        if (payload) payload[i] = words;
                    }
                    ++i;
                }
        *n_steps = i;
    });
}

int cpdb_shard_plan_ex(uint32_t order, int32_t strategy, uint64_t iterations,
                       const uint64_t* dims, uint64_t rank, int world, int32_t policy,
                       const cpdb_shard_cost* cost, cpdb_shard_step* steps, uint64_t cap_steps,
                       uint64_t* n_steps, int32_t* vop, uint64_t* vwords, uint64_t cap_updates,
                       uint64_t* n_updates, double* est) {
    return guarded([&] {
        if (strategy < 0 || strategy > 2) fail(CPDB_INVALID_ARGUMENT, "unknown strategy");
        if (policy < 0 || policy > 3) fail(CPDB_INVALID_ARGUMENT, "shard_plan: unknown policy");
        if (world < 1) fail(CPDB_INVALID_ARGUMENT, "shard_plan: world must be >= 1");
        if (dims == nullptr) fail(CPDB_INVALID_ARGUMENT, "shard_plan: null dims");
        if (rank == 0) fail(CPDB_INVALID_ARGUMENT, "shard_plan: rank must be >= 1");
        const cpdb::Plan p =
            cpdb::build_plan(order, static_cast<cpdb::Strategy>(strategy), iterations);
        cpdb::ShardCost cp;
        if (cost) {
            if (cost->tflops > 0) cp.tflops = cost->tflops;
            if (cost->bus_gbs > 0) cp.bus_gbs = cost->bus_gbs;
            if (cost->latency_s >= 0) cp.latency_s = cost->latency_s;
        }
        const cpdb::ShardPlan sp =
            cpdb::plan_shards(p, std::vector<uint64_t>(dims, dims + order), rank, world,
                              static_cast<cpdb::ShardPolicy>(policy), cp);
        uint64_t i = 0, u = 0;
        for (size_t sw = 0; sw < sp.steps.size(); ++sw)
            for (size_t b = 0; b < sp.steps[sw].size(); ++b) {
                for (const cpdb::StepShard& st : sp.steps[sw][b]) {
                    if (steps && i < cap_steps)
                        steps[i] = cpdb_shard_step{st.src.kind, st.src.mode, st.out.kind,
                                                   st.out.mode, st.red, st.scatter, st.words};
                    ++i;
                }
                const cpdb::UpdateShard& us = sp.updates[sw][b];
                if (u < cap_updates) {
                    if (vop) vop[u] = us.vop;
                    if (vwords) vwords[u] = us.vwords;
                }
                ++u;
            }
        if (n_steps) *n_steps = i;
        if (n_updates) *n_updates = u;
        if (est) {
            est[0] = sp.est_compute_s;
            est[1] = sp.est_comm_s;
        }
    });
}

int cpdb_set_shard_policy(cpdb_ctx* c, int32_t policy, const cpdb_shard_cost* cost) {
    return guarded([&] {
        if (!c) fail(CPDB_INVALID_ARGUMENT, "null context");
        if (policy < 0 || policy > 3) fail(CPDB_INVALID_ARGUMENT, "unknown shard policy");
        c->shard_policy = policy;
        if (cost) {
            if (cost->tflops > 0) c->shard_cost.tflops = cost->tflops;
            if (cost->bus_gbs > 0) c->shard_cost.bus_gbs = cost->bus_gbs;
            if (cost->latency_s >= 0) c->shard_cost.latency_s = cost->latency_s;
        }
    });
}

int cpdb_closed_form_cost(uint32_t order, int32_t strategy, const uint64_t* dims, uint64_t rank,
                          uint64_t* total) {
    return guarded([&] {
        if (strategy < 0 || strategy > 2) fail(CPDB_INVALID_ARGUMENT, "unknown strategy");
        *total = cpdb::closed_form_cost(order, static_cast<cpdb::Strategy>(strategy),
                                        std::vector<uint64_t>(dims, dims + order), rank);
    });
}

int cpdb_leading_flop_coefficient(uint32_t order, int32_t strategy, uint64_t* coeff) {
    return guarded([&] {
        if (strategy < 0 || strategy > 2) fail(CPDB_INVALID_ARGUMENT, "unknown strategy");
        *coeff = cpdb::leading_flop_coefficient(order, static_cast<cpdb::Strategy>(strategy));
    });
}

// ---------------------------------------------------------------- device execute()
int cpdb_exec_step(cpdb_ctx* c, uint32_t source, uint32_t contract, uint32_t produces,
                   const double* q, uint64_t rank) {
    return guarded([&] {
        use_device(c);
        if (c->world > 1) fail(CPDB_INVALID_ARGUMENT, "exec_step: single-GPU contexts only");
        cpdb::require_tensor(c);
        const uint32_t order = uint32_t(c->dims.size());
        if (contract >= order) fail(CPDB_INVALID_ARGUMENT, "execute: contract mode out of range");
        if (rank == 0) fail(CPDB_INVALID_ARGUMENT, "execute: rank must be >= 1");
        const double* src;
        std::vector<uint64_t> sd;
        if (source == CPDB_ROOT_KEY) {
            src = c->x;
            sd = c->ldims;
        } else {
            auto it = c->slots.find(source);
            if (it == c->slots.end() || !it->second.valid)
                fail(CPDB_LOGIC_ERROR, "execute: scheduled source missing from cache");
            src = it->second.buf.p;
            sd = it->second.dims;
        }
        if (source != CPDB_ROOT_KEY && source == produces)
            fail(CPDB_INVALID_ARGUMENT, "execute: produced set equals its source");
        const uint64_t K = sd[contract];
        std::vector<uint64_t> od = sd;
        od[contract] = rank;
        double* dq = c->scratch_a.ensure(K * rank);
        upload(c, dq, q, K * rank);
        cpdb::DevBuf packed;
        double* qp = nullptr;
        qp = packed.ensure(uint64_t(cpdb::ttm_kpad(K)) * cpdb::ttm_rpad(uint32_t(rank)));
        CPDB_CK(cpdb::pack_q(dq, qp, uint32_t(K), uint32_t(rank), c->stream));
        cpdb::Slot& sl = c->slots[produces];
        double* dst = sl.buf.ensure(cpdb::numel(od));
        cpdb::run_ttm(c, src, sd, contract, dq, qp, uint32_t(rank), dst);
        CPDB_CK(cudaStreamSynchronize(c->stream));
        sl.valid = true;
        sl.dims = od;
    });
}

int cpdb_cache_dims(cpdb_ctx* c, uint32_t key, uint64_t* dims, int32_t* present) {
    return guarded([&] {
        auto it = c->slots.find(key);
        const bool ok = it != c->slots.end() && it->second.valid;
        if (present) *present = ok ? 1 : 0;
        if (ok && dims)
            for (size_t k = 0; k < it->second.dims.size(); ++k) dims[k] = it->second.dims[k];
    });
}

int cpdb_cache_get(cpdb_ctx* c, uint32_t key, double* host) {
    return guarded([&] {
        use_device(c);
        auto it = c->slots.find(key);
        if (it == c->slots.end() || !it->second.valid)
            fail(CPDB_LOGIC_ERROR, "cache_get: key not present");
        download(c, host, it->second.buf.p, cpdb::numel(it->second.dims));
    });
}

int cpdb_cache_drop(cpdb_ctx* c, uint32_t key) {
    return guarded([&] {
        auto it = c->slots.find(key);
        if (it != c->slots.end()) it->second.valid = false;
    });
}

}  // extern "C"
