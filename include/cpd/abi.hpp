// Glue between the drop-in `cpd::` headers and libcpdb.so (include/cpdb.h).
//
// The reference library (/root/reference/proj/include/cpd) is header-only
// C++ that computes on the host.  These headers keep its names, signatures and
// value types, and route every hot-path computation through the C ABI into
// the sm_100a kernels.  There is no host fallback: without a B200 the first
// call throws `cpd::device_error`.
//
// Error mapping (cpdb.h status -> the exception type the reference throws):
//   CPDB_INVALID_ARGUMENT     std::invalid_argument
//   CPDB_STALE_INTERMEDIATE   cpd::stale_intermediate_error  (dim_tree.hpp:20-22)
//   CPDB_SINGULAR_TRIANGULAR  cpd::singular_triangular_error (linalg.hpp:18-25)
//   CPDB_LOGIC_ERROR          std::logic_error
//   CPDB_SINGULAR_SYSTEM      cpd::singular_system_error     (linalg.hpp:15-17)
//   anything else             cpd::device_error (CUDA / NCCL / OOM)
#pragma once

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cpdb.h"

namespace cpd {

struct singular_system_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct singular_triangular_error : std::runtime_error {
    singular_triangular_error(std::size_t col, double diag)
        : std::runtime_error("triangular solve: diagonal entry of column " + std::to_string(col) +
                             " is " + std::to_string(diag) +
                             " (rank-deficient Khatri-Rao factor)"),
          column(col) {}
    std::size_t column;
};

struct stale_intermediate_error : std::logic_error {
    using std::logic_error::logic_error;
};

// Device / driver failures: the reference has no counterpart (it never
// leaves the host); they are never mapped onto a host computation.
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace abi {

[[noreturn]] inline void raise(int status) {
    const std::string msg = cpdb_last_error();
    switch (status) {
        case CPDB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case CPDB_STALE_INTERMEDIATE: throw stale_intermediate_error(msg);
        case CPDB_SINGULAR_TRIANGULAR: throw singular_triangular_error(0, 0.0);
        case CPDB_LOGIC_ERROR: throw std::logic_error(msg);
        case CPDB_SINGULAR_SYSTEM: throw singular_system_error(msg);
        default: throw device_error("cpdb: " + msg);
    }
}

inline void check(int status) {
    if (status != CPDB_OK) raise(status);
}

// One device context per process for the value-type API (the reference's
// free functions carry no handle).  Device index from CPD_DEVICE (default 0).
class Context {
public:
    static cpdb_ctx* get() {
        static Context instance;
        return instance.ctx_;
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    ~Context() {
        if (ctx_) cpdb_destroy(ctx_);
    }

private:
    Context() {
        const char* env = std::getenv("CPD_DEVICE");
        check(cpdb_create(env ? std::atoi(env) : 0, &ctx_));
    }
    cpdb_ctx* ctx_ = nullptr;
};

inline cpdb_ctx* ctx() { return Context::get(); }

inline std::vector<uint64_t> u64(const std::vector<std::size_t>& v) {
    return std::vector<uint64_t>(v.begin(), v.end());
}

}  // namespace abi
}  // namespace cpd
