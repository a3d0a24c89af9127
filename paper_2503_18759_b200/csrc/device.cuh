// Shared device helpers for the sm_100a kernels of libcpdb.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cpdb {

constexpr int kWarp = 32;

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).  On sm_100a this
// is SASS DMMA.8x8x4 (tcgen05 has no f64 kind).  Fragment map:
//   A: lane holds A[lane/4][lane%4];  B: lane holds B[lane%4][lane/4];
//   C: lane holds C[lane/4][2*(lane%4) + {0,1}].
// Both operand fragments are "k = lane%4, other index = lane/4", so the same
// register can feed either side; swapping sides transposes the output tile.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async global->shared copy; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__host__ __device__ inline uint32_t ttm_rpad_dev(uint32_t R) { return ((R + 7) / 8) * 8; }

// Branch-free double reciprocal: MUFU approximation + two Newton steps
// (error <= 1 ulp; __drcp_rn's IEEE path carries a slow-path branch that
// keeps the scheduler from overlapping independent loads with it).
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// Programmatic dependent launch (PDL).  Hot-path kernels are launched with
// programmatic stream serialisation (launch_pdl / launch_cluster): the next
// kernel on the stream is scheduled while this one runs, and every kernel
// starts with pdl_wait() -- it returns once the previous grid has completed
// and its writes are visible (immediately when launched without PDL) -- then
// pdl_launch_dependents() lets the following kernel's launch overlap it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_entry() {
    pdl_wait();
    pdl_launch_dependents();
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

}  // namespace cpdb
