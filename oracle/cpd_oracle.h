/* C restatement of the reference CP-ALS-QR hot path (the CPU oracle).
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the GPU path is compared
 * against; it is loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg, never by the product library.  Every function restates
 * the reference algorithm in the same floating-point operation order so the
 * restatement is bit-identical to the reference (pinned in
 * tests/test_oracle_ref.py against oracle/_ref and tests/golden/).
 *
 * Citations are file:line under /root/reference/proj/include/cpd.
 */
#ifndef CPD_ORACLE_H
#define CPD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "cpd_abi_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same values as include/cpdb.h) */
#define CPDO_OK 0
#define CPDO_INVALID_ARGUMENT 1
#define CPDO_STALE 2
#define CPDO_SINGULAR_TRIANGULAR 3
#define CPDO_LOGIC 4
#define CPDO_OTHER 5

const char* cpdo_last_error(void);

/* rng.hpp:15-70 */
typedef struct {
    uint64_t s[4];
    double spare;
    int has_spare;
} cpdo_rng;
void cpdo_rng_seed(cpdo_rng* g, uint64_t seed);
uint64_t cpdo_rng_u64(cpdo_rng* g);
double cpdo_rng_uniform(cpdo_rng* g);
double cpdo_rng_normal(cpdo_rng* g);
int cpdo_rng_normals(uint64_t seed, uint64_t n, double* out);

/* tensor.hpp:288-315.  b is (b_rows x dims[mode]) row-major. */
int cpdo_ttm(const double* t, const uint64_t* dims, uint32_t order, const double* b,
             uint64_t b_rows, uint32_t mode, double* out);
/* tensor.hpp:217-250 */
int cpdo_unfold(const double* t, const uint64_t* dims, uint32_t order, uint32_t mode, double* out);
/* tensor.hpp:343-368, list order as given (last argument's row fastest) */
int cpdo_khatri_rao(const double* const* mats, const uint64_t* rows, uint32_t count, uint64_t cols,
                    double* out);
/* linalg.hpp:39-99 */
int cpdo_thin_qr(const double* a, uint64_t m, uint64_t n, double* q, double* r);
/* linalg.hpp:192-216: solve X L = RHS row-wise; *bad_column = failing column */
int cpdo_solve_rows_lower(const double* l, uint64_t n, const double* rhs, uint64_t rows,
                          double* out, int64_t* bad_column);
/* linalg.hpp:225-242 */
int cpdo_normalize_columns(const double* a, uint64_t m, uint64_t n, double* out, double* weights);
/* solvers.hpp:75-86 */
int cpdo_extrapolate_q0(const double* now, const double* prev, uint64_t rows, uint64_t cols,
                        double beta, double alpha, double* out);
/* solvers.hpp:92-101: returns 1 and sets *beta when extrapolation turns on */
int cpdo_select_beta(double prev, double now, double gap, double* beta);
/* kruskal.hpp:109-128 */
int cpdo_fitness_fast_qr(double norm_x_sq, const double* v, const double* a_hat, uint64_t rows,
                         const double* r0, const double* r_n, const double* lambda, uint64_t r,
                         double* fitness, double* raw);

/* dim_tree.hpp:386-426 flattened: per step {iteration, block, mode, source,
 * contract, produces}; cycle = {cycle_start, cycle_length} */
int cpdo_schedule(uint32_t order, int32_t strategy, uint64_t iterations, int64_t* out,
                  uint64_t cap_steps, uint64_t* n_steps, uint64_t* cycle);
/* dim_tree.hpp:433-465 */
int cpdo_retained_keys(uint32_t order, int32_t strategy, uint64_t iterations, uint64_t iter,
                       uint64_t block, uint32_t* out, uint64_t cap, uint64_t* n);
/* dim_tree.hpp:549-570 */
int cpdo_measured_cost(uint32_t order, int32_t strategy, const uint64_t* dims, uint64_t rank,
                       uint64_t iterations, uint64_t* total_flops, uint64_t* roots);

/* dim_tree.hpp:473-544 driven as dim_tree_test.cpp:37-73 */
int cpdo_execute_run(const double* x, const uint64_t* dims, uint32_t order, uint64_t rank,
                     int32_t strategy, uint64_t iterations, uint64_t seed,
                     const double* init_factors, double* y_out, uint64_t* flops_out);

/* solvers.hpp:215-336 (run_qr / cp_als_qr / als_qr_bre), resumable from a
 * sweep-boundary state (see cpd_abi_types.h) */
int cpdo_solve(const double* x, const uint64_t* dims, uint32_t order, const cpdo_config* cfg,
               cpdo_state* state, cpdo_trace_row* trace, uint64_t* trace_len, double* out_lambda,
               double* out_factors, double* factors_per_sweep, double* lambda_per_sweep,
               cpdo_q0_observer observer, void* observer_user);

/* kruskal.hpp:54-67 reconstruct (factors: sum I_k x R, mode after mode) */
int cpdo_reconstruct(const uint64_t* dims, uint32_t order, uint64_t rank, const double* lambda,
                     const double* factors, double* out);

/* BASELINE synthetic construction, same definition as cpdref_synth_baseline */
int cpdo_synth_baseline(int32_t kind, const uint64_t* dims, uint32_t order, uint64_t rank,
                        double rho, uint64_t seed, double* out, double* truth_factors);

#ifdef __cplusplus
}
#endif
#endif
