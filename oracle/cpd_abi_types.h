/* Plain-C value types shared by the two CPU checkers under oracle/ (the
 * reference runner oracle/ref_runner.cpp and the C restatement
 * oracle/cpd_oracle.c).  They mirror the layout of the product's types in
 * include/cpdb.h so one ctypes description serves all three libraries.
 *
 * TEST INFRASTRUCTURE ONLY: nothing on the product path includes this file.
 */
#ifndef CPD_ORACLE_ABI_TYPES_H
#define CPD_ORACLE_ABI_TYPES_H

#include <stdint.h>

#define CPDO_MAX_ORDER 8

/* reference: solvers.hpp:56-66 (TraceRow) */
typedef struct {
    uint64_t iteration;
    uint32_t order;
    uint32_t update_order[CPDO_MAX_ORDER];
    uint32_t pad0;
    double fitness;
    double raw_radicand;
    double wall_seconds;
    uint64_t root_ttm_count;
    uint64_t flops;
    double beta_used;
    int32_t regularized;
    int32_t pad1;
} cpdo_trace_row;

/* reference: solvers.hpp:25-50 (SolverConfig).  `extrapolate` selects
 * als_qr_bre (1, forces branch reuse, solvers.hpp:329-336) or cp_als_qr (0,
 * solvers.hpp:317-322). */
typedef struct {
    uint64_t rank;
    uint64_t max_iterations;
    double fitness_threshold;
    int32_t strategy; /* 0 naive, 1 dim-tree, 2 branch-reuse (dim_tree.hpp:25) */
    int32_t extrapolate;
    double alpha;
    int32_t has_beta_override;
    int32_t pad0;
    double beta_override;
    double activation_gap;
    uint64_t seed;
} cpdo_config;

/* Solver state at a sweep boundary: everything run_qr carries from one sweep
 * to the next except the branch-reuse cache, which the freshness invariant
 * (dim_tree.hpp:109-111) lets us rebuild from X and the current factors. */
typedef struct {
    uint64_t sweeps_done;     /* 0 = fresh run */
    double* lambda;           /* R */
    double* factors;          /* concatenated I_k x R, row-major, mode order */
    double* q0_history;       /* concatenated R^(N-1) x R per mode (reference row order) */
    uint32_t history_mask;    /* bit n: q0 history of mode n present */
    int32_t has_active_beta;
    double active_beta;
    int32_t has_prev_fitness; /* fitness of sweep `sweeps_done` (for the beta gate) */
    int32_t pad0;
    double prev_fitness;
} cpdo_state;

typedef void (*cpdo_q0_observer)(void* user, uint64_t sweep, uint32_t mode, const double* q0,
                                 uint64_t rows, uint64_t cols);

#endif
