/* cpdb -- C ABI of the B200-native CP-ALS-QR hot path (libcpdb.so).
 *
 * This is the drop-in boundary: the reference has no FFI of its own (it is
 * the header-only C++ library `cpd`, /root/reference/proj/include/cpd), so the
 * entry points below are exactly the calls its C++ API needs when it is
 * re-pointed at the GPU.  The C++ headers in include/cpd/*.hpp keep the
 * reference names and signatures and call only this ABI; INTEGRATION.md shows
 * the CMake/ctypes bindings.  Each entry point cites the reference interface
 * it replaces (path:line under /root/reference/proj/include/cpd).
 *
 * Conventions
 *  - plain pointers and sizes only; every tensor is FP64, row-major with the
 *    LAST index fastest (tensor.hpp:42-47), matrices row-major;
 *  - every call returns a status code (CPDB_OK == 0); cpdb_last_error() holds
 *    the message of the last failure on the calling thread.  The C++ headers
 *    rethrow the reference's exception type for each code (cli.hpp:230-250
 *    maps the same classes to exit codes);
 *  - a context owns one device, one stream and every device buffer; calls on
 *    one context are synchronous at return and not thread-safe (the reference
 *    is single-threaded);
 *  - there is no CPU fallback: without a usable B200 every compute call fails
 *    with CPDB_CUDA_ERROR.
 */
#ifndef CPDB_H
#define CPDB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define CPDB_OK 0
#define CPDB_INVALID_ARGUMENT 1     /* std::invalid_argument                       */
#define CPDB_STALE_INTERMEDIATE 2   /* stale_intermediate_error dim_tree.hpp:21-23  */
#define CPDB_SINGULAR_TRIANGULAR 3  /* singular_triangular_error linalg.hpp:19-26   */
#define CPDB_LOGIC_ERROR 4          /* std::logic_error (missing cache source ...)  */
#define CPDB_CUDA_ERROR 5           /* device / driver failure (no fallback)        */
#define CPDB_NCCL_ERROR 6
#define CPDB_OUT_OF_MEMORY 7
#define CPDB_FILE_ERROR 8           /* file_error   io.hpp:21-23 (open/read/write)  */
#define CPDB_FORMAT_ERROR 9         /* format_error io.hpp:25-27 (malformed file)   */
#define CPDB_SINGULAR_SYSTEM 10     /* singular_system_error linalg.hpp (solve_spd) */

#define CPDB_MAX_ORDER 8
#define CPDB_ROOT_KEY 0xFFFFFFFFu   /* "the input tensor X" as a step source       */

typedef struct cpdb_ctx cpdb_ctx;

/* reference: solvers.hpp:56-66 TraceRow */
typedef struct {
    uint64_t iteration;                    /* 1-based sweep                      */
    uint32_t order;                        /* entries used in update_order       */
    uint32_t update_order[CPDB_MAX_ORDER]; /* 0-based modes                      */
    uint32_t pad0;
    double fitness;
    double raw_radicand;
    double wall_seconds;                   /* device clock since the solve began */
    uint64_t root_ttm_count;               /* cumulative (dim_tree.hpp:143-158)  */
    uint64_t flops;                        /* cumulative TTM flops               */
    double beta_used;
    int32_t regularized;
    int32_t pad1;
} cpdb_trace_row;

/* reference: solvers.hpp:25-50 SolverConfig.  extrapolate=1 selects
 * als_qr_bre (forces branch reuse, solvers.hpp:329-336); 0 selects cp_als_qr
 * with `strategy` (solvers.hpp:317-322). */
typedef struct {
    uint64_t rank;
    uint64_t max_iterations;
    double fitness_threshold;
    int32_t strategy;      /* 0 naive, 1 dim-tree, 2 branch-reuse (dim_tree.hpp:25) */
    int32_t extrapolate;
    double alpha;
    int32_t has_beta_override;
    int32_t pad0;
    double beta_override;
    double activation_gap;
    uint64_t seed;         /* initial factors: Rng(seed) N(0,1), solvers.hpp:116-122 */
} cpdb_config;

/* Sweep-boundary solver state (resume / teacher forcing).  Everything
 * run_qr carries between sweeps except the branch-reuse cache, which is
 * rebuilt from X and the factors (freshness invariant dim_tree.hpp:109-111).
 * Buffers are caller-owned host memory; on return they hold the end state. */
typedef struct {
    uint64_t sweeps_done;
    double* lambda;        /* R                                                  */
    double* factors;       /* concatenated I_k x R, mode order                   */
    double* q0_history;    /* concatenated R^(N-1) x R per mode, reference row order */
    uint32_t history_mask; /* bit n: history of mode n valid                     */
    int32_t has_active_beta;
    double active_beta;
    int32_t has_prev_fitness;
    int32_t pad0;
    double prev_fitness;
} cpdb_state;

/* q0_observer (solvers.hpp:37-39): Q0 before extrapolation, reference row order */
typedef void (*cpdb_q0_observer)(void* user, uint64_t sweep, uint32_t mode, const double* q0,
                                 uint64_t rows, uint64_t cols);

/* Device-measured timing of the last cpdb_solve (CUDA events on the solve
 * stream).  Root TTM = a step whose source is X (dim_tree.hpp:526). */
typedef struct {
    uint64_t sweeps;
    double solve_ms;          /* first sweep start -> last sweep end               */
    double sweep1_ms;         /* sweep 1 (dim-tree sweep, two root TTMs)           */
    uint64_t root_ttms;       /* root TTM launches timed                           */
    double root_ttm_ms;       /* summed root TTM kernel time                       */
    double root_ttm_flops;    /* algorithmic 2*|Y|*I_c summed over timed launches  */
    double root_ttm_bytes;    /* algorithmic 8*(|X| + |Y| + I_c*R) summed          */
    double branch_ttm_ms;     /* non-root TTM steps                                */
    double mode_update_ms;    /* Z-QR, V-GEMM and finisher kernels (solve,
                                 normalise, factor QR, fit), summed; timed only
                                 with CPDB_TIME_TAILS=1, else 0                   */
    double comm_ms;           /* NCCL reductions (sharded contexts)                */
    uint64_t kernel_launches; /* device kernels launched by the solve              */
    uint64_t qr_shifted;      /* sweeps in which a CholeskyQR first pass needed the
                                 shifted retry (kappa beyond ~1e8)                 */
    uint64_t qr_householder;  /* solves restarted on the Householder kernels after
                                 a CholeskyQR breakdown the retry could not cure   */
    uint64_t gate_mispredictions; /* updates issued ahead on "the beta gate stays
                                 closed" and issued again when it opened (once
                                 per run at most)                                  */
} cpdb_profile;

/* ---- version / device ----------------------------------------------------- */
const char* cpdb_version(void);
const char* cpdb_last_error(void);
/* 1 when a device of compute capability 10.x is usable */
int cpdb_device_ok(int device);

/* ---- context ---------------------------------------------------------------- */
int cpdb_create(int device, cpdb_ctx** out);
/* One rank of a mode-1 (index 0) sharded run: X's leading mode is split in
 * contiguous slabs over `world` GPUs and TTMs that contract it are summed with
 * NCCL all-reduce.  nccl_id: 128 bytes from
 * cpdb_nccl_unique_id on rank 0, broadcast by the caller. */
int cpdb_create_sharded(int device, int rank, int world, const void* nccl_id, cpdb_ctx** out);
int cpdb_nccl_unique_id(void* out128);
/* The NCCL calls of the sharded path (all-reduce, all-gather, grouped
 * per-slice reduce-scatter) on a one-rank communicator of `device`:
 * *max_err = max |result - input| (0 when the transport works).  Checks the
 * dlopen'ed NCCL on a single-GPU box, where no multi-rank run is possible. */
int cpdb_nccl_selftest(int device, double* max_err);
/* `world` ranks of a mode-1 sharded run inside ONE process on ONE device,
 * each to be driven by its own host thread; the collectives go through a
 * shared device buffer and host barriers instead of NCCL.  For exercising the
 * sharded path on a single GPU (tests); out holds `world` contexts. */
int cpdb_create_local_group(int device, int world, cpdb_ctx** out);
void cpdb_destroy(cpdb_ctx* ctx);
/* Row range of the leading mode owned by `rank` (host-only, no device). */
int cpdb_shard_rows(uint64_t extent0, int rank, int world, uint64_t* begin, uint64_t* count);

/* ---- the tensor X (device-resident) ------------------------------------------ */
/* Upload from host memory.  Sharded contexts take the rank's slab of the
 * leading mode (rows [begin, begin+count) from cpdb_shard_rows) and the
 * GLOBAL dims. */
int cpdb_tensor_set(cpdb_ctx* ctx, const double* host, const uint64_t* dims, uint32_t order);
/* The same upload without waiting for it: the copy is queued on the context's
 * stream and every later call on the context is ordered behind it (the next
 * call that synchronises -- cpdb_solve, cpdb_session_begin, cpdb_tensor_norm_sq
 * -- also completes it).  `host` must stay valid and unchanged until then;
 * page-locked memory makes the copy truly asynchronous, so the host side of
 * the following cpdb_session_begin / cpdb_solve runs under it. */
int cpdb_tensor_set_async(cpdb_ctx* ctx, const double* host, const uint64_t* dims,
                          uint32_t order);
/* Borrow an existing device buffer (no copy; caller keeps it alive). */
int cpdb_tensor_set_device(cpdb_ctx* ctx, const double* device_ptr, const uint64_t* dims,
                           uint32_t order);
/* Fill X on the device with the BASELINE construction (DESIGN.md "Synthetic
 * inputs"): kind 0 i.i.d. N(0,1) factors, kind 1 congruent/log-scaled
 * columns; + rho-relative Gaussian noise.  Counter-based RNG: the bytes depend
 * on (seed, dims, rank) only, not on the shard layout. */
int cpdb_tensor_synth(cpdb_ctx* ctx, int32_t kind, const uint64_t* dims, uint32_t order,
                      uint64_t rank, double rho, uint64_t seed);
/* The truth factors cpdb_tensor_synth builds X from (sum I_k x R doubles,
 * mode after mode, lambda = 1): X_clean = reconstruct(factors) (kruskal.hpp:54-67). */
int cpdb_tensor_synth_truth(cpdb_ctx* ctx, int32_t kind, const uint64_t* dims, uint32_t order,
                            uint64_t rank, uint64_t seed, double* factors);
/* Of the context's last cpdb_tensor_synth: out[0] = ||X_clean||^2 and out[1] =
 * ||E||^2 of the unscaled noise draw (global over the ranks; 0 when rho = 0).
 * X = X_clean + rho sqrt(out[0] / out[1]) E. */
int cpdb_tensor_synth_norms(cpdb_ctx* ctx, double* out);
int cpdb_tensor_get(cpdb_ctx* ctx, double* host);
/* .cpdt tensor files (io.hpp:93-121: "CPDT", u8 version 1, u8 order, u64
 * extents, f64 values little-endian, row-major).  load streams the payload
 * straight into HBM through pinned double-buffered chunks (a sharded context
 * reads only its mode-0 slab) and rejects what decode_tensor rejects (bad
 * magic / version / extent, truncated or trailing bytes, non-finite values)
 * with CPDB_FORMAT_ERROR; save writes an unsharded context's X. */
int cpdb_tensor_load_cpdt(cpdb_ctx* ctx, const char* path);
int cpdb_tensor_save_cpdt(cpdb_ctx* ctx, const char* path);
/* Header only: order and extents (dims holds CPDB_MAX_ORDER entries). */
int cpdb_cpdt_info(const char* path, uint32_t* order, uint64_t* dims);
/* ||X||^2 (tensor.hpp:394-399 inner(x, x)), deterministic reduction */
int cpdb_tensor_norm_sq(cpdb_ctx* ctx, double* out);

/* ---- the solver (solvers.hpp:215-336) ------------------------------------------ */
/* Runs cp_als_qr / als_qr_bre on the context's X entirely in HBM.  state may
 * be NULL (fresh run).  trace holds max_iterations rows.  factors_per_sweep
 * (max_iterations x sum I_k R) and lambda_per_sweep (max_iterations x R) are
 * optional per-sweep dumps for parity checks.  Ranks up to 1024 (the tuned
 * kernels up to 64, rank-generic ones beyond).  A CholeskyQR breakdown that the
 * shifted retry cannot cure restarts the run on the Householder kernels, as
 * the reference's thin_qr (linalg.hpp:39-99) never breaks down
 * (cpdb_profile.qr_householder counts the restarts). */
int cpdb_solve(cpdb_ctx* ctx, const cpdb_config* cfg, cpdb_state* state, cpdb_trace_row* trace,
               uint64_t* trace_len, double* out_lambda, double* out_factors,
               double* factors_per_sweep, double* lambda_per_sweep, cpdb_q0_observer observer,
               void* observer_user);
/* The same run as a resumable session: begin = run_qr setup
 * (solvers.hpp:217-241), run = n more sweeps of the loop (:243-302), end =
 * model + sweep-boundary state (:304-308).  cfg->max_iterations bounds the
 * plan; *finished is set once it is exhausted or the fitness threshold hit.
 * While sweeps remain, run() leaves the next sweep's first update in flight
 * on the device (the following run() consumes it); end() takes it back, so
 * the exported state is the one after the sweeps that were run, and a
 * session that was ended in the middle accepts no further run()
 * (CPDB_LOGIC_ERROR): begin a new one from the exported state. */
typedef struct cpdb_session cpdb_session;
int cpdb_session_begin(cpdb_ctx* ctx, const cpdb_config* cfg, const cpdb_state* state,
                       cpdb_session** out);
int cpdb_session_run(cpdb_session* s, uint64_t sweeps, cpdb_trace_row* trace, uint64_t* rows,
                     int32_t* finished);
int cpdb_session_end(cpdb_session* s, cpdb_state* state, double* out_lambda,
                     double* out_factors);
void cpdb_session_destroy(cpdb_session* s);
int cpdb_profile_get(cpdb_ctx* ctx, cpdb_profile* out);
/* Enable/disable per-kernel event timing inside cpdb_solve (default on; off
 * removes the events from the stream), and the root-TTM overlap (default on:
 * a branch-reuse sweep's root TTM is issued on a low-priority stream under
 * the preceding update; off runs every TTM in schedule order on the solve
 * stream -- the kernel alone, e.g. for roofline measurements). */
int cpdb_set_options(cpdb_ctx* ctx, int32_t timing, int32_t overlap);

/* ---- CP-ALS through the normal equations ---------- */
/* reference: solvers.hpp:149-208 cp_als.  Device-resident run on the
 * context's tensor: per mode MTTKRP (TTM + Khatri-Rao contraction), Gamma =
 * Hadamard of the other Grams, solve_spd, normalize_columns, Gram; fitness
 * (fitness_fast_als) once per sweep.  init_factors (sum I_k x R, mode after
 * mode) / init_lambda (R) are the optional KruskalModel init; trace has
 * max_iterations rows (root_ttm_count 0, beta_used 0, regularized = a ridge
 * retry happened in the sweep).  CPDB_SINGULAR_SYSTEM when the ridge fails. */
int cpdb_als_solve(cpdb_ctx* ctx, const cpdb_config* cfg, const double* init_lambda,
                   const double* init_factors, cpdb_trace_row* trace, uint64_t* trace_len,
                   double* out_lambda, double* out_factors);
/* reference: tensor.hpp:453-488 mttkrp (and :494-518 mttkrp_materialized,
 * the same product).  t: host tensor; factors[k]: host I_k x R (factors[mode]
 * unused, may be NULL) with their shapes; out: dims[mode] x R. */
int cpdb_mttkrp(cpdb_ctx* ctx, const double* t, const uint64_t* dims, uint32_t order,
                const double* const* factors, const uint64_t* factor_rows,
                const uint64_t* factor_cols, uint32_t mode, double* out);
/* reference: linalg.hpp:132-187 solve_spd: x G = rhs (x, rhs: rows x n),
 * Cholesky with one 1e-12 trace/n ridge retry (*regularized = 1). */
int cpdb_solve_spd(cpdb_ctx* ctx, const double* g, uint64_t g_rows, uint64_t g_cols,
                   const double* rhs, uint64_t rows, uint64_t cols, double* x,
                   int32_t* regularized);
/* reference: kruskal.hpp:88-104 fitness_fast_als. */
int cpdb_fitness_fast_als(cpdb_ctx* ctx, double norm_x_sq, const double* m, const double* a_hat,
                          uint64_t rows, uint64_t cols, const double* gamma,
                          const double* lambda, uint64_t r, const double* s_last,
                          double* fitness, double* raw);

/* ---- dense primitives on host buffers (device compute) ------------------------ */
int cpdb_ttm(cpdb_ctx* ctx, const double* t, const uint64_t* dims, uint32_t order,
             const double* b, uint64_t b_rows, uint32_t mode, double* out); /* tensor.hpp:288 */
int cpdb_unfold(cpdb_ctx* ctx, const double* t, const uint64_t* dims, uint32_t order,
                uint32_t mode, double* out);                                   /* tensor.hpp:217 */
int cpdb_khatri_rao(cpdb_ctx* ctx, const double* const* mats, const uint64_t* rows,
                    uint32_t count, uint64_t cols, double* out);               /* tensor.hpp:343 */
int cpdb_thin_qr(cpdb_ctx* ctx, const double* a, uint64_t m, uint64_t n, double* q,
                 double* r);                                                   /* linalg.hpp:39 */
int cpdb_solve_rows_lower(cpdb_ctx* ctx, const double* l, uint64_t n, const double* rhs,
                          uint64_t rows, double* out, int64_t* bad_column);    /* linalg.hpp:192 */
int cpdb_normalize_columns(cpdb_ctx* ctx, const double* a, uint64_t m, uint64_t n, double* out,
                           double* weights);                                   /* linalg.hpp:225 */
int cpdb_extrapolate_q0(cpdb_ctx* ctx, const double* now, const double* prev, uint64_t rows,
                        uint64_t cols, double beta, double alpha, double* out); /* solvers.hpp:75 */
int cpdb_fitness_fast_qr(cpdb_ctx* ctx, double norm_x_sq, const double* v, const double* a_hat,
                         uint64_t rows, const double* r0, const double* r_n, const double* lambda,
                         uint64_t r, double* fitness, double* raw);            /* kruskal.hpp:109 */
int cpdb_inner(cpdb_ctx* ctx, const double* a, const double* b, uint64_t n, double* out);
/* select_beta (solvers.hpp:92-101) is host logic: returns 1 and sets *beta
 * when extrapolation activates, 0 when it stays off. */
int cpdb_select_beta(double fitness_prev, double fitness_now, double gap, double* beta);

/* ---- scheduler (host metadata, dim_tree.hpp:191-634) ------------------------- */
/* Steps flattened as 6 x int64: {iteration, block, mode, source, contract, produces}. */
int cpdb_schedule_build(uint32_t order, int32_t strategy, uint64_t iterations, int64_t* steps,
                        uint64_t cap_steps, uint64_t* n_steps, uint64_t* cycle /*[2]*/);
int cpdb_schedule_validate(uint32_t order, const int64_t* steps, uint64_t n_steps,
                           uint64_t iterations);
int cpdb_retained_keys(uint32_t order, const int64_t* steps, uint64_t n_steps,
                       uint64_t iterations, uint64_t cycle_start, uint64_t cycle_length,
                       uint64_t iteration, uint64_t block, uint32_t* keys, uint64_t cap,
                       uint64_t* n_keys);
int cpdb_measured_cost(uint32_t order, int32_t strategy, const uint64_t* dims, uint64_t rank,
                       uint64_t iterations, uint64_t* total_flops, uint64_t* root_ttms);
int cpdb_closed_form_cost(uint32_t order, int32_t strategy, const uint64_t* dims, uint64_t rank,
                          uint64_t* total);
int cpdb_leading_flop_coefficient(uint32_t order, int32_t strategy, uint64_t* coeff);

/* ---- mode-0 sharding plan (no reference counterpart: the
 * reference is single-process) ------------------------------------------------
 * For the steps of cpdb_schedule_build(order, strategy, iterations), in the
 * same order, flags[i] is a CPDB_SHARD_* bit set and payload[i] the number of
 * doubles the step exchanges (all-reduce of a partial sum, or the all-gather
 * of V = I_0 x R after the mode-0 update's last step), for `world` ranks over
 * dims (global extents).  The device session uses the same rule. */
#define CPDB_SHARD_SRC_SHARDED 1
#define CPDB_SHARD_ALLREDUCE 2
#define CPDB_SHARD_OUT_SHARDED 4
#define CPDB_SHARD_GATHER_V 8
int cpdb_shard_plan(uint32_t order, int32_t strategy, uint64_t iterations, const uint64_t* dims,
                    uint64_t rank, int world, int32_t* flags, uint64_t* payload, uint64_t cap,
                    uint64_t* n_steps);

/* The reduction strategy of the sharded session (csrc/shard.cpp).  A TTM
 * contracting the shard mode of its source yields per-rank partial sums:
 *   EAGER    all-reduce them at once (replicated afterwards);
 *   SCATTER  reduce-scatter them onto another free mode (sharded afterwards,
 *            downstream TTMs stay divided over the ranks);
 *   LAZY     keep them partial down the chain and all-reduce V (I_n x R);
 *   AUTO     per step, the cheapest of the three by the cost model over the
 *            step's consumer tree (FP64 rate, NCCL bus bandwidth, latency).
 * V of a sharded Y(n) is all-gathered (its rows), of a partial one all-reduced. */
#define CPDB_SHARD_EAGER 0
#define CPDB_SHARD_SCATTER 1
#define CPDB_SHARD_LAZY 2
#define CPDB_SHARD_AUTO 3
#define CPDB_LAYOUT_REPLICATED 0
#define CPDB_LAYOUT_SHARDED 1
#define CPDB_LAYOUT_PARTIAL 2
#define CPDB_RED_NONE 0
#define CPDB_RED_ALLREDUCE 1
#define CPDB_RED_SCATTER 2
#define CPDB_V_NONE 0
#define CPDB_V_GATHER 1
#define CPDB_V_ALLREDUCE 2
typedef struct {
    int32_t src_layout, src_mode;  /* layout of the step's source (mode: the split one) */
    int32_t out_layout, out_mode;  /* layout of its stored output                     */
    int32_t reduction;             /* CPDB_RED_* applied to the step's output          */
    int32_t scatter_mode;          /* CPDB_RED_SCATTER: the free mode scattered onto   */
    uint64_t words;                /* doubles reduced (global partial size)            */
} cpdb_shard_step;
typedef struct {
    double tflops;     /* FP64 rate of the TTMs per GPU (default 30)                 */
    double bus_gbs;    /* NCCL bus bandwidth (default 700, NVLink 5 / NVSwitch)      */
    double latency_s;  /* per collective (default 20e-6)                             */
} cpdb_shard_cost;
/* steps: one record per scheduled step (same order as cpdb_schedule_build);
 * vop / vwords: per mode update, V's collective and its size; est[0] / est[1]:
 * the model's per-rank compute / communication seconds for the whole plan.
 * cost may be NULL (defaults). */
int cpdb_shard_plan_ex(uint32_t order, int32_t strategy, uint64_t iterations,
                       const uint64_t* dims, uint64_t rank, int world, int32_t policy,
                       const cpdb_shard_cost* cost, cpdb_shard_step* steps, uint64_t cap_steps,
                       uint64_t* n_steps, int32_t* vop, uint64_t* vwords, uint64_t cap_updates,
                       uint64_t* n_updates, double* est);
/* The policy a context's sessions use (default AUTO; env CPDB_SHARD_POLICY
 * = eager|scatter|lazy|auto overrides at context creation). */
int cpdb_set_shard_policy(cpdb_ctx* ctx, int32_t policy, const cpdb_shard_cost* cost);

/* ---- device-resident execute() (dim_tree.hpp:473-544) ------------------------- */
/* One scheduled TTM on the device: reads X (source == CPDB_ROOT_KEY) or the
 * cache slot `source`, contracts `contract` with Q (I_c x R host matrix, the
 * reference passes transpose(Q), dim_tree.hpp:519) and writes cache slot
 * `produces`.  Freshness stamps and eviction policy stay in the caller
 * (include/cpd/dim_tree.hpp), exactly as the reference keeps them on the host. */
int cpdb_exec_step(cpdb_ctx* ctx, uint32_t source, uint32_t contract, uint32_t produces,
                   const double* q, uint64_t rank);
int cpdb_cache_dims(cpdb_ctx* ctx, uint32_t key, uint64_t* dims /*[order]*/, int32_t* present);
int cpdb_cache_get(cpdb_ctx* ctx, uint32_t key, double* host);
int cpdb_cache_drop(cpdb_ctx* ctx, uint32_t key);

#ifdef __cplusplus
}
#endif
#endif
