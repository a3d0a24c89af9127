// Launch interface of the libcpdb device kernels (host-callable).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cpdb {

// ---------------------------------------------------------------- K1/K2 TTM
struct TtmArgs {
    const double* x;   // source [outer][K][inner]
    double* y;         // result [outer][R][inner]
    const double* q;   // Q (K x R row-major) -- fallback path
    const double* qp;  // Q packed by pack_q -- tensor-core paths
    uint64_t outer, K, inner;
    uint32_t R, Rp;
    uint32_t Rtot;     // 0, or Y's extent when this launch writes a column block of it
    uint32_t tiles_per_cta;  // non-persistent form: tiles per CTA (0: CPDB_PREFETCH_TPC or 2)
    int one_tile_per_cta;  // non-persistent grid (a low-priority launch that
                           // yields SMs to concurrent work as its CTAs retire)
    int no_pdl;            // plain launch (the stream's previous op is an event wait)
    int no_tma;            // force the cp.async kernel (ttm.cu)
};
enum class TtmPath { groups, rows, simple };
TtmPath ttm_path(const TtmArgs& a);
cudaError_t launch_ttm(const TtmArgs& a, cudaStream_t s, int sms);
// warp-specialised TMA/DMMA kernel (ttm_tma.cu); cudaErrorNotSupported when
// the shape needs the cp.async kernel of ttm.cu
cudaError_t launch_ttm_tma(const TtmArgs& a, cudaStream_t s, int sms);
uint32_t ttm_kpad(uint64_t K);
uint32_t ttm_rpad(uint32_t R);
cudaError_t pack_q(const double* q, double* qp, uint32_t K, uint32_t R, cudaStream_t s);
// columns [c0, c0 + Rc) (Rc <= 64) of a K x ld row-major matrix, packed as a K x Rc Q
cudaError_t pack_q_cols(const double* q, uint32_t ld, uint32_t c0, uint32_t Rc, double* qp,
                        uint32_t K, cudaStream_t s);

// ---------------------------------------------------------------- K6 norms
constexpr int kNormBlocks = 1184;  // fixed (8 x 148): deterministic partition
cudaError_t norm_sq(const double* x, uint64_t n, double* partials, double* out, cudaStream_t s);
cudaError_t dot_dev(const double* a, const double* b, uint64_t n, double* partials, double* out,
                    cudaStream_t s);

// ---------------------------------------------------------------- K3 Z-QR
// Q0 / R0 of Z = KhatriRao(R_k, k != n) with Z's rows in the NATURAL order of
// the final Y (row-major over the other modes, ascending; the last fastest).
struct ZqrArgs {
    const double* rmats[8];  // R_k (R x R, upper), k != n, ascending mode order
    uint32_t nm;             // N - 1
    uint32_t R;
    uint64_t zrows;          // R^(N-1)
    double* q1;              // zrows x R scratch
    double* q0;              // zrows x R out
    double* r0;              // R x R out
    double* work;            // zqr_work_doubles(R, grid)
    int* status;             // device flag: non-zero = Cholesky breakdown
    unsigned long long* ts;  // optional phase timestamps (profiling)
    int pdl;                 // launch programmatically after the previous kernel
    int householder;         // rank-generic Householder kernels (widerank.cu) at any R
};
size_t zqr_work_doubles(uint32_t R);
cudaError_t launch_zqr(const ZqrArgs& a, cudaStream_t s, int sms);

// ---------------------------------------------------------------- K4 V-GEMM
// V[i][r] = sum_k Y(i,k) P[k][r] with Y(i, o*J + j) = y[(o*I + i)*J + j] and
// P = Q0 (+ beta*(Q0 - alpha*H) when extrap), optionally also Vfit with P = Q0.
struct VgemmArgs {
    const double* y;
    const double* q0;
    const double* hist;  // may be null when !extrap
    double beta, alpha;
    int extrap;
    int dual;            // also produce the unextrapolated V (fitness)
    uint64_t I, J, O;    // rows, inner, outer  (K = O*J)
    uint32_t R;
    double* vpart;       // nsplit x I x R
    double* vfitpart;    // nsplit x I x R (dual)
    double* v_out;       // I x R: final V when the kernel reduces on chip (may be null)
    double* vfit_out;    // I x R: final Vfit (dual)
    uint32_t nsplit;     // out: split count used
    int reduced;         // out: 1 = V written to v_out (no reduce_splits needed)
    uint32_t max_split;  // in: cap on the split count (0: vgemm_max_split())
    // device copy of the beta state (beta_gate); when set and extrap != 0 the
    // kernel extrapolates iff gate[0] != 0 && gate[1] != 0, with beta = gate[1]
    const double* gate;
};
// The beta state machine of run_qr (solvers.hpp:297-301) on the device, so the
// next sweep's first V-GEMM needs no host round trip.  gate = {has_beta, beta,
// has_prev, prev_fitness}; fit = the sweep's fitness (finisher output);
// allow = extrapolation on, no override, sweep >= 2.  Same arithmetic as
// cpdb_select_beta -> the host mirror takes identical decisions.
cudaError_t beta_gate(double* gate, const double* fit, int allow, double gap, cudaStream_t s);
cudaError_t launch_vgemm(VgemmArgs& a, cudaStream_t s, int sms);
uint32_t vgemm_max_split();

// ---------------------------------------------------------------- CP-ALS (als.cu)
// MTTKRP = TTM(X, A_c) + Khatri-Rao contraction of the other modes.
struct KrcArgs {
    const double* t;       // TTM output T
    const double* fac[8];  // A_k (I_k x R) of every mode
    uint64_t dims[8];
    uint32_t km[8];        // modes of the W table, ascending (not n, not c)
    uint32_t nkm;
    uint64_t rows_w;       // prod of dims[km]
    uint32_t R;
    int router;            // 0: T = [P, In, Q, R] (c = N-1); 1: T = [R, Q, In] (c = 0)
    uint64_t P, In, Q;
};
cudaError_t launch_kr_table(const KrcArgs& a, double* w, cudaStream_t s);
uint64_t krc_split(const KrcArgs& a, int sms);
// out: split x In x R partials (split == 1: M itself)
cudaError_t launch_krc(const KrcArgs& a, const double* w, double* out, uint64_t split,
                       cudaStream_t s);
// u_work: spd_work_doubles(n) doubles (n^2 up to n = 64, 2 n^2 beyond)
cudaError_t launch_spd_solve(const double* g, uint32_t n, double* u_work, double* x, uint64_t rows,
                             int* status, int* reg, cudaStream_t s, int sms);
size_t spd_work_doubles(uint32_t n);
struct GramList {
    const double* g[8];
    uint32_t n;
};
cudaError_t launch_or_flag(const int* src, int* dst, cudaStream_t s);  // *dst |= *src != 0
cudaError_t gram_dev(const double* a, uint64_t m, uint32_t n, double* g, cudaStream_t s);
cudaError_t hadamard_dev(const GramList& l, uint32_t r, double* out, cudaStream_t s);
cudaError_t launch_fitness_als(double nx2, const double* m, const double* ah, uint64_t n_mr,
                               const double* gamma, const double* lam, const double* s_last,
                               uint32_t r, double* out, cudaStream_t s);

// Per-mode tail of cp_als (solvers.hpp:177-197) as one 8-CTA cluster kernel:
// Gamma = Hadamard(G_k, k != n), solve_spd(Gamma, M) (Cholesky + ridge retry),
// normalize_columns -> A_n, lambda, G_n = gram(A_n), fitness_fast_als.
struct AlsFinishArgs {
    const double* m;           // I x R (MTTKRP)
    const double* grams[8];    // G_k, k != n (ascending)
    uint32_t ng;
    uint64_t I;
    uint32_t R;
    double* a_out;             // I x R normalised factor
    double* g_out;             // R x R Gram of a_out
    double* lambda;            // R
    int fitness;
    double norm_x_sq;
    double* fit_out;           // [fitness, raw]
    int* status;               // 4 singular after the ridge, 5 Gamma not symmetric
    int* regularized;          // set to 1 when the ridge retry was used
    unsigned long long* ts;
};
bool als_finish_fits(uint64_t I, uint32_t R);
cudaError_t launch_als_finish(const AlsFinishArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- finisher
// Per-mode tail: reduce V partials, A_hat = V R0^-T, normalise (lambda),
// CholQR2 of the factor -> Q_n, R_n, packed Q_n, and (last mode) the
// fast-QR fitness.  mode_init: factor given in `a_out`, QR only.
struct FinishArgs {
    int init;              // 1: only QR (+pack) of a_out
    const double* vpart;   // nsplit x I x R
    const double* vfitpart;
    uint32_t nsplit;
    int dual;
    const double* r0;      // R x R
    uint64_t I;
    uint32_t R;
    double* v_out;         // I x R  (V used for the fitness)
    double* a_out;         // I x R  normalised factor A_n
    double* q_out;         // I x R
    double* qp_out;        // packed Q_n for the TTM kernels
    double* r_out;         // R x R
    double* lambda;        // R
    double* scratch;       // I x (R+1) when the working matrix does not fit in smem
    int fitness;           // compute fitness
    double norm_x_sq;
    double* fit_out;       // [fitness, raw]
    int* status;           // 1 singular R0 (+col<<8), 2 Cholesky breakdown
    unsigned long long* ts;  // optional phase timestamps (profiling)
    int householder;         // rank-generic Householder kernels (widerank.cu) at any R
};
cudaError_t launch_finish(const FinishArgs& a, cudaStream_t s);
// true when launch_finish(I, R) sums FinishArgs::nsplit V partials itself
// (the cluster kernel); the single-CTA kernel needs nsplit == 1
bool finish_sums_splits(uint64_t I, uint32_t R);
// variants (cluster.cu / finish.cu): launch_finish picks the cluster kernel
// when its shared-memory plan fits, else the single-CTA one
cudaError_t launch_finish_cluster(const FinishArgs& a, cudaStream_t s);
cudaError_t launch_finish_single(const FinishArgs& a, cudaStream_t s);
size_t finish_cluster_smem(uint64_t I, uint32_t R);
bool zqr_cluster_fits(uint64_t zrows, uint32_t R, uint32_t nm);
cudaError_t launch_zqr_cluster(const ZqrArgs& a, cudaStream_t s);
cudaError_t launch_zqr_multi(const ZqrArgs& a, cudaStream_t s, int sms);
// out[e] = sum_{p < nsplit} part[p*n + e]  (fixed order)
cudaError_t reduce_splits(const double* part, uint32_t nsplit, uint64_t n, double* out,
                          cudaStream_t s);
// out[e] = sum_{r < world} slots[r*stride + e]  (fixed order; in-process rank groups)
// reduce-scatter through the in-process group's slots: this rank's chunk
// (rows [rank*chunk, (rank+1)*chunk) of every outer block) summed over ranks
cudaError_t sum_slots_scatter(const double* slots, uint64_t stride, uint32_t world,
                              uint64_t outer, uint64_t block, uint64_t chunk, uint32_t rank,
                              double* out, cudaStream_t s);
cudaError_t sum_slots(const double* slots, uint64_t stride, uint32_t world, uint64_t n,
                      double* out, cudaStream_t s);

// ---------------------------------------------------------------- wide ranks
// R > 64 (widerank.cu): the same launch interfaces served by rank-generic
// kernels (Khatri-Rao + cooperative Householder QR, row solves, exact
// normalisation) -- launch_zqr / launch_finish / launch_vgemm dispatch here.
bool wide_rank(uint32_t R);
size_t zqr_wide_work_doubles(uint32_t R);
size_t finish_wide_scratch_doubles(uint64_t I, uint32_t R);
cudaError_t launch_zqr_wide(const ZqrArgs& a, cudaStream_t s);
cudaError_t launch_finish_wide(const FinishArgs& a, cudaStream_t s);
// solve_spd for n > 64 (launch_spd_solve dispatches here); u_work: 2 n^2 doubles
cudaError_t launch_spd_solve_wide(const double* g, uint32_t n, double* u_work, double* x,
                                  uint64_t rows, int* status, int* reg, cudaStream_t s);
// thin_qr (linalg.hpp:39-99) on the cooperative kernel; work = m*n +
// zqr_wide_work_doubles(n)
cudaError_t householder_qr_wide(const double* a, uint64_t m, uint32_t n, double* work, double* q,
                                double* r, cudaStream_t s);

// ---------------------------------------------------------------- misc
// normalize_columns (linalg.hpp:225-242) with the reference's exact
// operation order (sequential column sums, no FMA contraction).
cudaError_t normalize_exact(double* a, uint64_t m, uint32_t n, double* weights, cudaStream_t s);
// Householder thin QR, reference algorithm (linalg.hpp:39-99), one CTA.
cudaError_t householder_qr(const double* a, uint64_t m, uint32_t n, double* work, double* q,
                           double* r, cudaStream_t s);
// Row-major gather: out[j] = in[perm[j]] rows of width w.
cudaError_t permute_rows(const double* in, double* out, const uint64_t* perm, uint64_t rows,
                         uint32_t w, cudaStream_t s);
// Synthetic BASELINE tensors on the device (counter-based RNG, synth.cu).
// pass1 writes the noiseless slab and scal[0..1] = (sum X^2, sum E^2) of the
// slab; sharded callers all-reduce scal before pass2 adds rho-scaled noise.
cudaError_t synth_pass1(double* x, const uint64_t* dims_host, const uint64_t* dims_dev,
                        uint32_t order, uint64_t rank, int32_t kind, uint64_t seed,
                        uint64_t row_begin, uint64_t row_count, double* factors,
                        double* partials, double* scal, cudaStream_t s);
cudaError_t synth_pass2(double* x, const uint64_t* dims_host, uint32_t order, uint64_t rank,
                        uint64_t seed, uint64_t row_begin, uint64_t row_count, const double* scal,
                        double rho, cudaStream_t s);
size_t synth_partials_doubles();
// the truth factors alone (sum I_k x R doubles, mode after mode)
cudaError_t synth_factors(double* factors, const uint64_t* dims_dev, uint32_t order,
                          uint64_t rank, int32_t kind, uint64_t seed, cudaStream_t s);

}  // namespace cpdb
