/* fastkf_b200.h — C ABI of the B200-native fast Kalman filter hot path (sm_100a).
 *
 * Drop-in boundary for the reference's header-only C++ API in
 * /root/reference/proj/include/fastkf (namespace fastkf).  The reference has no FFI;
 * each entry point below names the reference function it replaces (file:line).
 * The C++ shim include/fastkf_b200.hpp restores the reference's class/function
 * names and exception types on top of this ABI.
 *
 * Conventions:
 *  - status codes: 0 ok, 1 invalid argument (std::invalid_argument),
 *    2 runtime error (std::runtime_error), 3 CUDA error; fkb_last_error() has the text.
 *  - dense blocks are column-major FP64 with explicit leading dimensions (Eigen MatrixXd);
 *    fields are flat x-major vectors, index ix*ny + iy (grid.hpp:48).
 *  - CSR: int32 rowptr/col, FP64 values (SparseRowMatrix, grid.hpp:15).
 *  - one CUDA stream per covariance operator; calls on one operator/filter are
 *    serialized; host-buffer calls are synchronous; *_device calls take device pointers
 *    and are stream-ordered.
 */
#ifndef FASTKF_B200_H
#define FASTKF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FKB_OK 0
#define FKB_INVALID_ARGUMENT 1
#define FKB_RUNTIME_ERROR 2
#define FKB_CUDA_ERROR 3
#define FKB_DOMAIN_ERROR 4 /* std::domain_error (Box-Cox maps, boxcox.hpp:58-75) */

typedef struct fkb_cov fkb_cov;
typedef struct fkb_filter fkb_filter;
typedef struct fkb_ekf fkb_ekf;
typedef struct fkb_enkf fkb_enkf;
typedef struct fkb_ghep fkb_ghep;

const char* fkb_last_error(void);
unsigned long long fkb_launch_count(void); /* kernels launched by this library so far */
int fkb_version(void);
int fkb_device_count(void); /* CUDA devices visible (0 on a CPU-only host) */

/* ---- host-side setup (no GPU needed) ------------------------------------------ */
/* kernel_eval, kernel.hpp:51-63 (family 0 powered-exponential, 1 Matérn) */
int fkb_kernel_eval(int family, double theta, double length, double power, double nu, double alpha_scale, double r,
                    double* out);
/* detail::next_smooth, covariance.hpp:35-43 */
int fkb_next_smooth(int n);
/* trace_ray, tomography.hpp:29-86: segments in traversal order; *count = total segments */
int fkb_trace_ray(int nx, int ny, double lx, double ly, double sx, double sy, double rx, double ry, int cap,
                  long long* cells, double* lengths, int* count);
/* build_H, tomography.hpp:130-146 (rows source-major, columns ascending).  Call with
 * cap = 0 to query *nnz; rowptr needs n_src*n_rec+1 entries. */
int fkb_build_H(int nx, int ny, double lx, double ly, int n_src, const double* src_xy, int n_rec,
                const double* rec_xy, int* rows, long long* nnz, int* rowptr, int* col, double* val, long long cap);
/* small symmetric eigensolver used by the GHEP (stand-in for SelfAdjointEigenSolver,
 * lowrank.hpp:193): ascending eigenvalues w, eigenvectors Z (n×n column-major) */
int fkb_sym_eig(int n, const double* A, double* w, double* Z);
/* the same on the GPU (two-sided block Jacobi, eig.cu; ascending eigenvalues); *sweeps may be null */
int fkb_sym_eig_device(int n, const double* A, double* w, double* Z, int* sweeps);
/* the same by GPU Householder tridiagonalization + QL (rotations applied on the GPU):
 * w ascending, Z column-major (the GHEP and add_low_rank core eigensolves, lowrank.hpp:193, :265) */
int fkb_sym_eig_tridiag(int n, const double* A, double* w, double* Z);

/* ---- covariance operator Γ (CovarianceOperator FFT mode, covariance.hpp:69-353) ---- */
/* constructor covariance.hpp:71-79 + build_fft :238-260 (padding loop, acceptance) */
int fkb_cov_create(int nx, int ny, double lx, double ly, int family, double theta, double length, double power,
                   double nu, double alpha_scale, fkb_cov** out);
void fkb_cov_destroy(fkb_cov* c);
int fkb_cov_dims(const fkb_cov* c, int* mx, int* my);
/* spectrum(), covariance.hpp:207-211: mx*my row-major, clipped at 0 */
int fkb_cov_spectrum(fkb_cov* c, double* out);
/* apply_matrix, covariance.hpp:111-115 (host buffers; Y may equal X) */
int fkb_cov_apply(fkb_cov* c, const double* X, long long ldx, int ncols, double* Y, long long ldy);
int fkb_cov_apply_device(fkb_cov* c, const double* dX, long long ldx, int ncols, double* dY, long long ldy);
/* sample_pair, covariance.hpp:190-197,332-353 (host outputs, length nx*ny each) */
int fkb_cov_sample_pair(fkb_cov* c, uint64_t seed, uint64_t stream, double* a, double* b);
long long fkb_cov_apply_count(const fkb_cov* c); /* apply_count(), covariance.hpp:213 */
void* fkb_cov_stream(fkb_cov* c);                 /* the operator's cudaStream_t */

/* gaussian_matrix, rng.hpp:79-86, generated on the device (host output, column-major) */
int fkb_gaussian_matrix(long long rows, int cols, uint64_t seed, uint64_t base_stream, double* out);

/* ---- constant-H fast filter (FkfContext + LowRankState, fast_filter.hpp:21-125) ---- */
/* fkf_init, fast_filter.hpp:51-75: GHEP (lowrank.hpp:141-213, two-pass) with
 * a_apply = HᵀH/σ², G = HΓHᵀ, B = HU; the state starts at zero_start (:30-36). */
int fkb_fkf_init(fkb_cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val, double sigma2,
                 long long k_rank, long long p_oversample, uint64_t seed, fkb_filter** out);
void fkb_filter_destroy(fkb_filter* f);
int fkb_filter_rank(const fkb_filter* f, int* rank, int* kept_cols);
int fkb_filter_lambda(fkb_filter* f, double* out); /* GepResult::lambda, descending */
/* ghep_residual, lowrank.hpp:215-228: per pair ‖A u − λ Γ⁻¹u‖ / max(λ‖Γ⁻¹u‖, ε) with
 * A = HᵀH/σ², Γ⁻¹u taken from the GHEP's Ū = Γ⁻¹U (exact; the reference solves by CG) */
int fkb_filter_ghep_residual(fkb_filter* f, double* out);
/* which: 0 U (N×r), 1 Ū = Γ⁻¹U (N×r), 2 G = HΓHᵀ (m×m), 3 B = HU (m×r), 4 ‖U_j‖² (r) — host copies */
int fkb_filter_get(fkb_filter* f, int which, double* out);
/* fkf_step, fast_filter.hpp:84-125, advancing the device-resident state */
int fkb_fkf_step(fkb_filter* f, const double* y, long long ylen);
/* one step from host y AND the new state (α, d (r), mean (N)) in one round trip — the reference's
 * fkf_step returns the new LowRankState by value (fast_filter.hpp:84-125); d/mean may be null */
int fkb_fkf_step_state(fkb_filter* f, const double* y, long long ylen, double* alpha, double* d, double* mean);
/* nsteps fkf_steps over host observations (row t at ys + t·ldy) with every step's new state
 * returned: alphas[t], d row t (ld ldd ≥ r), mean row t (ld ldm ≥ N) — the driver's step loop
 * (driver.hpp:283-300) as one call; each step's outputs leave the GPU while the next step runs
 * (page-locked host arrays overlap best).  Outputs may be null.  A singular step raises (status
 * 2) naming it; the steps before it are committed and their outputs valid. */
int fkb_fkf_run(fkb_filter* f, const double* ys, int nsteps, long long ldy, double* alphas, double* d, long long ldd,
                double* mean, long long ldm);
/* the same with each new state's diag Σ (var row t, N) and `count` ≤ 8 FFT-mode realizations
 * (x: N×count block per step at x + t·N·count) from the fused U pass (uq.hpp:16-23, 86-112) */
int fkb_fkf_run_uq(fkb_filter* f, const double* ys, int nsteps, long long ldy, uint64_t seed, int count, double* x,
                   double* var, double* alphas, double* d, long long ldd, double* mean, long long ldm);
int fkb_fkf_step_device(fkb_filter* f, const double* d_y);
/* one step plus the UQ of the new state — diag Σ (var, N) and `count` ≤ 8 conditional
 * realizations (x, N×count; RealizationPropagator draws (seed, s/2), uq.hpp:86-112) — from ONE
 * pass over U fused with the mean update (the reference's fkf_step + variance +
 * RealizationPropagator::at calls, driver.hpp:292-300); host buffers, any output may be null */
int fkb_fkf_step_uq(fkb_filter* f, const double* y, long long ylen, uint64_t seed, int count, double* x, double* var,
                    double* alpha, double* d, double* mean);
/* device buffers, enqueued without a host sync like fkb_fkf_steps_async (fkb_fkf_sync checks and commits) */
int fkb_fkf_step_uq_device(fkb_filter* f, const double* d_y, uint64_t seed, int count, double* d_x, double* d_var);
/* nsteps device-resident observations (column k at d_ys + k*ldy) without host syncs;
 * fkb_fkf_sync performs the deferred singularity check and commits the state. */
int fkb_fkf_steps_async(fkb_filter* f, const double* d_ys, int nsteps, long long ldy);
int fkb_fkf_sync(fkb_filter* f, int nsteps);
/* LowRankState download / upload (d has `rank` entries, mean N) */
int fkb_filter_state(fkb_filter* f, double* alpha, int* step, int* rank, double* d, double* mean);
int fkb_filter_set_state(fkb_filter* f, double alpha, int step, int rank, const double* d, const double* mean);
int fkb_filter_reset(fkb_filter* f);
/* read-only view of the device mean: the steps carry H*mean = y - sigma2*z beside it (fast_filter.hpp:108
 * without the SpMV), so a new mean must go through fkb_filter_set_state */
int fkb_filter_mean_device(fkb_filter* f, const double** d_mean);

/* ---- UQ (uq.hpp:16-112) ---------------------------------------------------------- */
int fkb_variance(fkb_filter* f, double* out);              /* variance, uq.hpp:16-23 */
int fkb_variance_device(fkb_filter* f, double* d_out);
int fkb_trace_criterion(fkb_filter* f, double* out);       /* uq.hpp:27-34 */
int fkb_relative_entropy(fkb_filter* f, double* out);      /* uq.hpp:39-53 */
/* conditional realizations in FFT mode (uq.hpp:70-112 with the circulant root, SURVEY
 * App. A.4): draw s uses sample_pair(seed, s/2), Re for even s, Im for odd; count ≤ 8.
 * out: N×count column-major; var (optional) receives diag Σ from the same pass. */
int fkb_realizations(fkb_filter* f, uint64_t seed, int count, double* out);
int fkb_realizations_device(fkb_filter* f, uint64_t seed, int count, double* d_out, double* d_var);
/* host buffers, one pass over U for both: out (N×count, may be null when count = 0) and var
 * (diag Σ, may be null) */
int fkb_realizations_with_variance(fkb_filter* f, uint64_t seed, int count, double* out, double* var);
/* RealizationPropagator::at / conditional_sample (uq.hpp:68-112) for draw `draw` alone:
 * sample_pair(seed, draw/2), Re for even draw, Im for odd, on the filter's current state */
int fkb_realization_at(fkb_filter* f, uint64_t seed, uint64_t draw, double* out);
/* variance (uq.hpp:16-23) and the column norms ‖W_j‖² that trace_criterion needs (:27-34) for a
 * state with an explicit W (e.g. read_state, field_io.hpp:115-135): Σ = αΓ − W·diag(d)·Wᵀ,
 * W host N×r column-major (ld ≥ N); var (N) and colsq (r) may be null.  Computed on the GPU. */
int fkb_lowrank_uq(fkb_cov* c, long long n, int r, double alpha, const double* d, const double* w, long long ldw,
                   double* var, double* colsq);

/* The GHEP's W-block products on the DMMA path (device pointers, column-major, on `stream`):
 * which 0 — Gram C (p×q) = AᵀB, A n×p, B n×q (Ȳᵀ(ΓȲ), lowrank.hpp:53-106 block form);
 * which 1 — C (n×q) = A (n×p)·B (p×q) (U = Q·S, Ū = Q̄·S, lowrank.hpp:197-205);
 * which 2 — symmetric Gram C (p×p) = AᵀA, both triangles (the per-step capacitance kernel
 *           k_gram_sym, fast_filter.hpp:100-108 in Woodbury form; q must equal p, B unused). */
int fkb_dense_product(int which, long long n, int p, int q, const double* dA, const double* dB, double* dC,
                      void* stream);

/* ---- standalone randomized GHEP (lowrank.hpp:132-213 with A = HᵀH/σ², the a_apply of
 * fast_filter.hpp:63-66; the generic-LinOp overload is served for this operator only) ---- */
int fkb_ghep_run(fkb_cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val, double sigma2,
                 long long k, long long p, uint64_t seed, fkb_ghep** out);
void fkb_ghep_destroy(fkb_ghep* g);
int fkb_ghep_info(const fkb_ghep* g, int* rank, int* kept_cols);
/* which: 0 λ (rank, descending), 1 U (N×rank, Γ⁻¹-orthonormal), 2 Ū = Γ⁻¹U (N×rank) */
int fkb_ghep_get(fkb_ghep* g, int which, double* out);

/* ---- extended fast filter (fekf_step, fast_filter.hpp:127-224) --------------------- */
/* Binds Γ and the ray operator H (the reference passes both to every fekf_step call,
 * :142-144; all its callers keep them fixed, driver.hpp:305-333,555-580) and starts from
 * LowRankState::zero_start with mean = 0.  The state (α, step, mean, W, d) and W̄ = Γ⁻¹W
 * stay on the device. */
int fkb_ekf_create(fkb_cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val,
                   fkb_ekf** out);
void fkb_ekf_destroy(fkb_ekf* e);
/* zero_start with the given initial mean (driver.hpp:315-316: mean = forward(init_slowness)) */
int fkb_ekf_reset(fkb_ekf* e, const double* mean0);
/* fekf_step with FekfOptions {k_rank (−1 = m), oversampling, trunc_tol, relinearizations,
 * seed} (:127-134) and BoxCox{boxcox_alpha} (boxcox.hpp:14-17) */
int fkb_ekf_step(fkb_ekf* e, const double* y, long long ylen, double sigma2, double boxcox_alpha, long long k_rank,
                 long long oversampling, double trunc_tol, int relinearizations, uint64_t seed);
/* state sizes: α, step count, rank r = W.cols() */
int fkb_ekf_state(fkb_ekf* e, double* alpha, int* step, int* rank);
/* host copies of mean (N), d (r), W (N×r column-major) and W̄ = Γ⁻¹W (N×r); any may be null */
int fkb_ekf_read(fkb_ekf* e, double* mean, double* d, double* w, double* wbar);
/* trace_criterion (uq.hpp:25-34) and relative_entropy (uq.hpp:36-53) of the extended state */
int fkb_ekf_uq(fkb_ekf* e, double* trace, double* entropy);
/* diag Σ (var, N) and `count` ≤ 8 realizations (out, N×count; draws first_draw… as
 * fkb_realization_at) of the extended state, in the transformed (Box–Cox) space; either may be null */
int fkb_ekf_realizations(fkb_ekf* e, uint64_t seed, uint64_t first_draw, int count, double* out, double* var);
/* diagnostics of the last step: GHEP rank and relinearization sweeps run */
int fkb_ekf_last(fkb_ekf* e, int* gep_rank, int* sweeps);

/* ---- ensemble Kalman filter (enkf.hpp:15-94) ---------------------------------------- */
/* enkf_init (:30-34: n_members ≥ 2, all members zero) bound to Γ and H; members stay on the
 * device (n×n_members column-major). */
int fkb_enkf_init(fkb_cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val,
                  int n_members, fkb_enkf** out);
void fkb_enkf_destroy(fkb_enkf* e);
/* enkf_step (:49-94): forecast draws (seed, 1), perturbations (seed, 2) */
int fkb_enkf_step(fkb_enkf* e, const double* y, long long ylen, double sigma2, uint64_t seed);
/* Ensemble::members download / upload (n×n_members column-major), Ensemble::mean (:20) */
int fkb_enkf_members(fkb_enkf* e, double* out);
int fkb_enkf_set_members(fkb_enkf* e, const double* in);
int fkb_enkf_mean(fkb_enkf* e, double* out);

/* ---- kernels exposed for parity tests / benchmarks (device pointers) ------------- */
/* Y = H X (trans = 0) or Hᵀ X (trans = 1) with the filter's uploaded operator */
int fkb_filter_spmm(fkb_filter* f, int trans, const double* dX, long long ldx, int ncols, double* dY,
                    long long ldy);
/* same products on ROW-major blocks (X: cols × ncols, Y: rows × ncols, row stride ncols) */
int fkb_filter_spmm_rm(fkb_filter* f, int trans, const double* dX, int ncols, double* dY);
void* fkb_filter_stream(fkb_filter* f);
int fkb_filter_launches_per_step(fkb_filter* f);
/* innovation solve: 1 (default) Woodbury in the offline eigenbasis of G = HΓHᵀ with a
 * k×k capacitance factorization; 0 the reference order (form S, m×m LLT) */
int fkb_filter_set_solver(fkb_filter* f, int mode);
int fkb_filter_eig_sweeps(fkb_filter* f);
/* last step's capacitance solve: PCG iterations and whether the exact Cholesky fallback ran */
int fkb_filter_cap_stats(fkb_filter* f, int* iterations, int* fallback);
/* PCG iteration cap (default 200); 0 forces the exact cluster-Cholesky path (tests) */
int fkb_filter_set_pcg_maxit(fkb_filter* f, int maxit);
/* profiling aid: 64 %globaltimer stamps of the last PCG launch (needs FKB_PCG_STAMPS=1) */
int fkb_filter_pcg_stamps(fkb_filter* f, unsigned long long* out);
/* eigenpairs of G (θ unsorted, P m×m column-major) */
int fkb_filter_get_eig(fkb_filter* f, double* theta, double* P);
/* runs `reps` real steps un-graphed with CUDA events at phase boundaries; ms[i] = mean
 * duration of phase i, names = comma-separated phase names (advances the state) */
int fkb_filter_phase_times(fkb_filter* f, int reps, double* ms, char* names, int names_len, int* nphases);
/* in-graph kernel timing: on != 0 re-captures the step graph with timing events at every
 * phase boundary; graph_phase_times then returns the per-phase device ms of the LAST replay */
int fkb_filter_graph_timing(fkb_filter* f, int on);
int fkb_filter_graph_phase_times(fkb_filter* f, double* ms, char* names, int names_len, int* nphases);

/* capacitance factor+solve kernel on a host SPD matrix (test/profiling hook): L lower
 * factor, x = K⁻¹b; stamps (optional, 128 entries) receive %globaltimer phase stamps */
int fkb_chol_solve_small(int n, const double* K, const double* b, double* L, double* x,
                         unsigned long long* stamps);
/* capacitance Jacobi-PCG kernel on a host SPD matrix (test/profiling hook): x = K⁻¹b,
 * *iters = iterations; returns 2 if the iteration cap was hit; stamps: 64 entries */
int fkb_cap_pcg_test(int n, const double* K, const double* b, double* x, int* iters,
                     unsigned long long* stamps);

/* measured FP64 peak of this GPU (mode 0: DFMA pipe, 1: DMMA tensor path), TFLOP/s */
int fkb_fp64_peak(int mode, double* tflops);
/* measured L2→SM read bandwidth (GB/s) over an L2-resident buffer of mbytes MB */
int fkb_l2_peak(int mbytes, double* gbs);
int fkb_set_device(int device);  /* cudaSetDevice for this library's runtime */
int fkb_profiler(int on);        /* cudaProfilerStart/Stop (ncu --profile-from-start off) */

/* device memory helpers (so bindings need no CUDA runtime of their own) */
int fkb_dmalloc(void** p, size_t bytes);
int fkb_dfree(void* p);
int fkb_h2d(void* dst, const void* src, size_t bytes);
int fkb_d2h(void* dst, const void* src, size_t bytes);
int fkb_dsync(void);

#ifdef __cplusplus
}
#endif

#endif /* FASTKF_B200_H */
