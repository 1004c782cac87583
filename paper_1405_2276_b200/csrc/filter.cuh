// filter.cuh — the constant-H fast filter on the device (fkf_init / fkf_step / UQ).
#pragma once
#include <cstdlib>

#include <deque>
#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "cov.cuh"
#include "dense.cuh"
#include "sparse.cuh"

namespace fkb {

// randomized_ghep (lowrank.hpp:132-213) with A = HᵀH/σ² and B = Γ on the device; U is
// Γ⁻¹-orthonormal (N×r, column-major) and Ū = Γ⁻¹U comes with it.
struct GepDev {
    int r = 0, kept_cols = 0;
    std::vector<double> lambda_h;
    DBuf<double> lambda, U, Ubar;
    // device temporaries, kept across calls (the extended filter runs a GHEP every step)
    std::deque<DBuf<double>> scratch;  // deque: growing keeps references to earlier slots valid
    DBuf<double>& tmp(size_t slot, size_t count) {
        if (scratch.size() <= slot) scratch.resize(slot + 1);
        scratch[slot].ensure(std::max<size_t>(count, 1));
        return scratch[slot];
    }
};
void randomized_ghep_device(Cov* cov, const DevCsr& H, const DevCsr& HT, double sigma2, long long k, long long p,
                            uint64_t seed, DBuf<double>& ws, cudaStream_t s, GepDev& out);
// G = H·Γ·Hᵀ (m×m, ld m), symmetrized
// (scratch: a persistent N×batch workspace for repeated calls; else a temporary)
void build_hgh(Cov* cov, const DevCsr& H, double* G, cudaStream_t s, DBuf<double>* scratch = nullptr);
void symmetrize(int n, double* A, long long lda, cudaStream_t s);
// out[j] = ‖A[:, j]‖² for the n×r column-major A
void column_sumsq(long long n, int r, const double* A, double* out, cudaStream_t s);
// out (r×n column-major, i.e. row-major n×r) = in (n×r column-major)ᵀ
void transpose_cm(long long n, int r, const double* in, double* out, cudaStream_t s);
// shared helpers (filter.cu)
void check_nonneg_args(long long k, long long p, long long n);
std::vector<double> download(const double* p, size_t count, cudaStream_t s);
void upload(double* p, const std::vector<double>& h, cudaStream_t s);
void gram_tn(long long n, int p, int q, const double* A, const double* B, double* C, DBuf<double>& ws,
             cudaStream_t s);
void tall_times_small(long long n, int p, int q, const double* A, const double* W, double* C, cudaStream_t s);
std::vector<double> gram_inv_sqrt(int p, const std::vector<double>& Gh, double tol, int& kept);

// diag Σ, ‖W_j‖² and realizations of Σ = αΓ − W·diag(d)·Wᵀ (device buffers, filter.cu)
void lowrank_uq(Cov* cov, long long n, int r, const double* alpha_dev, const double* d, const double* W,
                const double* Wbar, const double* mean, uint64_t seed, uint64_t first, int count, double* X,
                double* var, double* colsq, DBuf<double>& scratch);

struct EpiCtzD;
struct Filter {
    EpiCtzD commit_epi();
    Cov* cov = nullptr;
    cudaStream_t s = nullptr;
    long long n = 0;
    int m = 0;
    double sigma2 = 0.0;
    DevCsr H, HT;

    // offline products (FkfContext, fast_filter.hpp:42-49); ΓHᵀ is not stored — the step
    // applies Γ to Hᵀz instead (same product)
    int r = 0;          // GEP rank
    int kept_cols = 0;  // columns surviving Γ-orthonormalization
    std::vector<double> lambda_h;
    DBuf<double> lambda, U, Ubar, G, B, colsq;
    DBuf<double> Urow;  // U row-major (N×r): the per-step U-pass streams it linearly

    // LowRankState (fast_filter.hpp:21-37), device resident; W ≡ U
    double alpha = 0.0;
    int step_no = 0;
    int state_rank = 0;
    DBuf<double> alpha_dev, d, mean;

    // Woodbury form of the innovation solve (solver = 1, default): G = P·diag(θ)·Pᵀ and
    // E = PᵀB precomputed once, so S(α,d)⁻¹ = P·[Λ_M − E·D·Eᵀ]⁻¹·Pᵀ with Λ_M = αθ + σ²
    // needs only the k×k capacitance K = I − D^½EᵀΛ_M⁻¹ED^½ per step.
    // solver = 0 reproduces the reference order: form S and LLT it (m×m) every step.
    int solver = 1;
    int eig_sweeps = 0;
    DBuf<double> P, Pt, theta, E, Erow, rt, ucap, st, rdg, pcgwork;
    DBuf<double> dsnap;  // committed d at the start of the step (read by the next-K side branch)
    // Per-step Woodbury scalars Λ_M⁻¹ (wsq), D^½ (sqd) and capacitance K, double-buffered by
    // step parity: step t reads buffer t&1 while its side branch forms step t+1's into the
    // other (they depend only on α and d, not on the observation).
    DBuf<double> wsqb[2], sqdb[2], Kb[2];
    double *wsq_c = nullptr, *sqd_c = nullptr, *K_c = nullptr;  // this step's (capture-time)
    double *wsq_n = nullptr, *sqd_n = nullptr, *K_n = nullptr;  // next step's
    int par_next = 0;  // parity of the next step to run
    DBuf<int> certb[2];          // K's positive-definiteness certificate per parity (k_cap_certificate)
    DBuf<double> Kchk, bchk, rdg2;  // the side branch's Cholesky certificate of a K Gershgorin cannot certify
    DBuf<int> cgate;             // [gate, info] of that factorization
    const int* cert_c = nullptr;  // this step's
    bool cert_force_fail = false; // FKB_CAP_CERT=fail: every step takes the exact path (tests)
    // Per-parity snapshots of what a step's N-space mean side needs once its m-space chain
    // has committed — z = S⁻¹(y − H·mean), dc = d ⊙ Bᵀz, the step's α, the new d (fused UQ)
    // and the commit gate — so step t's mean side can run beside step t+1's chain.
    DBuf<double> zb[2], cvb[2], dq[2], alphaq;
    DBuf<int> gateq;
    double *z_c = nullptr, *cv_c = nullptr, *dq_c = nullptr, *aq_c = nullptr;
    int* gate_c = nullptr;
    // the image hm = H·mean carried by the steps (k_step_prologue / EpiZHm), the step's
    // observation, the prologue's last-CTA ticket
    DBuf<double> hm, ycur;
    DBuf<unsigned> ticket;
    bool hm_valid = false;
    void prime_image();
    void select_parity(int p) {
        z_c = zb[p].p; cv_c = cvb[p].p; dq_c = dq[p].p; aq_c = alphaq.p + p; gate_c = gateq.p + p;
        hout_c = hostout.p + 5 * p;
        cert_c = certb[p].p;
        wsq_c = wsqb[p].p; sqd_c = sqdb[p].p; K_c = Kb[p].p;
        wsq_n = wsqb[p ^ 1].p; sqd_n = sqdb[p ^ 1].p; K_n = Kb[p ^ 1].p;
    }
    DBuf<unsigned long long> pcg_ts;  // %globaltimer stamps of the PCG kernel (FKB_PCG_STAMPS=1)
    DBuf<int> pcgflag;
    int pcg_maxit = 200;  // iteration cap before the exact Cholesky takes over (tests force 0)  // 1 when the capacitance PCG fell back to the cluster Cholesky

    // step workspaces (vsub = U·dc from the side-branch U pass)
    DBuf<double> S, t, vsub, ws, ws_step, potrf_ws;
    int upass_per_sm = 1;     // resident U-pass CTAs per SM beside the main chain (FKB_UPASS_CTAS);
                              // negative: a total CTA count (FKB_UPASS_GRID)
    int upass_threads = 256;  // threads per U-pass CTA (FKB_UPASS_THREADS: 128 or 256)
    int kfork = 1;            // where the next-K side branch forks (FKB_KFORK, enqueue_solve_woodbury)
    int ufork = 1;            // where the U pass forks (FKB_UFORK)
    bool fuse_rhs = false;    // capacitance RHS formed inside the PCG kernel (FKB_FUSE_RHS; measured slower)
    // fused chain (FKB_FUSED_CHAIN, default on): rotate_in → PCG (+ s̃ and the d/α commit) →
    // rotate_out; exact = the eager rerun of a step whose PCG did not verify (kInfoRetry)
    int fused_chain = 1;  // 0: unfused; 1: Woodbury tail in the PCG cluster; 2: k_woodbury_st PDL-launched after it
    bool exact = false;
    int pdl_mask = 0;  // FKB_PDL: 1 rotate_in after the residual, 2 rotate_out after k_woodbury_st_pdl
    DBuf<double> parts;  // rotate_in's per-CTA partials of Eᵀ(Λ_M⁻¹r̃), coldot_grid(m) × r
    void rerun_exact(int parity);
    // the device observations of the last asynchronous batch (rerun of a failed step)
    const double* batch_ys = nullptr;
    long long batch_ldy = 0;
    int batch_par0 = 0;
    template <class XL>
    void launch_u_pass(XL xl, cudaStream_t st, bool beside);
    void fork_upass();
    // the U pass runs beside the main chain (side branch) when it is short enough to hide
    // there: rank ≤ 320 (c2); otherwise after the forward FFT passes on the whole GPU (c4).
    // The fused step + UQ (c3) keeps its single pass k_mean_uq after Γ(Hᵀz).  FKB_UPASS_SIDE
    // = 0/1 forces either placement of the plain pass.
    int upass_side_mode = -1;
    bool upass_side() const { return upass_side_mode >= 0 ? upass_side_mode == 1 : (uq_count < 0 && r <= 320); }
    DBuf<int> info, flags;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};  // one per step parity
    // Pipelined batch variants per parity q of the step whose chain runs: [0] head — chain(q)
    // only; [1] steady — chain(q) beside the mean side of step q^1; [2] flush — the mean side
    // of step q alone (after the batch's last chain).
    cudaGraphExec_t graphv[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
    int launches_v[3] = {0, 0, 0};
    bool piped_ok = false;       // FKB_PIPED=1: batches overlap step t's mean side with step t+1's chain
    bool chain_deferred = false; // enqueue_chain: the mean side (and its U pass) is launched elsewhere
    cudaStream_t s4 = nullptr;   // the deferred mean side's stream
    cudaEvent_t ev_mfork = nullptr, ev_mjoin = nullptr;
    struct MeanSide {
        const double* z = nullptr;       // S⁻¹(y − H·mean)
        const double* cv = nullptr;      // d ⊙ Bᵀz
        const double* alpha1 = nullptr;  // alpha1[1] = the step's α
        const int* gate = nullptr;       // ≠ 0: the step did not commit
        const double* d = nullptr;       // the new d (fused UQ)
        const double* sqd = nullptr;
        const unsigned long long* hout = nullptr;
    };
    void enqueue_chain(const double* d_y, bool deferred, const std::function<void()>& after_prologue = {});
    cudaStream_t hs = nullptr;   // the stream of the chain's head (prologue, rotate_in): s, or s5 in early-PCG graphs
    cudaStream_t s5 = nullptr;
    cudaEvent_t ev_rfork = nullptr, ev_rjoin = nullptr;
    bool early_pcg = true;       // FKB_EARLY_PCG=0: pipelined graphs keep the PCG behind rotate_in
    DBuf<double> ready;          // epoch of the last complete set of rotate_in partials (PcgRhs::ready)
    int sm_count = 0, upass_leave = 0;
    void enqueue_mean_side(const MeanSide& ms, cudaStream_t sm, bool deferred);
    MeanSide snapshot_side(int q);
    bool piped() const { return piped_ok && solver == 1 && r > 0 && !phase_events && !gtime; }
    void launch_piped(int variant, int q);  // replay (capturing on first use) the variant for parity q
    void run_piped(int t);       // step t of a pipelined batch: head (t = 0) or steady graph
    bool graph_ready[2] = {false, false};
    void drop_graphs();
    // side stream for the independent branches of a step (captured into the same graph):
    // fork() makes it wait for the main stream, join() makes the main stream wait for it.
    // Phase timing runs the branches serially on the main stream.
    cudaStream_t s2 = nullptr;
    cudaStream_t s3 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr, ev_ctz = nullptr;
    cudaStream_t side() const { return phase_events ? s : s2; }
    void fork();
    void join(cudaEvent_t ev);
    // The capacitance K = I − D^½EᵀΛ_M⁻¹ED^½ depends only on α and d, so each step computes
    // the NEXT step's K on the side branch as soon as d and α are updated (overlapping the
    // Γ(Hᵀz) and U passes); k_valid says Kcap/wsq/sqd hold it.  Invalidated by reset,
    // set_state and set_solver; prime_capacitance() recomputes it eagerly when needed.
    bool k_valid = false;
    // mode 0: K for α_dev[0]+1 and the committed d (priming); mode 1: K for the step after the
    // one being enqueued (α_dev[1]+1 and d updated from α_dev[1]), written to the next buffers
    void enqueue_capacitance(cudaStream_t b, int mode, double* wsq_o, double* sqd_o, double* K_o);
    void prime_capacitance();
    int launches_per_step = 0;

    // cached realization draws (RealizationPropagator, uq.hpp:86-112)
    uint64_t draw_seed = 0;
    int draw_count = 0;
    DBuf<double> draws, draw_proj;  // N×count, r×count (Ūᵀz)
    void prepare_draws(uint64_t seed, int count);
    // fused step + UQ (c3-style workloads): −1 = plain step graphs; 0..8 = the captured step's U
    // pass also writes diag Σ (uq_var) and uq_count realizations (uq_x) of the new state
    int uq_count = -1;
    DBuf<double> uq_x, uq_var;
    void set_step_uq(bool on, uint64_t seed = 0, int count = 0);
    void step_uq(const double* d_y, uint64_t seed, int count, double* d_x, double* d_var);
    DBuf<double> sig_minus;

    DBuf<double> ybuf;
    // the step's observation source (k_step_prologue): {base, ld, row}; per-call mode {ybuf, 0, ·},
    // host batch {uploaded block, m, row advanced by the step's last kernel}
    DBuf<long long> ysrc;
    DBuf<double> ys_dev;
    void set_ysrc(const double* base, long long ld);
    long long* h_ysrc = nullptr;  // page-locked staging of the two ysrc configurations
    DBuf<double> host_out;  // staging for the host-buffer UQ calls

    Filter(Cov* cov, int m, int h_cols, const int* rowptr, const int* col, const double* val, double sigma2,
           long long k, long long p, uint64_t seed);
    ~Filter();
    void ghep(long long k, long long p, uint64_t seed);  // lowrank.hpp:141-213
    void step(const double* d_y);                        // fast_filter.hpp:84-125 (device y)
    void step_host(const double* h_y);                   // same, y from host memory
    void step_host_state(const double* h_y, double* h_d, double* h_mean);  // + new state, one sync
    int* h_info = nullptr;                               // pinned failure-flag staging
    // mapped host outputs of the step graph: [0] mean, [1] d, [2] failure flag (0 = none)
    DBuf<unsigned long long> hostout;
    // [3] realizations, [4] diag Σ of the fused step + UQ
    unsigned long long hostout_cache[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const unsigned long long* hout_c = nullptr;  // the slots of the parity being enqueued
    void set_hostout_all(const unsigned long long (&want)[10]);
    // pipelined host batch (run_host): per-parity device snapshots of the outputs, a copy stream
    DBuf<double> snap_mean[2], snap_d[2], snap_x[2], snap_v[2];
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_done[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
    void run_host(const double* h_ys, int nsteps, long long ldy, double* h_alpha, double* h_d, long long ldd,
                  double* h_mean, long long ldm, int count = -1, uint64_t seed = 0, double* h_x = nullptr,
                  double* h_var = nullptr);
    unsigned long long* h_hostout = nullptr;
    void set_hostout(unsigned long long hm, unsigned long long hd, unsigned long long hi, unsigned long long hx = 0,
                     unsigned long long hv = 0);
    void step_uq_host(const double* h_y, uint64_t seed, int count, double* h_x, double* h_var, double* h_d,
                      double* h_mean);
    // k steps over device-resident observations (column k at d_ys + k·ldy), no host sync;
    // finish_async() performs the deferred singularity check and commits host mirrors.
    void steps_async(const double* d_ys, int nsteps, long long ldy);
    void finish_async(int nsteps);
    void enqueue_step(const double* d_y);                // kernels only, no host sync
    void enqueue_solve_dense();                          // z ← S⁻¹z, reference order (solver 0)
    void enqueue_solve_woodbury();                       // z ← S⁻¹z via G's eigenbasis (solver 1)
    void set_solver(int mode);
    // Un-graphed steps with CUDA events at phase boundaries: average ms per phase.
    std::vector<std::pair<std::string, double>> phase_times(int reps);
    std::vector<cudaEvent_t>* phase_events = nullptr;
    std::vector<std::string> phase_names;
    void mark(const char* name) { mark_on(s, name); }
    void mark_on(cudaStream_t st, const char* name);
    // In-graph kernel timing: with gtime set, the captured step graph records external timing
    // events at every phase boundary (on the phase's own stream), so per-kernel device times
    // come from real graph replays (bench.py's roofline) rather than from un-graphed steps.
    bool gtime = false, capturing = false;
    int gt_last_par = 0;  // parity of the last replayed graph
    std::vector<cudaEvent_t> gt_ev[2];
    std::vector<std::string> gt_name[2];
    std::vector<int> gt_prev[2];
    std::vector<std::pair<cudaStream_t, int>> gt_last;
    void set_graph_timing(bool on);
    std::vector<std::pair<std::string, double>> graph_phase_times();
    void launch_step();                                  // graph replay of enqueue_step(ybuf)
    void check_info();                                   // throws on a singular innovation system
    [[noreturn]] void fail_step(const std::string& msg); // clears the sticky flag, throws
    void reset();                                        // zero_start (:30-36)
    void variance(double* d_out);                        // uq.hpp:16-23
    std::vector<double> ghep_residual();                 // lowrank.hpp:215-228 with Γ⁻¹U = Ū
    double trace_criterion();                            // uq.hpp:27-34
    double relative_entropy();                           // uq.hpp:39-53
    void realizations(uint64_t seed, int count, double* d_out, double* d_var);
    // draw `draw` alone (RealizationPropagator(cov, seed, draw).at(state), uq.hpp:86-112)
    void realization_at(uint64_t seed, uint64_t draw, double* d_out);
    DBuf<double> uq_scratch;
    std::vector<double> d_host() const;
};

}  // namespace fkb
