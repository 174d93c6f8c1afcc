/*
 * symnmf.h -- C ABI of the B200 (sm_100a) hot path of randomized SymNMF
 *             (Hayashi, Aggarwal, Kannan, Ballard, "Randomized Algorithms for
 *              Symmetric Nonnegative Matrix Factorization", arXiv 2402.08134).
 *
 * Citations: P:<n> = line n of the paper's LaTeX source; Z<n> =
 * reading n of the ambiguity ledger in DESIGN.md.
 *
 * Conventions (all functions):
 *  - Matrices are row-major (C order).  Every float/double/int pointer in an
 *    argument list is a CUDA DEVICE pointer unless its name ends in `_host`.
 *  - The caller owns every buffer, including the workspace `ws`.  The library
 *    never allocates device memory and keeps no global mutable state; calls
 *    on different streams with different workspaces are independent.
 *  - Workspace query: call with ws == NULL; *ws_bytes receives the size,
 *    nothing is enqueued, SYMNMF_OK is returned.  A later call whose
 *    *ws_bytes is smaller returns SYMNMF_ERR_WORKSPACE.  The workspace must be
 *    256-byte aligned.  Its first 256 bytes hold a device status word (see
 *    symnmf_status_read) that kernels set on device-side failure; kernels
 *    downstream of a failure become no-ops.
 *  - Asynchrony: every function except symnmf_iterate, symnmf_solve,
 *    symnmf_rangefinder_adaptive (its stopping test reads residuals on the host),
 *    symnmf_bpp_update with nonconv_host != NULL, symnmf_solver_create / _stats /
 *    _run_until / _pgrad / _profile / _graph_nodes / _destroy and symnmf_status_read
 *    only enqueues work on `st` (no host sync) and is CUDA-graph capturable
 *    (tests/test_gpu_api_contract.py captures the per-half ABI sequence).
 *  - Errors never cross the ABI as exceptions; every entry point returns a
 *    symnmf_status.  SYMNMF_ERR_ARG is returned synchronously, before any work
 *    is enqueued, for null pointers, n < 1, k < 1 or k > 64, s < 1,
 *    tau outside (0, 1], alpha < 0, l > n or l > 96, a CSR/3XTF32 mismatch.
 *  - Floating point: inputs fp32; Grams, theta/xi, sampling weights and
 *    residual reductions fp64 (Z27).  No fast-math.
 */
#ifndef SYMNMF_H_
#define SYMNMF_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SYMNMF_OK = 0,
  SYMNMF_ERR_ARG = 1,          /* invalid argument (synchronous)                         */
  SYMNMF_ERR_NOT_PD = 2,       /* Cholesky of a k x k / l x l Gram failed after 1 jitter  */
  SYMNMF_ERR_WORKSPACE = 3,    /* *ws_bytes smaller than required                        */
  SYMNMF_ERR_CUDA = 4,         /* CUDA launch / runtime error                            */
  SYMNMF_ERR_UNSUPPORTED = 5,  /* device is not sm_100 or mode not built                 */
  SYMNMF_ERR_CAPACITY = 6      /* plan capacity smaller than s_D or |U| (device side)    */
} symnmf_status;

enum { SYMNMF_DENSE = 0, SYMNMF_CSR = 1 };        /* symnmf_matrix.kind              */
enum { SYMNMF_FP32 = 0, SYMNMF_3XTF32 = 1 };      /* precision of a dense product     */
enum { SYMNMF_EXACT = 0, SYMNMF_LVS = 1, SYMNMF_LAI = 2 };  /* symnmf_iterate mode     */
/* OR-ed into a mode: Update() by exact per-row NLS with block principal pivoting (ANLS-BPP,
 * P:155, App. G) instead of one HALS sweep (NEXT-1; k <= 64, else SYMNMF_ERR_UNSUPPORTED). */
enum { SYMNMF_RULE_BPP = 16 };
/* Solver mode flag (LvS): keep the scores and plan of every half in device memory for
 * symnmf_solver_plan_history (costs ~20 n bytes per half; for parity tests, not for timing). */
enum { SYMNMF_RECORD_PLANS = 32 };

/* Symmetric n x n input A (Eq. 2.2).  The caller guarantees
 * A = A^T.  DENSE: val is n x lda fp32 (lda >= n, lda % 4 == 0 for 3XTF32).
 * CSR: both triangles stored ("row/column slicing ... because the
 * matrix is symmetric"), rowptr int64 [n+1], colidx int32 [nnz] sorted and
 * unique within a row, val fp32 [nnz]; empty rows are allowed, and nnz = 0 (A = 0, colidx
 * and val may be NULL). */
typedef struct {
  int32_t kind;
  int32_t reserved;
  int64_t n;
  const float* val;
  int64_t lda;
  const int64_t* rowptr;
  const int32_t* colidx;
  int64_t nnz;
} symnmf_matrix;

/* Device-resident hybrid sampling plan S_H = diag(S_D, S_R) (Eq. 4.1-4.2,
 * P:722-741), written by symnmf_hybrid_sample and read by symnmf_sampled_ah.
 *   det_idx  int32 [cap]  I_D = {i : l_i >= tau k} in increasing order (Z1)
 *   draw_idx int32 [s]    the s_R i.i.d. draws in draw order (Z4, Z6)
 *   uniq_idx int32 [cap]  U = I_D u {drawn rows}, increasing
 *   uniq_w   fp64  [cap]  omega_i: 1 on I_D, c_i * (W / (s_R * w_i)) on drawn rows (Z5)
 *   counts   int64 [4]    s_D, s_R, |U|, W (integer mass of I_R, Z3)
 *   mass     fp64  [2]    theta = sum_{I_D} l_i, xi = k - theta
 * cap >= min(n, s) is required; SYMNMF_ERR_CAPACITY is raised on device if
 * s_D or |U| exceeds cap (possible only for tau < 1/s, Z2). */
typedef struct {
  int64_t cap;
  int32_t* det_idx;
  int32_t* draw_idx;
  int32_t* uniq_idx;
  double* uniq_w;
  int64_t* counts;
  double* mass;
} symnmf_plan;

/* Per half-iteration statistics recorded by the solver (E7). */
typedef struct {
  int64_t s_d;
  int64_t s_r;
  int64_t n_uniq;
  double theta;
} symnmf_half_stats;

/* Tuning knobs read from the environment when a call is enqueued (host only; results are
 * the same up to fp32 summation order):
 *   SYMNMF_CSR_SPMM=rows|nnz       EXACT solver on CSR: the row-group SpMM or (k in {8,16,32,64})
 *                                  the nnz-balanced one (chunks of 256 nonzeros); default: nnz-
 *                                  balanced from 16M nonzeros.
 *   SYMNMF_SWEEP=fused|stream      k in {8,16,32}: the register-tile sweep or the streaming
 *                                  (cp.async-staged, two CTAs/SM) sweep; default: streaming from
 *                                  2^20 rows.
 *   SYMNMF_SWEEP_CMEM=0            streaming sweep and leverage scores: G / R from shared memory
 *                                  instead of the constant bank (a solver holds one of 4 constant
 *                                  slots; beyond 4 live solvers the shared-memory form is used).
 *   SYMNMF_SCATTER_SLICE_MB=<mb>   sampled CSR scatter product: rows of Y per destination-range
 *                                  pass, so each pass's slice of Y stays in L2 (default 48 MB when the
 *                                  passes are merged into one launch, k in {16,32,64}; else 86 MB).
 *   SYMNMF_SCATTER_SPLIT=<w>       sampled CSR scatter product: warps per sampled row and pass (each
 *                                  takes a contiguous part of the row's in-range nonzeros; default 2
 *                                  with merged passes, else 4).
 *   SYMNMF_SCATTER_SHFL=0          sampled CSR scatter product (k in {16,32,64}): every lane group loads
 *                                  its own entries (broadcast loads) instead of the warp loading 32
 *                                  consecutive entries once, a batch ahead, and shuffling them.
 *   SYMNMF_SCATTER_MERGE=0         sampled CSR scatter product: one launch per destination-range pass instead
 *                                  of one launch whose block range p works on pass p.
 *   SYMNMF_PDL=0|1                 programmatic dependent launch between the kernels of a call / of the
 *                                  solver's graph: forced off / on (default: on only in solver graphs
 *                                  below 2^15 rows).
 *   SYMNMF_YALPHA=0                LvS on CSR with the streaming sweep: re-zero Y for each scatter and
 *                                  read F in the sweep, instead of the scatter accumulating onto
 *                                  Y = alpha F left by the previous sweep (state kept across runs).
 *   SYMNMF_SAMPLED_DENSE=simt|tc   sampled dense product: the fp32 SIMT kernel, or the tcgen05 3xTF32
 *                                  one (k <= 64, n % 4 == lda % 4 == 0); default: tcgen05 from n = 16384.
 *   SYMNMF_LAI_FUSED=never         LAI solver (k = 64, l <= 80): use the four-kernel half (U^T F,
 *                                  Lambda scaling, U M, sweep) instead of the fused launch.
 * CSR inputs: every row's column indices must be sorted, unique and in [0, n) (both triangles
 * stored); symnmf_solver_create checks this on the device and returns SYMNMF_ERR_ARG otherwise. */

/* Library version (major*10000 + minor*100 + patch).  Host only. */
int32_t symnmf_version(void);

/* Sync `st`, then copy the device status word of `ws` to *status_host. */
symnmf_status symnmf_status_read(const void* ws, int32_t* status_host, cudaStream_t st);

/* (a1) G = F^T F ("G_H := H^T H").  F n x k fp32,
 * G k x k fp64 (exactly symmetric).  fp32 products, per-tile fp32 partial
 * sums flushed to fp64, fixed-order (deterministic) fp64 combine. */
symnmf_status symnmf_gram(const float* F, int64_t n, int32_t k, double* G,
                          void* ws, size_t* ws_bytes, cudaStream_t st);

/* (a10) Y = A F ("the product XH"), F and Y n x k fp32.
 * DENSE: precision SYMNMF_FP32 (SIMT fp32, chunked accumulation) or
 * SYMNMF_3XTF32 (tcgen05 tensor cores, split a = a_hi + a_lo).  CSR: fp32
 * SpMM; precision must be SYMNMF_FP32. */
symnmf_status symnmf_ah(const symnmf_matrix* A, const float* F, int32_t k, float* Y,
                        int32_t precision, void* ws, size_t* ws_bytes, cudaStream_t st);

/* (a1-a3) Leverage scores l_i = f_i (F^T F)^{-1} f_i^T (Eq. 2.10 P:280-286,
 * Alg. LvS-SymNMF) by CholeskyQR: fp64 Gram,
 * fp64 Cholesky F^T F = R^T R (one jitter retry of 1e-12 tr(G)/k, then
 * SYMNMF_ERR_NOT_PD on the device status word), l_i = ||f_i R^{-1}||^2.
 * lev fp32 [n]; G_out (nullable) receives F^T F. */
symnmf_status symnmf_leverage_scores(const float* F, int64_t n, int32_t k, float* lev,
                                     double* G_out, void* ws, size_t* ws_bytes, cudaStream_t st);

/* (a4-a7) Hybrid deterministic + random leverage-score sampling plan
 * (Eq. 2.11).  I_D = {i : (double)lev_i >= tau*k} (Z1),
 * s_R = max(0, s - s_D) (Z2; 0 if the remaining mass is 0), integer mass
 * w_i = floor(lev_i 2^40) on I_R and its inclusive prefix P (Z3, Z6), draw j
 * = first i with P_i > floor(u_j W / 2^64), u_j from Philox4x32-10 with
 * counter (j, 0, 2*iteration + side, 0) and key (seed lo, seed hi) (Z6).
 * Bit-exact given lev and (seed, iteration, side). */
symnmf_status symnmf_hybrid_sample(const float* lev, int64_t n, int32_t k, int64_t s, double tau,
                                   uint64_t seed, uint32_t iteration, uint32_t side,
                                   const symnmf_plan* plan, void* ws, size_t* ws_bytes, cudaStream_t st);

/* (a8, a9) Sampled products of Alg. LvS-SymNMF:
 * Y_s = (S A)^T (S F) = sum_{i in U} omega_i A[i,:]^T f_i   (n x k fp32, Z28)
 * G_s = F^T S^T S F  = sum_{i in U} omega_i f_i^T f_i      (k x k fp64, nullable)
 * The alpha terms are not sampled. */
symnmf_status symnmf_sampled_ah(const symnmf_matrix* A, const float* F, int32_t k,
                                const symnmf_plan* plan, float* Y, double* G_s,
                                void* ws, size_t* ws_bytes, cudaStream_t st);

/* (a12) Alg. RRF + Alg. Apx-EVD on dense symmetric A:
 * Omega n x l Gaussian (Philox counter (e/2, 0, 0, 1), Box-Muller, Z18),
 * Y = A Omega, Q = orth(Y); q times {Q = orth(A Q); Q = orth(A Q)} (Z16),
 * T = sym(Q^T A Q), T = V Lambda V^T (Jacobi, fp64), U = Q V, ordered by
 * |lambda| descending (Z17).  orth = CholeskyQR2 with fp64 Gram/Cholesky.
 * U n x l fp32, lambda fp64 [l].  2q + 2 applications of A. */
symnmf_status symnmf_rangefinder(const symnmf_matrix* A, int32_t l, int32_t q, uint64_t seed,
                                 int32_t precision, float* U, double* lambda,
                                 void* ws, size_t* ws_bytes, cudaStream_t st);

/* (a12) The Gaussian test matrix Omega alone (n x l fp32), for parity tests. */
symnmf_status symnmf_gaussian(int64_t n, int32_t l, uint64_t seed, float* Omega, cudaStream_t st);

/* (a13) LAI product Y = U (Lambda (U^T F)), U n x l fp32,
 * lambda fp64 [l], F and Y n x k fp32. */
symnmf_status symnmf_lai_ah(const float* U, const double* lambda, int64_t n, int32_t l,
                            const float* F, int32_t k, float* Y,
                            void* ws, size_t* ws_bytes, cudaStream_t st);

/* (a11) One efficient symmetric HALS sweep (Eq. 2.6, App. G
 * P:1649-1653) of Update(G + alpha I, Y + alpha F^T):
 * for every row r, for i = 0..k-1 in order (Gauss-Seidel, Z9)
 *   X[r,i] <- max(0, (Y[r,i] + alpha F[r,i] - sum_{j != i} X[r,j] G[j,i]) / (G[i,i] + alpha))
 * (a column with G[i,i] + alpha == 0 is left unchanged).  G fp64 k x k
 * WITHOUT alpha I; Y, F, X n x k fp32; X updated in place.  G_new
 * (nullable) receives X^T X of the updated X (the next half's Gram). */
symnmf_status symnmf_hals_sweep(const double* G, const float* Y, const float* F, float* X,
                                int64_t n, int32_t k, double alpha, double* G_new,
                                void* ws, size_t* ws_bytes, cudaStream_t st);

/* NEXT-1 Update by block principal pivoting (App. G; Kim & Park full exchange
 * with the backup rule): X[r,:] = argmin_{x >= 0} x^T (G + alpha I) x - 2 (Y[r,:] + alpha F[r,:])^T x
 * for every row r, fp64 solves (G fp64 k x k, Y F X n x k fp32, k <= 64); X is overwritten
 * (its entry value is not used).  G_new (nullable)
 * receives X^T X.  nonconv_host (nullable; host-synchronising) receives the number of rows that
 * hit the 256-step pivoting cap (their last iterate, clipped at 0, is written). */
symnmf_status symnmf_bpp_update(const double* G, const float* Y, const float* F, float* X, int64_t n, int32_t k,
                                double alpha, double* G_new, int32_t* nonconv_host, void* ws, size_t* ws_bytes,
                                cudaStream_t st);

/* (a15) Normalised residual ||A - H H^T||_F / ||A||_F in fp64 (P:101-103,
 * P:1530-1532).  DENSE: direct sum of (A_ij - h_i.h_j)^2; CSR: the trace
 * identity ||A||^2 - 2 tr(H^T A H) + ||H^T H||^2.
 * out fp64 device [4] = {residual, ||A||_F^2, tr(H^T A H), ||H^T H||_F^2}. */
symnmf_status symnmf_residual(const symnmf_matrix* A, const float* H, int32_t k, double* out,
                              void* ws, size_t* ws_bytes, cudaStream_t st);

/* NEXT-2 Alg. Ada-RRF (App. E) + Apx-EVD on dense symmetric A: Q = qr(A Omega);
 * then per pass j = 1, 2, ...: B^T = A Q, residual ||A - Q B||_F / ||A||_F from the trick
 * ||A||^2 - ||B||^2 (fp64), Q = qr(B^T); stop when j = q_max or the residual
 * decreased by no more than `tol` since the previous pass (tol = 1e-3; reading Z31),
 * else Y = A Q, Q = qr(Y).  Then T = sym(Q^T A Q) = V Lambda V^T, U = Q V (as
 * symnmf_rangefinder).  Host-synchronising (one 8-byte read-back per pass).  passes_host
 * receives the number of passes, resid_host (nullable, q_max entries) the residual per pass. */
symnmf_status symnmf_rangefinder_adaptive(const symnmf_matrix* A, int32_t l, int32_t q_max, double tol, uint64_t seed,
                                          int32_t precision, float* U, double* lambda, int32_t* passes_host,
                                          double* resid_host, void* ws, size_t* ws_bytes, cudaStream_t st);

/* NEXT-3 projected gradient of the SymNMF objective f(H) = ||A - H H^T||_F^2 (App. D,
 * P:1560-1590): grad = 4 (H (H^T H) - A H), entries kept where grad < 0 or
 * H > 0 (the KKT mask).  A H uses `precision` as in symnmf_ah (CSR: FP32);
 * H^T H and the norms are fp64.  out fp64 device [2] = {||P grad||_F, ||grad||_F}. */
symnmf_status symnmf_projected_gradient(const symnmf_matrix* A, const float* H, int32_t k, int32_t precision,
                                        double* out, void* ws, size_t* ws_bytes, cudaStream_t st);

/* (a14) Iteration driver of Alg. LvS-SymNMF, LAI-SymNMF
 * or exact HALS: per iteration t the W-half (side 0, F = H) then
 * the H-half (side 1, F = W) (Z11-Z13); iteration index first_iter + t keys
 * the sampler so a resumed run is bit-reproducible.  W, H n x k fp32 in/out.
 *   EXACT: G = F^T F, Y = A F (precision as in symnmf_ah)
 *   LVS  : scores of F, hybrid plan (s, tau, seed), G_s, Y_s
 *   LAI  : G = F^T F, Y = U (Lambda (U^T F)) (U, lambda, l from symnmf_rangefinder; A may be NULL
 *          unless resid_host is given)
 * then X <- sweep(G, Y, F, X, alpha).  The per-iteration body is captured
 * once as a CUDA graph and replayed.  stats_host (nullable, 2*iters
 * entries) receives the per-half plan statistics (LVS); resid_host
 * (nullable, iters entries) receives ||A - H H^T||/||A|| after every
 * iteration (one extra exact product per iteration).  Synchronises `st` and
 * returns the device status. */
symnmf_status symnmf_iterate(const symnmf_matrix* A, int64_t n, float* W, float* H, int32_t k, double alpha,
                             int32_t mode, int32_t precision, int64_t s, double tau, uint64_t seed,
                             int32_t first_iter, int32_t iters,
                             const float* U, const double* lambda, int32_t l,
                             symnmf_half_stats* stats_host, double* resid_host,
                             void* ws, size_t* ws_bytes, cudaStream_t st);

/* Reusable solver handle (caller-owned state; the library still holds no
 * global state): symnmf_solver_create captures the iteration graph once,
 * symnmf_solver_run enqueues `iters` iterations without a host sync (the
 * device iteration counter continues from the previous run), and
 * symnmf_solver_stats syncs and copies the recorded statistics.  The
 * arguments have the meaning of symnmf_iterate's; `max_iters` bounds the
 * total number of iterations whose statistics are recorded. */
typedef struct symnmf_solver symnmf_solver;
symnmf_status symnmf_solver_create(symnmf_solver** out, const symnmf_matrix* A, int64_t n, float* W, float* H,
                                   int32_t k, double alpha, int32_t mode, int32_t precision, int64_t s,
                                   double tau, uint64_t seed, int32_t first_iter, int32_t max_iters,
                                   const float* U, const double* lambda, int32_t l, int32_t with_residual,
                                   void* ws, size_t* ws_bytes, cudaStream_t st);
symnmf_status symnmf_solver_run(symnmf_solver* solver, int32_t iters, cudaStream_t st);
symnmf_status symnmf_solver_stats(symnmf_solver* solver, int32_t* iters_done_host,
                                  symnmf_half_stats* stats_host, double* resid_host, cudaStream_t st);
symnmf_status symnmf_solver_destroy(symnmf_solver* solver);
/* NEXT-3 convergence protocol (solver created with with_residual = 1, else SYMNMF_ERR_ARG):
 * runs iterations one at a time, reading back the normalised residual after each (8 bytes,
 * one stream synchronisation), and stops once it has failed to decrease by more than `tol`
 * for `patience` consecutive iterations (tol = 1e-4, patience = 4; reading Z30), or
 * after max_iters iterations, or when max_iters recorded slots are used up.
 * *iters_run_host receives the number of iterations run. */
symnmf_status symnmf_solver_run_until(symnmf_solver* solver, int32_t max_iters, double tol, int32_t patience,
                                      int32_t* iters_run_host, cudaStream_t st);
/* NEXT-2/3 driver (host-synchronising): iterations of `mode` (arguments as symnmf_iterate) until
 * the stopping rule of P:1086 (tol, patience; see symnmf_solver_run_until) or max_iters; with
 * refine = 1 (Iterative Refinement, P:557-563, P:1088 -- meant for mode = LAI) it then continues
 * with EXACT iterations on the full A from the factors reached, under the same rule.
 * iters_host (nullable) [2] = iterations of each phase; resid_host (nullable, 2 * max_iters) =
 * the residual after every iteration of phase 0 then phase 1.  One workspace serves both phases. */
symnmf_status symnmf_solve(const symnmf_matrix* A, int64_t n, float* W, float* H, int32_t k, double alpha,
                           int32_t mode, int32_t precision, int64_t s, double tau, uint64_t seed,
                           const float* U, const double* lambda, int32_t l, int32_t max_iters, double tol,
                           int32_t patience, int32_t refine, int32_t* iters_host, double* resid_host,
                           void* ws, size_t* ws_bytes, cudaStream_t st);
/* Per-iteration projected-gradient norms ||P grad f(H)||_F of the recorded iterations (solver
 * created with with_residual = 1); syncs `st`. */
symnmf_status symnmf_solver_pgrad(symnmf_solver* solver, double* pgrad_host, cudaStream_t st);
/* Per-kernel device timing (host only, synchronising): runs `iters` iterations EAGERLY (not
 * from the graph; W and H advance exactly as with symnmf_solver_run) with a CUDA event after
 * every launch site, and returns for each site of one iteration (in launch order) its name
 * (names_host[i], NUL terminated) and mean duration in ms (ms_host[i]); *count_host <= cap. */
symnmf_status symnmf_solver_profile(symnmf_solver* solver, int32_t iters, int32_t cap, char (*names_host)[48],
                                    float* ms_host, int32_t* count_host, cudaStream_t st);
/* Inspection (LvS solvers only; enqueued on `st`, no host sync): copies the sampling state the
 * solver left after the last half it ran -- the leverage scores of the factor that half held fixed
 * (lev_out: n floats) and its plan (uniq_idx_out: n int32, uniq_w_out: n doubles, of which the
 * first counts_out[2] are valid; counts_out: 4 int64 {s_D, s_R, n_uniq, W}; mass_out: 2 doubles
 * {theta, xi}) -- into caller-owned device buffers.  The fused sampler does not materialise
 * det_idx / draw_idx.  Returns SYMNMF_ERR_ARG for a non-LvS solver or a null pointer. */
symnmf_status symnmf_solver_last_plan(const symnmf_solver* solver, float* lev_out, int32_t* uniq_idx_out,
                                      double* uniq_w_out, int64_t* counts_out, double* mass_out, cudaStream_t st);
/* LvS solver created with SYMNMF_RECORD_PLANS: copy the scores and plan the solver drew in half
 * `side` of iteration first_iter + t (same outputs as symnmf_solver_last_plan).  Returns
 * SYMNMF_ERR_ARG if plans were not recorded or (t, side) has not run. */
symnmf_status symnmf_solver_plan_history(const symnmf_solver* solver, int32_t t, int32_t side, float* lev_out,
                                         int32_t* uniq_idx_out, double* uniq_w_out, int64_t* counts_out,
                                         double* mass_out, cudaStream_t st);
/* ---------------------------------------------------------------- NEXT-4 row sharding
 * Building blocks of the row-sharded solver (driver: paper_2402_08134_b200/shard.py).
 * A shard owns the row block [row0, row0 + n) of A (CSR rows, global column indices), W and H.
 * The collectives between the calls (allreduce of k x k Grams, allgather of the shards' masses and
 * plan rows) are the caller's.  All pointers are device pointers unless stated; enqueue only. */

/* lev = scores of the rows of F (n x k block) given G = F_all^T F_all of the whole factor (fp64
 * k x k): l_i = f_i G^{-1} f_i^T by CholeskyQR.  SYMNMF_ERR_NOT_PD on the status word. */
symnmf_status symnmf_leverage_scores_gram(const float* F, int64_t n, int32_t k, const double* G, float* lev,
                                          void* ws, size_t* ws_bytes, cudaStream_t st);
/* The block's share of the sampler totals (readings Z1-Z6): *W_out = sum floor(l 2^40)
 * over its rows outside I_D (uint64, exact), *sD_out = |I_D ∩ block|, *theta_out = sum_{I_D} l. */
symnmf_status symnmf_hybrid_shard_sums(const float* lev, int64_t n, int32_t k, double tau, uint64_t* W_out,
                                       int64_t* sD_out, double* theta_out, void* ws, size_t* ws_bytes,
                                       cudaStream_t st);
/* The block's part of the global plan, given (host values) the exclusive prefix W_offset of the
 * shards' masses before this one, the global W_total and sD_total: its I_D rows and the global
 * draws j < s_R = s - sD_total whose target mulhi(u_j, W_total) falls in [W_offset, W_offset + W_b),
 * weights omega = c W_total / (s_R w) (the same IEEE operations as symnmf_hybrid_sample).
 * plan->uniq_idx holds global row ids; counts = {s_D of the block, s_R, n_uniq of the block, W_total};
 * det_idx holds block-local rows; draw_idx is not written.  The shards' uniq_idx / uniq_w
 * concatenated in row order equal symnmf_hybrid_sample's on the whole score vector, bit for bit. */
symnmf_status symnmf_hybrid_shard_plan(const float* lev, int64_t n, int64_t row0, int32_t k, int64_t s, double tau,
                                       uint64_t seed, uint32_t iteration, uint32_t side, uint64_t W_offset,
                                       uint64_t W_total, int64_t sD_total, const symnmf_plan* plan, void* ws,
                                       size_t* ws_bytes, cudaStream_t st);
/* Z[t] = omega_t f_{u_t} (fp32, n_uniq x k) for the block's plan rows (F = the block's rows, u_t
 * global), and (G_s nullable) the block's share of the sampled Gram sum_t omega_t f_t^T f_t (fp64). */
symnmf_status symnmf_plan_rows_scaled(const float* F, int64_t row0, int32_t k, const symnmf_plan* plan, float* Z,
                                      double* G_s, void* ws, size_t* ws_bytes, cudaStream_t st);
/* Rows of the sampled product for the block as a pull: Y[c] = sum_{i in U} a_ci Z[slot(i)]
 * over the block's CSR rows (a_ci = a_ic by symmetry), U = uniq[0 .. *n_uniq_dev) global row
 * ids of the whole plan, Z their scaled rows in plan order (n_uniq x k); Y is the block's n x k. */
symnmf_status symnmf_sampled_ah_rows(const symnmf_matrix* A_block, int64_t n_total, const int32_t* uniq,
                                     const int64_t* n_uniq_dev, int64_t cap, const float* Z, int32_t k, float* Y,
                                     void* ws, size_t* ws_bytes, cudaStream_t st);
/* LAI on row blocks (Eq. 3.1: A ~ U Lambda U^T, so A F ~ U (Lambda (U^T F))).  The l x k
 * projection U^T F is a sum over rows: each shard forms its block's share
 *   Z_b = U_b^T F_b   (fp64, l x k row-major; U_b, F_b = the block's n rows of U and F),
 * the caller allreduces the shares into Z, and symnmf_lai_apply_rows writes the block's rows
 *   Y_b = U_b (Lambda Z)   (fp32 n x k; lambda = the l eigenvalues, fp64).
 * With one block the two calls compose to symnmf_lai_ah.  1 <= l <= 80, k as everywhere. */
symnmf_status symnmf_lai_project_rows(const float* U, int64_t n, int32_t l, const float* F, int32_t k, double* Z,
                                      void* ws, size_t* ws_bytes, cudaStream_t st);
symnmf_status symnmf_lai_apply_rows(const float* U, const double* lambda, int64_t n, int32_t l, const double* Z,
                                    int32_t k, float* Y, void* ws, size_t* ws_bytes, cudaStream_t st);

/* Kernel and memset node counts of the captured per-iteration graph (host only). */
symnmf_status symnmf_solver_graph_nodes(const symnmf_solver* solver, int32_t* kernels_host, int32_t* memsets_host);

#ifdef __cplusplus
}
#endif
#endif /* SYMNMF_H_ */
