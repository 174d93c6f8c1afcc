// Host-side launchers of the libsymnmf kernels (internal; the ABI is in api.cu).
#pragma once
#include "common.cuh"

namespace symnmf {

// ---------------------------------------------------------------- gram.cu
// Grid used for a cross Gram over `rows_cap` rows (fixes the partial-buffer size).
int gram_grid(int64_t rows_cap);
size_t gram_partial_doubles(int ka, int kb, bool sym, int grid);
// out[a*ldo + b] = sum_r w_r A[g(r), a] B[g(r), b]  (a < ka, b < kb), fp64; rows r < nrows
// (or < *nrows_dev if non-null); g(r) = gather ? gather[r] : r; w_r = wts ? wts[r] : 1.
// sym => A == B and ka == kb: only the upper 4x4 blocks are computed, output mirrored.
void launch_cross_gram(const float* A, int64_t lda, int ka, const float* B, int64_t ldb, int kb, bool sym,
                       int64_t nrows, const int64_t* nrows_dev, const int32_t* gather, const double* wts,
                       double* partial, int grid, double* out, int ldo, const int32_t* status, cudaStream_t st,
                       bool fp64_products = false);
// One-CTA fp64 Cholesky G = R^T R (upper) with one jitter retry, then R^{-1}.
// Writes R^{-1} as fp32 (ld ldr32, zero padded to padk) and/or fp64 (ld ldr64).
void launch_chol_inv(const double* G, int k, float* Rinv32, int ldr32, int padk32, double* Rinv64, int ldr64,
                     int32_t* status, cudaStream_t st, double shift_rel = 0.0);

// ---------------------------------------------------------------- leverage.cu
void launch_leverage(const float* F, int64_t n, int k, const float* Rinv32, float* lev,
                     const int32_t* status, cudaStream_t st);

// ---------------------------------------------------------------- sampler.cu
constexpr int kSampBlock = 1024;  // elements per block of the sampler passes
inline int64_t samp_blocks(int64_t n) { return (n + kSampBlock - 1) / kSampBlock; }
struct SamplerWs {
  uint64_t* bw;      // [nb] block mass, then exclusive offsets
  uint32_t* bd;      // [nb] block det counts, then offsets
  double* bt;        // [nb] block theta
  uint32_t* bu;      // [nb] block unique counts, then offsets
  uint64_t* P;       // [n] inclusive prefix of w
  int32_t* cnt;      // [n] draw multiplicities (kept zero between calls)
};
// Philox stream = 2 * it + side with it = *iter_dev if iter_dev else iteration.
void launch_hybrid_sample(const float* lev, int64_t n, int k, int64_t s, double T, uint64_t seed,
                          const int32_t* iter_dev, uint32_t iteration, uint32_t side, const symnmf_plan& plan,
                          const SamplerWs& w, int32_t* status, cudaStream_t st);

// sampler passes used by the sharded sampler (shard.cu)
void launch_samp_block_sums(const float* lev, int64_t n, double T, const SamplerWs& w, int32_t* status,
                            cudaStream_t st);
void launch_samp_scan_blocks(int64_t n, int64_t s, int k, const symnmf_plan& plan, const SamplerWs& w,
                             int32_t* status, cudaStream_t st);
void launch_samp_uniq(const float* lev, int64_t n, double T, const SamplerWs& w, const symnmf_plan& plan,
                      int32_t* status, cudaStream_t st);

// ---------------------------------------------------------------- shard.cu (NEXT-4)
void launch_shard_sums(const float* lev, int64_t n, double T, const SamplerWs& w, uint64_t* W_out, int64_t* sD_out,
                       double* theta_out, int32_t* status, cudaStream_t st);
void launch_shard_plan(const float* lev, int64_t n, int64_t row0, int k, int64_t s, double T, uint64_t seed,
                       uint32_t iteration, uint32_t side, uint64_t W_off, uint64_t W_total, int64_t sD_total,
                       const symnmf_plan& plan, const SamplerWs& w, uint64_t* wloc, int32_t* status,
                       cudaStream_t st);
void launch_plan_rows_scaled(const float* F, int64_t row0, int k, const symnmf_plan& plan, float* Z,
                             const int32_t* status, cudaStream_t st);
void launch_sampled_rows_pull(const symnmf_matrix& Ab, int64_t n_total, const int32_t* uniq,
                              const int64_t* n_uniq_dev, int64_t cap, const float* Z, int k, float* Y, int32_t* slot,
                              const int32_t* status, cudaStream_t st);

// ---------------------------------------------------------------- spmm.cu / dense.cu
void launch_spmm_csr(const symnmf_matrix& A, const float* F, int k, float* Y, const int32_t* status, cudaStream_t st);
void launch_sampled_csr(const symnmf_matrix& A, const float* F, int k, const int32_t* uniq, const double* w,
                        const int64_t* n_uniq_dev, int64_t cap, float* Y, const int32_t* status, cudaStream_t st);
void launch_dense_ah_simt(const float* A, int64_t lda, int64_t n, const float* F, int64_t ldf, int k, float* Y,
                          int64_t ldy, const int32_t* status, cudaStream_t st);
void launch_sampled_dense(const float* A, int64_t lda, int64_t n, const float* F, int k, const int32_t* uniq,
                          const double* w, const int64_t* n_uniq_dev, int64_t cap, float* Y, const int32_t* status,
                          cudaStream_t st);
// tcgen05 3xTF32 dense product (tc_gemm.cu); returns false if unavailable for the shape.
bool launch_dense_ah_tc(const float* A, int64_t lda, int64_t n, const float* F, int64_t ldf, int k, float* Y,
                        int64_t ldy, void* scratch, size_t scratch_bytes, const int32_t* status, cudaStream_t st);
size_t dense_ah_tc_scratch(int64_t n, int k);
// tcgen05 3xTF32 sampled dense product (tc_sampled.cu): k <= 64, lda % 4 == n % 4 == 0, A 16-B aligned;
// scratch: sampled_dense_tc_scratch(cap, k) bytes.
bool sampled_dense_tc_enabled(int64_t n);
bool sampled_dense_tc_supported(const float* A, int64_t lda, int64_t n, int k);
size_t sampled_dense_tc_scratch(int64_t cap, int k);
void launch_sampled_dense_tc(const float* A, int64_t lda, int64_t n, const float* F, int k, const int32_t* uniq,
                             const double* w, const int64_t* n_uniq_dev, int64_t cap, int64_t u_hint, float* Y,
                             void* scratch, const int32_t* status, cudaStream_t st);

// ---------------------------------------------------------------- hals.cu
void launch_hals_sweep(const double* G, const float* Y, const float* F, float* X, int64_t n, int k, double alpha,
                       const int32_t* status, cudaStream_t st);

// ---------------------------------------------------------------- lai.cu
void launch_gaussian(int64_t n, int l, uint64_t seed, float* Omega, cudaStream_t st);
// Y[r, :kb] = sum_a X[r, a] M[a, :]  (row apply of a small ka x kb matrix M), fp32 or fp64 M.
void launch_rowapply32(const float* X, int64_t ldx, int64_t n, int ka, const float* M, int kb, float* Y, int64_t ldy,
                       const int32_t* status, cudaStream_t st);
void launch_rowapply64(const float* X, int64_t ldx, int64_t n, int ka, const double* M, int kb, float* Y,
                       int64_t ldy, const int32_t* status, cudaStream_t st);
// M32[a, b] = lambda[a] * Z[a, b] (fp64 in, fp32 out)
void launch_scale_rows(const double* Z, int l, int k, const double* lambda, float* M32, const int32_t* status,
                       cudaStream_t st);
// One-CTA Jacobi EVD of symmetric T (l x l fp64); sorts by |lambda| desc; V (ld l) fp64.
void launch_jacobi_evd(double* T, int l, double* V, double* lambda, int32_t* status, cudaStream_t st);
void launch_symmetrize(double* T, int l, cudaStream_t st);

// ---------------------------------------------------------------- fused.cu (solver hot loop)
// Gacc: zeroed kGramReplicas x k x k fp64 accumulator (left zeroed); counter: zeroed uint (left zeroed).
// Replicas of the fp64 Gram accumulators (CTA b adds into replica b % kGramReplicas; the last CTA
// sums them).  Measured (LvS it/s, 16 / 8 / 2 / 1 replicas): c2 8.05k / 8.26k / 8.34k / 8.27k,
// c1 12.54k / 12.18k / 12.21k / 12.41k; c3, c4 (LvS and EXACT) and c5 unchanged.  2 kept (the
// default bench line is c2): fewer replicas shorten the last CTA's reads more than the extra
// contention on the red.add costs.
constexpr int kGramReplicas = 2;
void launch_gram_fused(const float* F, int64_t n, int k, double* Gacc, double* Gout, float* Rinv32,
                       unsigned int* counter, int32_t* status, cudaStream_t st);
void launch_sweep_fused(const double* G, double alpha, float* Y, const float* F, float* X, int64_t n, int k,
                        bool zeroY, double* Gacc, double* Gout, float* Rinv32, unsigned int* counter,
                        int32_t* status, cudaStream_t st);
// tab >= 0 (kpad(k) == k <= 32): R through constant table tab (2 * sweep slot + side)
void launch_leverage_fused(const float* F, int64_t n, int k, const float* Rinv, float* lev, double T,
                           const SamplerWs& w, int64_t s, const symnmf_plan& plan, unsigned int* counter,
                           int32_t* status, cudaStream_t st, int tab = -1);
void launch_uniq_count_fused(const float* lev, int64_t n, double T, const SamplerWs& w, const symnmf_plan& plan,
                             const int32_t* iter_dev, int32_t first_iter, int32_t max_iters, int side,
                             symnmf_half_stats* stats, unsigned int* counter, int32_t* status, cudaStream_t st);
void launch_sampled_gram_fused(const float* F, int k, const symnmf_plan& plan, double* Gacc, double* Gout,
                               unsigned int* counter, int32_t* status, cudaStream_t st);
// sampler.cu passes used by the fused path
void launch_samp_prefix(const float* lev, int64_t n, double T, const SamplerWs& w, const symnmf_plan& plan,
                        int32_t* status, cudaStream_t st);
void launch_samp_draws(const SamplerWs& w, int64_t n, int64_t s, uint64_t seed, const int32_t* iter_dev,
                       uint32_t iteration, uint32_t side, const symnmf_plan& plan, int32_t* status, cudaStream_t st);
void launch_samp_uniq_write(const float* lev, int64_t n, double T, const SamplerWs& w, const symnmf_plan& plan,
                            int32_t* status, cudaStream_t st);
// sampled CSR scatter into a Y the caller has zeroed
// Scatter pass boundaries per row of A (once per A; (passes - 1) x n int32, see spmm.cu).
int sampled_csr_passes(int64_t n, int k);
void launch_sampled_pass_bounds(const symnmf_matrix& A, int k, int32_t* ppos, cudaStream_t st);
void launch_sampled_csr_nozero(const symnmf_matrix& A, const float* F, int k, const int32_t* uniq, const double* w,
                               const int64_t* n_uniq_dev, int64_t cap, float* Y, const int32_t* status,
                               cudaStream_t st, const int32_t* ppos = nullptr);

// ---------------------------------------------------------------- spmm_nnz.cu
// Exact CSR product balanced by nonzeros (k in {8,16,32,64}); chunk_row from launch_spmm_nnz_rows
// (once per A), carry: spmm_nnz_carry_floats floats.
int64_t spmm_nnz_chunks(int64_t nnz);
size_t spmm_nnz_carry_floats(int64_t nnz, int k);
bool spmm_nnz_supported(int k);
void launch_spmm_nnz_rows(const symnmf_matrix& A, int64_t* chunk_row, cudaStream_t st);
void launch_spmm_nnz(const symnmf_matrix& A, const int64_t* chunk_row, const float* F, int k, float* Y, float* carry,
                     const int32_t* status, cudaStream_t st);
// *bad = 1 if a row's column indices are not sorted, unique and in [0, n) (caller zeroes *bad).
void launch_csr_check(const symnmf_matrix& A, int32_t* bad, cudaStream_t st);

// ---------------------------------------------------------------- sweep.cu
// Streaming HALS sweep (k in {8, 16, 32}): cp.async-staged tiles, thread per row, fused Gram + Cholesky.
// tab >= 0: G through constant table tab = 2 * slot + side (slot from sweep_cslot_acquire), built in
// `scratch` (sweep_table_floats() floats); tab < 0: G in shared memory.
bool sweep_stream_supported(int k);
void launch_sweep_stream(const double* G, double alpha, float* Y, const float* F, float* X, int64_t n, int k,
                         bool zeroY, double* Gacc, double* Gout, float* Rf32, unsigned int* counter, int32_t* status,
                         cudaStream_t st, int tab = -1, float* scratch = nullptr, bool yalpha = false);
// Y = alpha F (count floats, count % 4 == 0)
void launch_scale_copy(const float* F, double alpha, float* Y, int64_t count, cudaStream_t st);
int sweep_cslot_acquire();
void sweep_cslot_release(int slot);
size_t sweep_table_floats();

// ---------------------------------------------------------------- bpp.cu (NEXT-1)
// X <- exact per-row NLS with (G + alpha I, Y + alpha F) (block principal pivoting, k <= 32);
// zeroY re-zeroes Y after reading; *nonconv counts rows that hit the pivoting-step cap.
bool bpp_supported(int k);
void launch_bpp(const double* G, float* Y, const float* F, float* X, int64_t n, int k, double alpha, bool zeroY,
                int32_t* nonconv, int32_t* status, cudaStream_t st);

// ---------------------------------------------------------------- lai_fused.cu
int lai_lp(int l);
bool lai_fused_supported(int k, int l);
void launch_lai_sweep_fused(const float* U, int l, int64_t n, int k, const float* Mcur, const double* G, double alpha,
                            const float* F, float* X, const double* lam, double* GXacc, double* UXacc, double* Gout,
                            float* Mnext, unsigned int* counter, int32_t* status, cudaStream_t st);

// ---------------------------------------------------------------- residual.cu
void launch_residual(const symnmf_matrix& A, const float* H, int k, const float* AH, const double* G,
                     double* partial, int grid, double* out, const int32_t* status, cudaStream_t st);
int residual_grid(int64_t n);
// NEXT-3 projected gradient: out[0] = ||P grad||_F, out[1] = ||grad||_F, grad = 4 (H G - AH), G = H^T H.
void launch_pgrad(const float* H, const float* AH, const double* G, int64_t n, int k, double* partial, int grid,
                  double* out, const int32_t* status, cudaStream_t st);
int pgrad_grid(int64_t n);
// out[0] = sum of squares (fp64) of a rows x cols block (leading dimension ld); partial: sumsq_grid() doubles.
void launch_sumsq(const float* X, int64_t rows, int64_t cols, int64_t ld, double* partial, double* out,
                  const int32_t* status, cudaStream_t st);
int sumsq_grid();

}  // namespace symnmf
