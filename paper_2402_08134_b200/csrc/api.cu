// The C ABI of libsymnmf (include/symnmf.h): argument validation, workspace
// carving, kernel sequencing, and the CUDA-graph iteration driver.
#include <cstdio>
#include <new>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include "kernels.cuh"

using namespace symnmf;

namespace {

bool device_ok() {
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return false;
  return major == 10;
}

bool bad_k(int k) { return k < 1 || k > kMaxK; }

bool bad_matrix(const symnmf_matrix* A) {
  if (!A || A->n < 1) return true;
  if (A->kind == SYMNMF_DENSE) return !A->val || A->lda < A->n;
  if (A->kind == SYMNMF_CSR) return !A->rowptr || A->nnz < 0 || (A->nnz > 0 && (!A->colidx || !A->val));
  return true;
}

// Workspace protocol: query (ws == NULL) or check size/alignment.
symnmf_status ws_protocol(void* ws, size_t* ws_bytes, size_t need, bool* query) {
  *query = false;
  if (!ws_bytes) return SYMNMF_ERR_ARG;
  if (!ws) { *ws_bytes = need; *query = true; return SYMNMF_OK; }
  if (*ws_bytes < need) return SYMNMF_ERR_WORKSPACE;
  if (reinterpret_cast<uintptr_t>(ws) % 256) return SYMNMF_ERR_ARG;
  return SYMNMF_OK;
}

symnmf_status finish() {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) { (void)cudaGetLastError(); return SYMNMF_ERR_CUDA; }
  return SYMNMF_OK;
}

__global__ void set_i32(int32_t* p, int32_t v) { *p = v; }
__global__ void bump_iter(int32_t* it) {
  pdl_trigger();
  pdl_wait();
  *it += 1;
}
__global__ void record_stats(const int32_t* iter_dev, int32_t first, int32_t max_iters, int side,
                             const int64_t* counts, const double* mass, symnmf_half_stats* stats) {
  const int t = *iter_dev - first;
  if (t < 0 || t >= max_iters) return;
  symnmf_half_stats h;
  h.s_d = counts[0]; h.s_r = counts[1]; h.n_uniq = counts[2]; h.theta = mass[0];
  stats[2 * t + side] = h;
}
__global__ void record_resid(const int32_t* iter_dev, int32_t first, int32_t max_iters, const double* rout,
                             double* resid) {
  pdl_trigger();
  pdl_wait();
  const int t = *iter_dev - first;
  if (t < 0 || t >= max_iters) return;
  resid[t] = rout[0];
}

// Dense or CSR exact product into Y (n x k, ld k).
bool enqueue_product(const symnmf_matrix& A, const float* F, int k, float* Y, int precision, void* tcs,
                     size_t tcs_bytes, const int32_t* status, cudaStream_t st) {
  if (A.kind == SYMNMF_CSR) { launch_spmm_csr(A, F, k, Y, status, st); return true; }
  if (precision == SYMNMF_3XTF32)
    return launch_dense_ah_tc(A.val, A.lda, A.n, F, k, k, Y, k, tcs, tcs_bytes, status, st);
  launch_dense_ah_simt(A.val, A.lda, A.n, F, k, k, Y, k, status, st);
  return true;
}

void enqueue_gram(const float* F, int64_t n, int k, double* partial, int grid, double* G, const int32_t* status,
                  cudaStream_t st) {
  launch_cross_gram(F, k, k, F, k, k, true, n, nullptr, nullptr, nullptr, partial, grid, G, k, status, st);
}

}  // namespace

extern "C" int32_t symnmf_version(void) { return 100; }   // 0.1.0

extern "C" symnmf_status symnmf_status_read(const void* ws, int32_t* status_host, cudaStream_t st) {
  if (!ws || !status_host) return SYMNMF_ERR_ARG;
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(status_host, ws, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
  return SYMNMF_OK;
}

// ---------------------------------------------------------------- (a1)
extern "C" symnmf_status symnmf_gram(const float* F, int64_t n, int32_t k, double* G, void* ws, size_t* ws_bytes,
                                     cudaStream_t st) {
  if (!F || !G || n < 1 || bad_k(k)) return SYMNMF_ERR_ARG;
  const int grid = gram_grid(n);
  Carver c(nullptr);
  c.take<double>(gram_partial_doubles(k, k, true, grid));
  bool q;
  symnmf_status s = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (s != SYMNMF_OK || q) return s;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  double* part = w.take<double>(gram_partial_doubles(k, k, true, grid));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  enqueue_gram(F, n, k, part, grid, G, ws_status(ws), st);
  return finish();
}

// ---------------------------------------------------------------- (a10)
extern "C" symnmf_status symnmf_ah(const symnmf_matrix* A, const float* F, int32_t k, float* Y, int32_t precision,
                                   void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (bad_matrix(A) || !F || !Y || bad_k(k)) return SYMNMF_ERR_ARG;
  if (precision != SYMNMF_FP32 && precision != SYMNMF_3XTF32) return SYMNMF_ERR_ARG;
  if (A->kind == SYMNMF_CSR && precision != SYMNMF_FP32) return SYMNMF_ERR_ARG;
  const size_t tcs = (A->kind == SYMNMF_DENSE && precision == SYMNMF_3XTF32) ? dense_ah_tc_scratch(A->n, k) : 0;
  Carver c(nullptr);
  c.take<char>(tcs);
  bool q;
  symnmf_status s = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (s != SYMNMF_OK || q) return s;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  void* scratch = w.take<char>(tcs);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  if (!enqueue_product(*A, F, k, Y, precision, scratch, tcs, ws_status(ws), st)) return SYMNMF_ERR_UNSUPPORTED;
  return finish();
}

// ---------------------------------------------------------------- (a1)-(a3)
extern "C" symnmf_status symnmf_leverage_scores(const float* F, int64_t n, int32_t k, float* lev, double* G_out,
                                                void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (!F || !lev || n < 1 || bad_k(k)) return SYMNMF_ERR_ARG;
  const int grid = gram_grid(n), kp = kpad(k);
  auto layout = [&](Carver& c, double** part, double** G, float** R) {
    *part = c.take<double>(gram_partial_doubles(k, k, true, grid));
    *G = c.take<double>((size_t)k * k);
    *R = c.take<float>((size_t)kp * kp);
  };
  double *part, *G;
  float* R;
  Carver c(nullptr);
  layout(c, &part, &G, &R);
  bool q;
  symnmf_status s = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (s != SYMNMF_OK || q) return s;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  layout(w, &part, &G, &R);
  if (G_out) G = G_out;
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  enqueue_gram(F, n, k, part, grid, G, status, st);
  launch_chol_inv(G, k, R, kp, kp, nullptr, 0, status, st);
  launch_leverage(F, n, k, R, lev, status, st);
  return finish();
}

// ---------------------------------------------------------------- (a4)-(a7)
static void sampler_layout(Carver& c, int64_t n, SamplerWs* sw) {
  const int64_t nb = samp_blocks(n);
  sw->bw = c.take<uint64_t>(nb);
  sw->bd = c.take<uint32_t>(nb);
  sw->bt = c.take<double>(nb);
  sw->bu = c.take<uint32_t>(nb);
  sw->P = c.take<uint64_t>(n);
  sw->cnt = c.take<int32_t>(n);
}

static bool bad_plan(const symnmf_plan* p) {
  return !p || p->cap < 1 || !p->det_idx || !p->draw_idx || !p->uniq_idx || !p->uniq_w || !p->counts || !p->mass;
}

extern "C" symnmf_status symnmf_hybrid_sample(const float* lev, int64_t n, int32_t k, int64_t s, double tau,
                                              uint64_t seed, uint32_t iteration, uint32_t side,
                                              const symnmf_plan* plan, void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (!lev || n < 1 || bad_k(k) || s < 1 || !(tau > 0.0 && tau <= 1.0) || side > 1 || bad_plan(plan))
    return SYMNMF_ERR_ARG;
  SamplerWs sw;
  Carver c(nullptr);
  sampler_layout(c, n, &sw);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  sampler_layout(w, n, &sw);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(sw.cnt, 0, sizeof(int32_t) * n, st));
  const double T = tau * (double)k;   // reading Z1: threshold on p_i = l_i / k
  launch_hybrid_sample(lev, n, k, s, T, seed, nullptr, iteration, side, *plan, sw, ws_status(ws), st);
  return finish();
}

// ---------------------------------------------------------------- NEXT-4 row-sharded building blocks (shard.cu)
extern "C" symnmf_status symnmf_leverage_scores_gram(const float* F, int64_t n, int32_t k, const double* G, float* lev,
                                                     void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (!F || !G || !lev || n < 1 || bad_k(k)) return SYMNMF_ERR_ARG;
  const int kp = kpad(k);
  Carver c(nullptr);
  c.take<float>((size_t)kp * kp);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  float* R = w.take<float>((size_t)kp * kp);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_chol_inv(G, k, R, kp, kp, nullptr, 0, status, st);
  launch_leverage(F, n, k, R, lev, status, st);
  return finish();
}

extern "C" symnmf_status symnmf_hybrid_shard_sums(const float* lev, int64_t n, int32_t k, double tau, uint64_t* W_out,
                                                  int64_t* sD_out, double* theta_out, void* ws, size_t* ws_bytes,
                                                  cudaStream_t st) {
  if (!lev || n < 1 || bad_k(k) || !(tau > 0.0 && tau <= 1.0) || !W_out || !sD_out || !theta_out)
    return SYMNMF_ERR_ARG;
  SamplerWs sw;
  Carver c(nullptr);
  sampler_layout(c, n, &sw);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  sampler_layout(w, n, &sw);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_shard_sums(lev, n, tau * (double)k, sw, W_out, sD_out, theta_out, ws_status(ws), st);
  return finish();
}

extern "C" symnmf_status symnmf_hybrid_shard_plan(const float* lev, int64_t n, int64_t row0, int32_t k, int64_t s,
                                                  double tau, uint64_t seed, uint32_t iteration, uint32_t side,
                                                  uint64_t W_offset, uint64_t W_total, int64_t sD_total,
                                                  const symnmf_plan* plan, void* ws, size_t* ws_bytes,
                                                  cudaStream_t st) {
  if (!lev || n < 1 || row0 < 0 || bad_k(k) || s < 1 || !(tau > 0.0 && tau <= 1.0) || side > 1 || bad_plan(plan) ||
      sD_total < 0)
    return SYMNMF_ERR_ARG;
  SamplerWs sw;
  auto layout = [&](Carver& c, uint64_t** wloc) {
    sampler_layout(c, n, &sw);
    *wloc = c.take<uint64_t>(1);
  };
  uint64_t* wloc;
  Carver c(nullptr);
  layout(c, &wloc);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  layout(w, &wloc);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(sw.cnt, 0, sizeof(int32_t) * n, st));
  launch_shard_plan(lev, n, row0, k, s, tau * (double)k, seed, iteration, side, W_offset, W_total, sD_total, *plan, sw,
                    wloc, ws_status(ws), st);
  return finish();
}

extern "C" symnmf_status symnmf_plan_rows_scaled(const float* F, int64_t row0, int32_t k, const symnmf_plan* plan,
                                                 float* Z, double* G_s, void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (!F || row0 < 0 || bad_k(k) || bad_plan(plan) || !Z) return SYMNMF_ERR_ARG;
  const int grid = gram_grid(plan->cap);
  Carver c(nullptr);
  c.take<double>(gram_partial_doubles(k, k, true, grid));
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  double* part = w.take<double>(gram_partial_doubles(k, k, true, grid));
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_plan_rows_scaled(F, row0, k, *plan, Z, status, st);
  // the block's share of G_s = sum_t omega_t f_t^T f_t (rows u_t - row0 of the block's F)
  if (G_s)
    launch_cross_gram(F - row0 * k, k, k, F - row0 * k, k, k, true, plan->cap, plan->counts + 2, plan->uniq_idx,
                      plan->uniq_w, part, grid, G_s, k, status, st);
  return finish();
}

extern "C" symnmf_status symnmf_sampled_ah_rows(const symnmf_matrix* A_block, int64_t n_total, const int32_t* uniq,
                                                const int64_t* n_uniq_dev, int64_t cap, const float* Z, int32_t k,
                                                float* Y, void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (!A_block || A_block->kind != SYMNMF_CSR || A_block->n < 1 || !A_block->rowptr || n_total < 1 || !uniq ||
      !n_uniq_dev || cap < 1 || !Z || bad_k(k) || !Y)
    return SYMNMF_ERR_ARG;
  Carver c(nullptr);
  c.take<int32_t>((size_t)n_total);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  int32_t* slot = w.take<int32_t>((size_t)n_total);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_sampled_rows_pull(*A_block, n_total, uniq, n_uniq_dev, cap, Z, k, Y, slot, status, st);
  return finish();
}

// ---------------------------------------------------------------- (a8), (a9)
extern "C" symnmf_status symnmf_sampled_ah(const symnmf_matrix* A, const float* F, int32_t k, const symnmf_plan* plan,
                                           float* Y, double* G_s, void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (bad_matrix(A) || !F || !Y || bad_k(k) || bad_plan(plan)) return SYMNMF_ERR_ARG;
  const int grid = gram_grid(std::min<int64_t>(plan->cap, A->n));
  const int64_t cap = std::min<int64_t>(plan->cap, A->n);
  const size_t sbs_bytes = (A->kind == SYMNMF_DENSE && sampled_dense_tc_enabled(A->n) &&
                            sampled_dense_tc_supported(A->val, A->lda, A->n, k))
                               ? sampled_dense_tc_scratch(cap, k)
                               : 0;
  Carver c(nullptr);
  c.take<double>(gram_partial_doubles(k, k, true, grid));
  c.take<char>(sbs_bytes);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  double* part = w.take<double>(gram_partial_doubles(k, k, true, grid));
  char* sbs = w.take<char>(sbs_bytes);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  if (A->kind == SYMNMF_CSR)
    launch_sampled_csr(*A, F, k, plan->uniq_idx, plan->uniq_w, plan->counts + 2, cap, Y, status, st);
  else if (sbs_bytes)
    launch_sampled_dense_tc(A->val, A->lda, A->n, F, k, plan->uniq_idx, plan->uniq_w, plan->counts + 2, cap, cap, Y,
                            sbs, status, st);
  else
    launch_sampled_dense(A->val, A->lda, A->n, F, k, plan->uniq_idx, plan->uniq_w, plan->counts + 2, cap, Y, status, st);
  if (G_s)
    launch_cross_gram(F, k, k, F, k, k, true, cap, plan->counts + 2, plan->uniq_idx, plan->uniq_w, part, grid, G_s, k,
                      status, st);
  return finish();
}

// ---------------------------------------------------------------- (a12)
extern "C" symnmf_status symnmf_gaussian(int64_t n, int32_t l, uint64_t seed, float* Omega, cudaStream_t st) {
  if (n < 1 || l < 1 || !Omega) return SYMNMF_ERR_ARG;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  launch_gaussian(n, l, seed, Omega, st);
  return finish();
}

namespace {
struct RfLayout {
  float *Om, *Yb, *Q1, *Q;
  double *Gl, *R64, *part, *T, *V;
  void* tcs;
  size_t tcs_bytes;
  int grid;
};
void rf_layout(Carver& c, int64_t n, int l, int precision, RfLayout* L) {
  L->grid = gram_grid(n);
  L->Om = c.take<float>((size_t)n * l);
  L->Yb = c.take<float>((size_t)n * l);
  L->Q1 = c.take<float>((size_t)n * l);
  L->Q = c.take<float>((size_t)n * l);
  L->Gl = c.take<double>((size_t)l * l);
  L->R64 = c.take<double>((size_t)l * l);
  L->T = c.take<double>((size_t)l * l);
  L->V = c.take<double>((size_t)l * l);
  L->part = c.take<double>(gram_partial_doubles(l, l, false, L->grid));
  L->tcs_bytes = precision == SYMNMF_3XTF32 ? dense_ah_tc_scratch(n, l) : 0;
  L->tcs = c.take<char>(L->tcs_bytes);
}
// orth(Yb) -> Q by shifted CholeskyQR2 with fp64 Gram, Cholesky and row apply: the
// first pass factors G + 1e-14 tr(G) I (span(Q1) = span(Y) is unchanged; a sketch
// that is rank deficient to fp32 precision, e.g. an exact low-rank A, stays
// factorable), the second pass restores orthonormality.
void enqueue_orth(const RfLayout& L, int64_t n, int l, const float* Yin, float* Qout, int32_t* status, cudaStream_t st) {
  launch_cross_gram(Yin, l, l, Yin, l, l, true, n, nullptr, nullptr, nullptr, L.part, L.grid, L.Gl, l, status, st,
                    true);
  launch_chol_inv(L.Gl, l, nullptr, 0, 0, L.R64, l, status, st, 1e-14);
  launch_rowapply64(Yin, l, n, l, L.R64, l, L.Q1, l, status, st);
  launch_cross_gram(L.Q1, l, l, L.Q1, l, l, true, n, nullptr, nullptr, nullptr, L.part, L.grid, L.Gl, l, status, st,
                    true);
  launch_chol_inv(L.Gl, l, nullptr, 0, 0, L.R64, l, status, st);
  launch_rowapply64(L.Q1, l, n, l, L.R64, l, Qout, l, status, st);
}
bool enqueue_dense_apply(const symnmf_matrix& A, const float* X, int l, float* Y, int precision, const RfLayout& L,
                         const int32_t* status, cudaStream_t st) {
  if (precision == SYMNMF_3XTF32)
    return launch_dense_ah_tc(A.val, A.lda, A.n, X, l, l, Y, l, L.tcs, L.tcs_bytes, status, st);
  launch_dense_ah_simt(A.val, A.lda, A.n, X, l, l, Y, l, status, st);
  return true;
}
}  // namespace

extern "C" symnmf_status symnmf_rangefinder(const symnmf_matrix* A, int32_t l, int32_t q, uint64_t seed,
                                            int32_t precision, float* U, double* lambda, void* ws, size_t* ws_bytes,
                                            cudaStream_t st) {
  if (bad_matrix(A) || A->kind != SYMNMF_DENSE || l < 1 || l > kMaxL || l > A->n || q < 0 || !U || !lambda)
    return SYMNMF_ERR_ARG;
  if (precision != SYMNMF_FP32 && precision != SYMNMF_3XTF32) return SYMNMF_ERR_ARG;
  const int64_t n = A->n;
  RfLayout L;
  Carver c(nullptr);
  rf_layout(c, n, l, precision, &L);
  bool qq;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &qq);
  if (r != SYMNMF_OK || qq) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  rf_layout(w, n, l, precision, &L);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_gaussian(n, l, seed, L.Om, st);                                   // Alg. RRF line "Draw Omega"
  if (!enqueue_dense_apply(*A, L.Om, l, L.Yb, precision, L, status, st)) return SYMNMF_ERR_UNSUPPORTED;
  enqueue_orth(L, n, l, L.Yb, L.Q, status, st);
  for (int t = 0; t < q; ++t) {                                             // (A A^T)^q with re-orthonormalisation
    for (int h = 0; h < 2; ++h) {
      enqueue_dense_apply(*A, L.Q, l, L.Yb, precision, L, status, st);
      enqueue_orth(L, n, l, L.Yb, L.Q, status, st);
    }
  }
  enqueue_dense_apply(*A, L.Q, l, L.Yb, precision, L, status, st);        // Z = A Q
  launch_cross_gram(L.Q, l, l, L.Yb, l, l, false, n, nullptr, nullptr, nullptr, L.part, L.grid, L.T, l, status, st,
                    true);
  launch_symmetrize(L.T, l, st);                                            // T = Q^T A Q
  launch_jacobi_evd(L.T, l, L.V, lambda, status, st);                       // T = V Lambda V^T
  launch_rowapply64(L.Q, l, n, l, L.V, l, U, l, status, st);                // U = Q V
  return finish();
}

// ---------------------------------------------------------------- NEXT-2 Ada-RRF
extern "C" symnmf_status symnmf_rangefinder_adaptive(const symnmf_matrix* A, int32_t l, int32_t q_max, double tol,
                                                     uint64_t seed, int32_t precision, float* U, double* lambda,
                                                     int32_t* passes_host, double* resid_host, void* ws,
                                                     size_t* ws_bytes, cudaStream_t st) {
  // Alg. Ada-RRF (App. E) + Apx-EVD; reading Z31 (symnmf.h)
  if (bad_matrix(A) || A->kind != SYMNMF_DENSE || l < 1 || l > kMaxL || l > A->n || q_max < 1 || !U || !lambda ||
      !(tol >= 0.0))
    return SYMNMF_ERR_ARG;
  if (precision != SYMNMF_FP32 && precision != SYMNMF_3XTF32) return SYMNMF_ERR_ARG;
  const int64_t n = A->n;
  RfLayout L;
  double *sq_part = nullptr, *sq = nullptr;
  auto layout = [&](Carver& c) {
    rf_layout(c, n, l, precision, &L);
    sq_part = c.take<double>(sumsq_grid());
    sq = c.take<double>(2);
  };
  Carver c(nullptr);
  layout(c);
  bool qq;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &qq);
  if (r != SYMNMF_OK || qq) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  layout(w);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  double a2 = 0.0, b2 = 0.0;
  launch_sumsq(A->val, n, n, A->lda, sq_part, sq, status, st);              // ||A||_F^2
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(&a2, sq, sizeof(double), cudaMemcpyDeviceToHost, st));
  launch_gaussian(n, l, seed, L.Om, st);                                   // Draw Omega
  if (!enqueue_dense_apply(*A, L.Om, l, L.Yb, precision, L, status, st)) return SYMNMF_ERR_UNSUPPORTED;
  enqueue_orth(L, n, l, L.Yb, L.Q, status, st);                             // Q = qr(A Omega)
  SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
  double prev = 0.0;
  int32_t j = 0;
  for (;;) {
    ++j;
    // B^T = A^T Q = A Q, always by the fp32 SIMT product: the residual trick subtracts ||B||^2 from
    // ||A||^2, so a relative bias eps in B moves r by ~eps / r.  3xTF32 carries the tensor core's
    // truncation bias (-1.6e-6, tc_gemm.cu), which at r = 5e-3 is a 3% error in r; round-to-
    // nearest fp32 errors are unbiased and cancel in the fp64 sum of squares (reading R3).
    enqueue_dense_apply(*A, L.Q, l, L.Yb, SYMNMF_FP32, L, status, st);
    launch_sumsq(L.Yb, n, l, l, sq_part, sq, status, st);                   // ||B||_F^2
    SYMNMF_CUDA_TRY(cudaMemcpyAsync(&b2, sq, sizeof(double), cudaMemcpyDeviceToHost, st));
    enqueue_orth(L, n, l, L.Yb, L.Q, status, st);                           // Q = qr(B^T)
    SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
    const double res = std::sqrt(std::max(a2 - b2, 0.0)) / std::sqrt(a2);  // QB residual trick
    if (resid_host) resid_host[j - 1] = res;
    if (j >= q_max || (j > 1 && prev - res <= tol)) break;                 // stopping criterion
    prev = res;
    enqueue_dense_apply(*A, L.Q, l, L.Yb, precision, L, status, st);      // Y = A Q
    enqueue_orth(L, n, l, L.Yb, L.Q, status, st);                           // Q = qr(Y)
  }
  if (passes_host) *passes_host = j;
  enqueue_dense_apply(*A, L.Q, l, L.Yb, precision, L, status, st);        // Z = A Q
  launch_cross_gram(L.Q, l, l, L.Yb, l, l, false, n, nullptr, nullptr, nullptr, L.part, L.grid, L.T, l, status, st,
                    true);
  launch_symmetrize(L.T, l, st);                                            // T = Q^T A Q
  launch_jacobi_evd(L.T, l, L.V, lambda, status, st);                       // T = V Lambda V^T
  launch_rowapply64(L.Q, l, n, l, L.V, l, U, l, status, st);                // U = Q V
  return finish();
}

// ---------------------------------------------------------------- (a13)
extern "C" symnmf_status symnmf_lai_ah(const float* U, const double* lambda, int64_t n, int32_t l, const float* F,
                                       int32_t k, float* Y, void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (!U || !lambda || !F || !Y || n < 1 || l < 1 || l > kMaxL || bad_k(k)) return SYMNMF_ERR_ARG;
  const int grid = gram_grid(n);
  auto layout = [&](Carver& c, double** part, double** Z, float** M) {
    *part = c.take<double>(gram_partial_doubles(l, k, false, grid));
    *Z = c.take<double>((size_t)l * k);
    *M = c.take<float>((size_t)l * k);
  };
  double *part, *Z;
  float* M;
  Carver c(nullptr);
  layout(c, &part, &Z, &M);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  layout(w, &part, &Z, &M);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_cross_gram(U, l, l, F, k, k, false, n, nullptr, nullptr, nullptr, part, grid, Z, k, status, st);
  launch_scale_rows(Z, l, k, lambda, M, status, st);
  launch_rowapply32(U, l, n, l, M, k, Y, k, status, st);
  return finish();
}

// NEXT-4: the two halves of symnmf_lai_ah for a row block (the l x k allreduce between them is the caller's).
extern "C" symnmf_status symnmf_lai_project_rows(const float* U, int64_t n, int32_t l, const float* F, int32_t k,
                                                 double* Z, void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (!U || !F || !Z || n < 1 || l < 1 || l > kMaxL || bad_k(k)) return SYMNMF_ERR_ARG;
  const int grid = gram_grid(n);
  Carver c(nullptr);
  c.take<double>(gram_partial_doubles(l, k, false, grid));
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  double* part = w.take<double>(gram_partial_doubles(l, k, false, grid));
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_cross_gram(U, l, l, F, k, k, false, n, nullptr, nullptr, nullptr, part, grid, Z, k, status, st);
  return finish();
}

extern "C" symnmf_status symnmf_lai_apply_rows(const float* U, const double* lambda, int64_t n, int32_t l,
                                               const double* Z, int32_t k, float* Y, void* ws, size_t* ws_bytes,
                                               cudaStream_t st) {
  if (!U || !lambda || !Z || !Y || n < 1 || l < 1 || l > kMaxL || bad_k(k)) return SYMNMF_ERR_ARG;
  Carver c(nullptr);
  c.take<float>((size_t)l * k);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  float* M = w.take<float>((size_t)l * k);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_scale_rows(Z, l, k, lambda, M, status, st);
  launch_rowapply32(U, l, n, l, M, k, Y, k, status, st);
  return finish();
}

// ---------------------------------------------------------------- (a11)
extern "C" symnmf_status symnmf_hals_sweep(const double* G, const float* Y, const float* F, float* X, int64_t n,
                                           int32_t k, double alpha, double* G_new, void* ws, size_t* ws_bytes,
                                           cudaStream_t st) {
  if (!G || !Y || !F || !X || n < 1 || bad_k(k) || !(alpha >= 0.0)) return SYMNMF_ERR_ARG;
  const int grid = gram_grid(n);
  Carver c(nullptr);
  c.take<double>(gram_partial_doubles(k, k, true, grid));
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  double* part = w.take<double>(gram_partial_doubles(k, k, true, grid));
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  launch_hals_sweep(G, Y, F, X, n, k, alpha, status, st);
  if (G_new) enqueue_gram(X, n, k, part, grid, G_new, status, st);
  return finish();
}

// ---------------------------------------------------------------- NEXT-1 BPP update
extern "C" symnmf_status symnmf_bpp_update(const double* G, const float* Y, const float* F, float* X, int64_t n,
                                           int32_t k, double alpha, double* G_new, int32_t* nonconv_host, void* ws,
                                           size_t* ws_bytes, cudaStream_t st) {
  if (!G || !Y || !F || !X || n < 1 || bad_k(k) || !(alpha >= 0.0)) return SYMNMF_ERR_ARG;
  if (!bpp_supported(k)) return SYMNMF_ERR_UNSUPPORTED;
  const int grid = gram_grid(n);
  auto layout = [&](Carver& c, double** part, int32_t** nc) {
    *part = c.take<double>(gram_partial_doubles(k, k, true, grid));
    *nc = c.take<int32_t>(1);
  };
  double* part;
  int32_t* nc;
  Carver c(nullptr);
  layout(c, &part, &nc);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  layout(w, &part, &nc);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(nc, 0, sizeof(int32_t), st));
  launch_bpp(G, const_cast<float*>(Y), F, X, n, k, alpha, false, nc, status, st);
  if (G_new) enqueue_gram(X, n, k, part, grid, G_new, status, st);
  if (nonconv_host) {
    SYMNMF_CUDA_TRY(cudaMemcpyAsync(nonconv_host, nc, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return finish();
}

// ---------------------------------------------------------------- (a15)
extern "C" symnmf_status symnmf_residual(const symnmf_matrix* A, const float* H, int32_t k, double* out, void* ws,
                                         size_t* ws_bytes, cudaStream_t st) {
  if (bad_matrix(A) || !H || !out || bad_k(k)) return SYMNMF_ERR_ARG;
  const int64_t n = A->n;
  const int rgrid = residual_grid(n), ggrid = gram_grid(n);
  const bool csr = A->kind == SYMNMF_CSR;
  auto layout = [&](Carver& c, double** rp, float** AH, double** G, double** gp) {
    *rp = c.take<double>((size_t)2 * rgrid);
    *AH = c.take<float>(csr ? (size_t)n * k : 0);
    *G = c.take<double>(csr ? (size_t)k * k : 0);
    *gp = c.take<double>(csr ? gram_partial_doubles(k, k, true, ggrid) : 0);
  };
  double *rp, *G, *gp;
  float* AH;
  Carver c(nullptr);
  layout(c, &rp, &AH, &G, &gp);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  layout(w, &rp, &AH, &G, &gp);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  if (csr) {
    launch_spmm_csr(*A, H, k, AH, status, st);
    enqueue_gram(H, n, k, gp, ggrid, G, status, st);
  }
  launch_residual(*A, H, k, AH, G, rp, rgrid, out, status, st);
  return finish();
}

// ---------------------------------------------------------------- NEXT-3 projected gradient
extern "C" symnmf_status symnmf_projected_gradient(const symnmf_matrix* A, const float* H, int32_t k,
                                                   int32_t precision, double* out, void* ws, size_t* ws_bytes,
                                                   cudaStream_t st) {
  if (bad_matrix(A) || !H || !out || bad_k(k)) return SYMNMF_ERR_ARG;
  if (precision != SYMNMF_FP32 && precision != SYMNMF_3XTF32) return SYMNMF_ERR_ARG;
  if (A->kind == SYMNMF_CSR && precision != SYMNMF_FP32) return SYMNMF_ERR_ARG;
  const int64_t n = A->n;
  const int pg = pgrad_grid(n), ggrid = gram_grid(n);
  const size_t tcs_bytes = (A->kind == SYMNMF_DENSE && precision == SYMNMF_3XTF32) ? dense_ah_tc_scratch(n, k) : 0;
  auto layout = [&](Carver& c, double** pp, float** AH, double** G, double** gp, char** tcs) {
    *pp = c.take<double>((size_t)2 * pg);
    *AH = c.take<float>((size_t)n * k);
    *G = c.take<double>((size_t)k * k);
    *gp = c.take<double>(gram_partial_doubles(k, k, true, ggrid));
    *tcs = c.take<char>(tcs_bytes);
  };
  double *pp, *G, *gp;
  float* AH;
  char* tcs;
  Carver c(nullptr);
  layout(c, &pp, &AH, &G, &gp, &tcs);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  layout(w, &pp, &AH, &G, &gp, &tcs);
  int32_t* status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, sizeof(int32_t), st));
  if (!enqueue_product(*A, H, k, AH, precision, tcs, tcs_bytes, status, st)) return SYMNMF_ERR_UNSUPPORTED;
  enqueue_gram(H, n, k, gp, ggrid, G, status, st);
  launch_pgrad(H, AH, G, n, k, pp, pg, out, status, st);
  return finish();
}

// ---------------------------------------------------------------- (a14) solver
// SYMNMF_RECORD_PLANS: copy this half's scores and plan into history slot 2 (it - first) + side.
__global__ void record_plan(int64_t n, const float* __restrict__ lev, const int32_t* __restrict__ uniq,
                            const double* __restrict__ w, const int64_t* __restrict__ counts,
                            const double* __restrict__ mass, const int32_t* __restrict__ iter_dev, int32_t first_iter,
                            int32_t max_iters, int side, int64_t cap, float* __restrict__ hlev,
                            int32_t* __restrict__ huniq, double* __restrict__ hw, int64_t* __restrict__ hcounts,
                            double* __restrict__ hmass, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int t = *iter_dev - first_iter;
  if (t < 0 || t >= max_iters) return;
  const size_t h = (size_t)2 * t + side;
  const int64_t nu = counts[2];
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0; i < n; i += step) hlev[h * n + i] = lev[i];
  for (int64_t i = i0; i < nu; i += step) { huniq[h * cap + i] = uniq[i]; hw[h * cap + i] = w[i]; }
  if (i0 < 4) hcounts[h * 4 + i0] = counts[i0];
  if (i0 < 2) hmass[h * 2 + i0] = mass[i0];
}

struct symnmf_solver {
  symnmf_matrix A;
  bool hasA;
  int64_t n;
  float *W, *H;
  int k;
  double alpha;
  int mode, precision;
  int64_t s;
  double T;
  uint64_t seed;
  int32_t first_iter, max_iters;
  const float* U;
  const double* lam;
  int l;
  int with_resid;
  // workspace carve
  int32_t* status;
  int32_t* iter_dev;
  unsigned int* counter;   // last-CTA counter of the fused kernels (kept zero between launches)
  double* Gacc;            // zeroed fp64 Gram accumulator of the fused kernels
  double* Gbuf[2];         // Gbuf[side]: F^T F of the fixed factor of half `side`
  float* AHres;            // A H for the residual (CSR), separate from the sampled Y
  int ggrid, rgrid;
  double *G, *Gs, *gpart;
  float* Rinv32;
  float* lev;
  SamplerWs sw;
  symnmf_plan plan;
  float* Y;
  bool bpp;                // Update rule: exact per-row NLS by block principal pivoting (NEXT-1)
  int32_t* nonconv;        // BPP rows that hit the pivoting cap (device counter)
  int32_t* ppos;           // LvS on CSR: per-row boundaries of the scatter's destination passes
  bool yalpha;             // LvS on CSR, streaming sweep: Y carries alpha F between halves (sweep.cu)
  void* sbs;               // LvS on dense A: scratch of the tensor-core sampled product (tc_sampled.cu)
  size_t sbs_bytes;
  bool nnzsp;              // EXACT on CSR (kpad(k) == k): the nnz-balanced SpMM (spmm_nnz.cu)
  int64_t* chunk_row;
  float* carry;
  int cslot;               // constant-table slot of the streaming sweep (-1: G in shared memory)
  float* ctab;             // scratch for the table copied to the constant bank
  bool record;             // SYMNMF_RECORD_PLANS: per-half copies of the scores and plan
  float* hlev;
  int32_t* huniq;
  double* hw;
  int64_t* hcounts;
  double* hmass;
  symnmf_half_stats* stats;
  double *resid, *rpart, *rout, *GH;
  double *pgrad, *ppart, *pout;   // NEXT-3: per-iteration projected-gradient norm (with_resid)
  float* AHpg;                      // A H of the updated H for the projected gradient
  int pgrid;
  double *Zpart, *Z;
  float* M32;
  bool lai_fused;          // LAI: one fused launch per half (lai_fused.cu)
  float* Mside[2];         // Mside[side] = Lambda U^T F of half `side` (LP x k fp32)
  double* UXacc;           // zeroed kGramReplicas x LP x k accumulator of U^T X
  void* tcs;
  size_t tcs_bytes;
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  cudaStream_t side;                   // second branch of the iteration graph (G_s || Y_s)
  cudaEvent_t ev_fork[2], ev_join[2];  // per half
  int32_t iters_done;
  // profiling (symnmf_solver_profile): an event after every launch site of an eager iteration
  struct Prof {
    static constexpr int kMax = 64;
    cudaEvent_t ev[kMax + 1];
    const char* name[kMax];
    int n;
  }* prof;
};

namespace {

// Graph, exec, side stream, events and the constant-table slot of a solver (null-safe: used by
// destroy and by every failure path of create).
void release_solver_resources(symnmf_solver& S) {
  if (S.exec) cudaGraphExecDestroy(S.exec);
  if (S.graph) cudaGraphDestroy(S.graph);
  if (S.side) cudaStreamDestroy(S.side);
  for (int h = 0; h < 2; ++h) {
    if (S.ev_fork[h]) cudaEventDestroy(S.ev_fork[h]);
    if (S.ev_join[h]) cudaEventDestroy(S.ev_join[h]);
  }
  sweep_cslot_release(S.cslot);
  S.exec = nullptr; S.graph = nullptr; S.side = nullptr; S.cslot = -1;
  for (int h = 0; h < 2; ++h) S.ev_fork[h] = S.ev_join[h] = nullptr;
}

// The sweep's G through the constant bank (sweep.cu) unless SYMNMF_SWEEP_CMEM=0 (symnmf.h)
bool sweep_cmem_enabled() {
  const char* e = getenv("SYMNMF_SWEEP_CMEM");
  return !(e && !strcmp(e, "0"));
}

// The streaming sweep (sweep.cu) for k in {8, 16, 32}; SYMNMF_SWEEP=fused selects the register-tile
// sweep_fused instead (symnmf.h)
bool sweep_stream_enabled(int64_t n) {
  const char* e = getenv("SYMNMF_SWEEP");
  if (e && !strcmp(e, "fused")) return false;
  if (e && !strcmp(e, "stream")) return true;
  return n >= (1ll << 20);   // c4: 0.33 vs 0.43 ms; c2 (n = 100k, L2 resident): 31 vs 29 us
}

// Update(G + alpha I, Y + alpha F^T): one HALS sweep with the next half's Gram (and R) fused, or
// (rule BPP) the exact per-row NLS followed by the Gram of the new factor.
void enqueue_sweep(const symnmf_solver& S, int side, const double* G, const float* F, float* X, bool zeroY, double* Gnext,
                   float* Rf32, int32_t* status, cudaStream_t st) {
  if (S.bpp) {
    launch_bpp(G, S.Y, F, X, S.n, S.k, S.alpha, zeroY, S.nonconv, status, st);
    launch_gram_fused(X, S.n, S.k, S.Gacc, Gnext, Rf32, S.counter, status, st);
    return;
  }
  if (sweep_stream_supported(S.k) && sweep_stream_enabled(S.n))
    launch_sweep_stream(G, S.alpha, S.Y, F, X, S.n, S.k, zeroY, S.Gacc, Gnext, Rf32, S.counter, status, st,
                        S.cslot >= 0 ? 2 * S.cslot + side : -1, S.ctab, S.yalpha && zeroY);
  else
    launch_sweep_fused(G, S.alpha, S.Y, F, X, S.n, S.k, zeroY, S.Gacc, Gnext, Rf32, S.counter, status, st);
}

// LvS on CSR: Y carries alpha F between halves (default) or is re-zeroed (SYMNMF_YALPHA=0, symnmf.h)
bool yalpha_enabled() {
  const char* e = getenv("SYMNMF_YALPHA");
  return !(e && !strcmp(e, "0"));
}

// LAI: the fused one-launch half (k = 64, l <= 80); SYMNMF_LAI_FUSED=never disables it (symnmf.h)
bool lai_enabled() {
  const char* e = getenv("SYMNMF_LAI_FUSED");
  return !(e && !strcmp(e, "never"));
}

// EXACT CSR (kpad(k) == k): the nnz-balanced SpMM by default, the row-group SpMM with
// SYMNMF_CSR_SPMM=rows (symnmf.h)
bool csr_spmm_nnz(int64_t nnz) {
  const char* e = getenv("SYMNMF_CSR_SPMM");
  if (e && !strcmp(e, "rows")) return false;
  if (e && !strcmp(e, "nnz")) return true;
  return nnz >= (16ll << 20);   // c2 (2M nonzeros): row groups 26 us vs 60 us; c4: 5.4 ms vs 1.8 ms
}

// Profiling hook: records an event after the launch site just enqueued (no-op unless profiling).
void mark(symnmf_solver& S, cudaStream_t st, const char* name) {
  if (!S.prof || S.prof->n >= symnmf_solver::Prof::kMax) return;
  S.prof->name[S.prof->n] = name;
  cudaEventRecord(S.prof->ev[++S.prof->n], st);
}

__global__ void spin_kernel(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}

void solver_layout(symnmf_solver& S, Carver& c) {
  const int64_t n = S.n;
  const int k = S.k, kp = kpad(k);
  S.status = reinterpret_cast<int32_t*>(c.base);   // header
  S.iter_dev = c.take<int32_t>(4);
  S.counter = c.take<unsigned int>(4);
  S.Gacc = c.take<double>((size_t)kGramReplicas * k * k);
  S.Gbuf[0] = c.take<double>((size_t)k * k);
  S.Gbuf[1] = c.take<double>((size_t)k * k);
  S.AHres = c.take<float>((S.with_resid && S.hasA && S.A.kind == SYMNMF_CSR) ? (size_t)n * k : 0);
  S.ggrid = gram_grid(n);
  S.G = c.take<double>((size_t)k * k);
  S.Gs = c.take<double>((size_t)k * k);
  S.GH = c.take<double>((size_t)k * k);
  S.gpart = c.take<double>(gram_partial_doubles(k, k, true, S.ggrid));
  S.nnzsp = S.hasA && S.A.kind == SYMNMF_CSR && kp == k && S.mode == SYMNMF_EXACT && csr_spmm_nnz(S.A.nnz);
  S.chunk_row = c.take<int64_t>(S.nnzsp ? (size_t)spmm_nnz_chunks(S.A.nnz) : 0);
  S.carry = c.take<float>(S.nnzsp ? spmm_nnz_carry_floats(S.A.nnz, k) : 0);
  S.ctab = c.take<float>(sweep_table_floats());
  S.nonconv = c.take<int32_t>(1);
  S.Y = c.take<float>((size_t)n * k);
  S.stats = c.take<symnmf_half_stats>((size_t)2 * S.max_iters);
  S.resid = c.take<double>((size_t)S.max_iters);
  S.rgrid = residual_grid(n);
  S.rpart = c.take<double>((size_t)2 * S.rgrid);
  S.rout = c.take<double>(4);
  S.pgrid = pgrad_grid(n);
  S.pgrad = c.take<double>(S.with_resid ? (size_t)S.max_iters : 0);
  S.ppart = c.take<double>(S.with_resid ? (size_t)2 * S.pgrid : 0);
  S.pout = c.take<double>(S.with_resid ? 2 : 0);
  // CSR reuses AHres for the projected gradient; dense needs its own A H
  S.AHpg = c.take<float>((S.with_resid && S.hasA && S.A.kind == SYMNMF_DENSE) ? (size_t)n * k : 0);
  if (S.mode == SYMNMF_LVS) {
    S.Rinv32 = c.take<float>((size_t)kp * kp + kp);   // R (upper) | 1 / diag(R)
    S.lev = c.take<float>(n);
    sampler_layout(c, n, &S.sw);
    S.plan.cap = n;
    S.plan.det_idx = c.take<int32_t>(n);
    S.plan.draw_idx = c.take<int32_t>(S.s);
    S.plan.uniq_idx = c.take<int32_t>(n);
    S.plan.uniq_w = c.take<double>(n);
    S.plan.counts = c.take<int64_t>(4);
    S.plan.mass = c.take<double>(2);
    S.sbs_bytes = (S.hasA && S.A.kind == SYMNMF_DENSE && sampled_dense_tc_enabled(n) &&
                   sampled_dense_tc_supported(S.A.val, S.A.lda, n, k))
                      ? sampled_dense_tc_scratch(S.plan.cap, k)
                      : 0;
    S.sbs = c.take<char>(S.sbs_bytes);
    const int passes = (S.hasA && S.A.kind == SYMNMF_CSR) ? sampled_csr_passes(n, k) : 1;
    S.ppos = c.take<int32_t>(passes > 1 ? (size_t)passes * n : 0);
    const size_t halves = S.record ? (size_t)2 * S.max_iters : 0;
    S.hlev = c.take<float>(halves * n);
    S.huniq = c.take<int32_t>(halves * S.plan.cap);
    S.hw = c.take<double>(halves * S.plan.cap);
    S.hcounts = c.take<int64_t>(halves * 4);
    S.hmass = c.take<double>(halves * 2);
  }
  if (S.mode == SYMNMF_LAI) {
    S.Zpart = c.take<double>(gram_partial_doubles(S.l, k, false, S.ggrid));
    S.Z = c.take<double>((size_t)S.l * k);
    S.M32 = c.take<float>((size_t)S.l * k);
    S.lai_fused = lai_fused_supported(k, S.l) && lai_enabled() && !S.bpp;
    const size_t lp = S.lai_fused ? (size_t)lai_lp(S.l) : 0;
    S.Mside[0] = c.take<float>(lp * k);
    S.Mside[1] = c.take<float>(lp * k);
    S.UXacc = c.take<double>(lp * k * kGramReplicas);
  }
  S.tcs_bytes = (S.hasA && S.A.kind == SYMNMF_DENSE && S.precision == SYMNMF_3XTF32) ? dense_ah_tc_scratch(n, k) : 0;
  S.tcs = c.take<char>(S.tcs_bytes);
}

bool enqueue_half(symnmf_solver& S, int side, cudaStream_t st) {
  const int64_t n = S.n;
  const int k = S.k;
  float* F = side == 0 ? S.H : S.W;   // W-half: H fixed (Alg. LvS-SymNMF)
  float* X = side == 0 ? S.W : S.H;   // H-half: W fixed (lines 690-696)
  int32_t* status = S.status;
  // F^T F of the fixed factor was produced by the previous sweep (fused Gram of its output),
  // or at solver creation for the first half; the sweep below produces X^T X for the next half.
  const double* Gf = S.Gbuf[side];
  double* Gnext = S.Gbuf[side ^ 1];
  const bool lvs = S.mode == SYMNMF_LVS;
  if (S.mode == SYMNMF_EXACT && S.nnzsp) {
    launch_spmm_nnz(S.A, S.chunk_row, F, k, S.Y, S.carry, status, st);
    mark(S, st, "spmm_csr");
    enqueue_sweep(S, side, Gf, F, X, false, Gnext, nullptr, status, st);
    mark(S, st, S.bpp ? "bpp_update" : "hals_sweep");
  } else if (S.mode == SYMNMF_EXACT) {
    if (!enqueue_product(S.A, F, k, S.Y, S.precision, S.tcs, S.tcs_bytes, status, st)) return false;
    mark(S, st, S.A.kind == SYMNMF_CSR ? "spmm_csr" : (S.precision == SYMNMF_3XTF32 ? "gemm_3xtf32" : "gemm_fp32"));
    enqueue_sweep(S, side, Gf, F, X, false, Gnext, nullptr, status, st);
    mark(S, st, S.bpp ? "bpp_update" : "hals_sweep");
  } else if (lvs) {
    // scores of F from R^{-1} (computed with F^T F) fused with sampler pass S1/S2
    launch_leverage_fused(F, n, k, S.Rinv32, S.lev, S.T, S.sw, S.s, S.plan, S.counter, status, st,
                          S.cslot >= 0 ? 2 * S.cslot + side : -1);
    mark(S, st, "leverage");
    launch_samp_prefix(S.lev, n, S.T, S.sw, S.plan, status, st);
    mark(S, st, "samp_prefix");
    launch_samp_draws(S.sw, n, S.s, S.seed, S.iter_dev, 0, (uint32_t)side, S.plan, status, st);
    mark(S, st, "samp_draws");
    launch_uniq_count_fused(S.lev, n, S.T, S.sw, S.plan, S.iter_dev, S.first_iter, S.max_iters, side, S.stats,
                            S.counter, status, st);
    mark(S, st, "samp_uniq_count");
    launch_samp_uniq_write(S.lev, n, S.T, S.sw, S.plan, status, st);
    mark(S, st, "samp_uniq_write");
    if (S.record)
      launch_pdl(record_plan, 148 * 4, 256, 0, st, n, S.lev, S.plan.uniq_idx, S.plan.uniq_w, S.plan.counts,
                 S.plan.mass, S.iter_dev, S.first_iter, S.max_iters, side, S.plan.cap, S.hlev, S.huniq, S.hw,
                 S.hcounts, S.hmass, status);
    // G_s and Y_s only read the plan: G_s runs on a second branch of the graph, concurrently
    cudaEventRecord(S.ev_fork[side], st);
    cudaStreamWaitEvent(S.side, S.ev_fork[side], 0);
    launch_sampled_gram_fused(F, k, S.plan, S.Gacc, S.Gs, S.counter, status, S.side);
    cudaEventRecord(S.ev_join[side], S.side);
    if (S.A.kind == SYMNMF_CSR) {
      launch_sampled_csr_nozero(S.A, F, k, S.plan.uniq_idx, S.plan.uniq_w, S.plan.counts + 2, S.plan.cap, S.Y,
                                status, st, S.ppos);
      mark(S, st, "sampled_ah_csr");
    } else {
      if (S.sbs_bytes)
        launch_sampled_dense_tc(S.A.val, S.A.lda, n, F, k, S.plan.uniq_idx, S.plan.uniq_w, S.plan.counts + 2,
                                S.plan.cap, std::min<int64_t>(S.s, n), S.Y, S.sbs, status, st);
      else
        launch_sampled_dense(S.A.val, S.A.lda, n, F, k, S.plan.uniq_idx, S.plan.uniq_w, S.plan.counts + 2, S.plan.cap,
                             S.Y, status, st);
      mark(S, st, "sampled_ah_dense");
    }
    cudaStreamWaitEvent(st, S.ev_join[side], 0);
    // Update(G_s + alpha I, Y_s + alpha F^T); Y re-zeroed for the next scatter; X^T X and its R^{-1}
    // Y re-zeroed by the sweep for the next scatter (CSR); the dense sampled products write every
    // row of Y themselves, so there the sweep leaves Y as is (k * 4 bytes per row less)
    enqueue_sweep(S, side, S.Gs, F, X, S.A.kind == SYMNMF_CSR, Gnext, S.Rinv32, status, st);
    mark(S, st, S.bpp ? "bpp_update" : "hals_sweep");
  } else if (S.lai_fused) {
    // Y = U (Lambda U^T F), sweep, X^T X and Lambda U^T X for the next half, in one launch
    launch_lai_sweep_fused(S.U, S.l, n, k, S.Mside[side], Gf, S.alpha, F, X, S.lam, S.Gacc, S.UXacc, Gnext,
                           S.Mside[side ^ 1], S.counter, status, st);
    mark(S, st, "lai_fused");
  } else {
    launch_cross_gram(S.U, S.l, S.l, F, k, k, false, n, nullptr, nullptr, nullptr, S.Zpart, S.ggrid, S.Z, k, status,
                      st);
    mark(S, st, "lai_utf");
    launch_scale_rows(S.Z, S.l, k, S.lam, S.M32, status, st);
    launch_rowapply32(S.U, S.l, n, S.l, S.M32, k, S.Y, k, status, st);
    mark(S, st, "lai_uz");
    enqueue_sweep(S, side, Gf, F, X, false, Gnext, nullptr, status, st);
    mark(S, st, S.bpp ? "bpp_update" : "hals_sweep");
  }
  return true;
}

bool enqueue_iteration(symnmf_solver& S, cudaStream_t st) {
  if (!enqueue_half(S, 0, st) || !enqueue_half(S, 1, st)) return false;
  if (S.with_resid) {
    if (S.A.kind == SYMNMF_CSR) launch_spmm_csr(S.A, S.H, S.k, S.AHres, S.status, st);
    // Gbuf[0] now holds H^T H of the updated H (fused Gram of the H-half sweep)
    launch_residual(S.A, S.H, S.k, S.AHres, S.Gbuf[0], S.rpart, S.rgrid, S.rout, S.status, st);
    launch_pdl(record_resid, 1, 1, 0, st, S.iter_dev, S.first_iter, S.max_iters, S.rout, S.resid);
    // projected gradient of the SymNMF objective at the new H (App. D)
    float* AH = S.A.kind == SYMNMF_CSR ? S.AHres : S.AHpg;
    if (S.A.kind == SYMNMF_DENSE &&
        !enqueue_product(S.A, S.H, S.k, AH, S.precision, S.tcs, S.tcs_bytes, S.status, st))
      return false;
    launch_pgrad(S.H, AH, S.Gbuf[0], S.n, S.k, S.ppart, S.pgrid, S.pout, S.status, st);
    launch_pdl(record_resid, 1, 1, 0, st, S.iter_dev, S.first_iter, S.max_iters, S.pout, S.pgrad);
    mark(S, st, "residual");
  }
  launch_pdl(bump_iter, 1, 1, 0, st, S.iter_dev);
  mark(S, st, "bump_iter");
  return true;
}

}  // namespace

extern "C" symnmf_status symnmf_solver_create(symnmf_solver** out, const symnmf_matrix* A, int64_t n, float* W,
                                              float* H, int32_t k, double alpha, int32_t mode, int32_t precision,
                                              int64_t s, double tau, uint64_t seed, int32_t first_iter,
                                              int32_t max_iters, const float* U, const double* lambda, int32_t l,
                                              int32_t with_residual, void* ws, size_t* ws_bytes, cudaStream_t st) {
  if (n < 1 || !W || !H || bad_k(k) || !(alpha >= 0.0) || max_iters < 1 || first_iter < 0) return SYMNMF_ERR_ARG;
  const bool bpp = (mode & SYMNMF_RULE_BPP) != 0;
  const bool record = (mode & SYMNMF_RECORD_PLANS) != 0;
  mode &= ~(SYMNMF_RULE_BPP | SYMNMF_RECORD_PLANS);
  if (mode != SYMNMF_EXACT && mode != SYMNMF_LVS && mode != SYMNMF_LAI) return SYMNMF_ERR_ARG;
  if (bpp && !bpp_supported(k)) return SYMNMF_ERR_UNSUPPORTED;
  if (precision != SYMNMF_FP32 && precision != SYMNMF_3XTF32) return SYMNMF_ERR_ARG;
  const bool needA = mode != SYMNMF_LAI || with_residual;
  if (needA && (bad_matrix(A) || A->n != n)) return SYMNMF_ERR_ARG;
  if (A && !bad_matrix(A) && A->kind == SYMNMF_CSR && precision != SYMNMF_FP32) return SYMNMF_ERR_ARG;
  if (mode == SYMNMF_LVS && (s < 1 || !(tau > 0.0 && tau <= 1.0))) return SYMNMF_ERR_ARG;
  if (mode == SYMNMF_LAI && (!U || !lambda || l < 1 || l > kMaxL || l > n)) return SYMNMF_ERR_ARG;
  symnmf_solver S{};
  S.hasA = A && !bad_matrix(A);
  if (S.hasA) S.A = *A;
  S.n = n; S.W = W; S.H = H; S.k = k; S.alpha = alpha; S.mode = mode; S.precision = precision; S.bpp = bpp;
  S.record = record && mode == SYMNMF_LVS;
  S.s = mode == SYMNMF_LVS ? s : 0;
  S.T = tau * (double)k;   // reading Z1
  S.seed = seed; S.first_iter = first_iter; S.max_iters = max_iters;
  S.U = U; S.lam = lambda; S.l = l; S.with_resid = with_residual ? 1 : 0;
  Carver c(nullptr);
  solver_layout(S, c);
  bool q;
  symnmf_status r = ws_protocol(ws, ws_bytes, c.bytes(), &q);
  if (r != SYMNMF_OK || q) return r;
  if (!out) return SYMNMF_ERR_ARG;
  if (!device_ok()) return SYMNMF_ERR_UNSUPPORTED;
  Carver w(ws);
  solver_layout(S, w);
  S.status = ws_status(ws);
  SYMNMF_CUDA_TRY(cudaMemsetAsync(ws, 0, kWsHeader, st));
  if (mode == SYMNMF_LVS) SYMNMF_CUDA_TRY(cudaMemsetAsync(S.sw.cnt, 0, sizeof(int32_t) * n, st));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(S.stats, 0, sizeof(symnmf_half_stats) * 2 * max_iters, st));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(S.resid, 0, sizeof(double) * max_iters, st));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(S.counter, 0, sizeof(unsigned int) * 4, st));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(S.nonconv, 0, sizeof(int32_t), st));
  SYMNMF_CUDA_TRY(cudaMemsetAsync(S.Gacc, 0, sizeof(double) * kGramReplicas * k * k, st));
  if (S.mode == SYMNMF_LAI && S.lai_fused) {
    const size_t lp = (size_t)lai_lp(S.l);
    SYMNMF_CUDA_TRY(cudaMemsetAsync(S.UXacc, 0, sizeof(double) * lp * k * kGramReplicas, st));
    SYMNMF_CUDA_TRY(cudaMemsetAsync(S.Mside[0], 0, sizeof(float) * lp * k, st));
    SYMNMF_CUDA_TRY(cudaMemsetAsync(S.Mside[1], 0, sizeof(float) * lp * k, st));
    // Lambda U^T H for the first W-half; later halves get theirs from the preceding launch
    launch_cross_gram(S.U, S.l, S.l, H, k, k, false, n, nullptr, nullptr, nullptr, S.Zpart, S.ggrid, S.Z, k, S.status,
                      st);
    launch_scale_rows(S.Z, S.l, k, S.lam, S.Mside[0], S.status, st);
  }
  // LvS on CSR with the streaming sweep: the scatter accumulates onto Y = alpha F (the first half's
  // F is H) and each sweep leaves alpha X for the next half, so the sweep never reads F; the solver
  // keeps this state across run calls, as it keeps F^T F (W and H are the solver's between runs)
  S.yalpha = mode == SYMNMF_LVS && S.hasA && S.A.kind == SYMNMF_CSR && !S.bpp && sweep_stream_supported(k) &&
             sweep_stream_enabled(n) && yalpha_enabled();
  if (S.yalpha) launch_scale_copy(H, alpha, S.Y, n * k, st);
  else if (mode == SYMNMF_LVS && S.Y) SYMNMF_CUDA_TRY(cudaMemsetAsync(S.Y, 0, sizeof(float) * n * k, st));
  if (S.hasA && S.A.kind == SYMNMF_CSR) {
    // every sparse path assumes each row's columns sorted, unique and in range (the destination
    // ranges of the sampled scatter binary-search them)
    int32_t* bad = S.nonconv;
    SYMNMF_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int32_t), st));
    launch_csr_check(S.A, bad, st);
    int32_t hbad = 0;
    SYMNMF_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
    SYMNMF_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int32_t), st));
    if (hbad) return SYMNMF_ERR_ARG;
  }
  if (S.nnzsp) launch_spmm_nnz_rows(S.A, S.chunk_row, st);
  if (S.ppos) launch_sampled_pass_bounds(S.A, k, S.ppos, st);
  set_i32<<<1, 1, 0, st>>>(S.iter_dev, first_iter);
  // H^T H (and its CholeskyQR factor for LvS) for the first W-half; later halves get
  // theirs from the fused Gram of the preceding sweep.
  launch_gram_fused(H, n, k, S.Gacc, S.Gbuf[0], mode == SYMNMF_LVS ? S.Rinv32 : nullptr, S.counter, S.status, st);
  if (finish() != SYMNMF_OK) return SYMNMF_ERR_CUDA;
  // Capture one iteration on a private stream (the caller's may be the legacy default stream).
  // Every failure from here on releases what was created (release_solver_resources).
  S.cslot = (sweep_stream_supported(k) && sweep_stream_enabled(n) && sweep_cmem_enabled()) ? sweep_cslot_acquire() : -1;
  symnmf_status rs = SYMNMF_OK;
  cudaStream_t cs = nullptr;
  cudaGraph_t g = nullptr;
  bool ok = false;
  cudaError_t ce = cudaSuccess;
  if (cudaStreamCreateWithFlags(&S.side, cudaStreamNonBlocking) != cudaSuccess) rs = SYMNMF_ERR_CUDA;
  for (int h = 0; h < 2 && rs == SYMNMF_OK; ++h) {
    if (cudaEventCreateWithFlags(&S.ev_fork[h], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&S.ev_join[h], cudaEventDisableTiming) != cudaSuccess)
      rs = SYMNMF_ERR_CUDA;
  }
  if (rs == SYMNMF_OK && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) rs = SYMNMF_ERR_CUDA;
  if (rs == SYMNMF_OK) {
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      rs = SYMNMF_ERR_CUDA;
    } else {
      {
        pdl_scope pdl(S.n < (1ll << 15));   // common.cuh: PDL edges pay only for the small problems
        ok = enqueue_iteration(S, cs);
      }
      ce = cudaStreamEndCapture(cs, &g);
      if (!ok) rs = SYMNMF_ERR_UNSUPPORTED;
      else if (ce != cudaSuccess || !g) rs = SYMNMF_ERR_CUDA;
    }
  }
  if (cs) cudaStreamDestroy(cs);
  if (rs == SYMNMF_OK && cudaGraphInstantiate(&S.exec, g, 0) != cudaSuccess) rs = SYMNMF_ERR_CUDA;
  S.graph = g;
  S.iters_done = 0;
  symnmf_solver* p = nullptr;
  if (rs == SYMNMF_OK) {
    p = new (std::nothrow) symnmf_solver(S);
    if (!p) rs = SYMNMF_ERR_ARG;
  }
  if (rs != SYMNMF_OK) {
    (void)cudaGetLastError();
    release_solver_resources(S);
    return rs;
  }
  *out = p;
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_solver_run(symnmf_solver* S, int32_t iters, cudaStream_t st) {
  if (!S || iters < 0) return SYMNMF_ERR_ARG;
  for (int t = 0; t < iters; ++t) SYMNMF_CUDA_TRY(cudaGraphLaunch(S->exec, st));
  S->iters_done += iters;
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_solver_run_until(symnmf_solver* S, int32_t max_iters, double tol, int32_t patience,
                                                 int32_t* iters_run_host, cudaStream_t st) {
  // NEXT-3 stopping rule (reading Z30): stop once the normalised residual has failed to
  // decrease by more than tol for `patience` consecutive iterations.  One residual read-back
  // (8 bytes, a stream synchronisation) per iteration.
  if (!S || max_iters < 0 || !(tol >= 0.0) || patience < 1 || !S->with_resid) return SYMNMF_ERR_ARG;
  int32_t run = 0, done = 0;
  double prev = 0.0;
  for (int32_t t = 0; t < max_iters; ++t) {
    const int32_t slot = S->iters_done;
    if (slot >= S->max_iters) break;
    SYMNMF_CUDA_TRY(cudaGraphLaunch(S->exec, st));
    S->iters_done += 1;
    ++done;
    double r = 0.0;
    SYMNMF_CUDA_TRY(cudaMemcpyAsync(&r, S->resid + slot, sizeof(double), cudaMemcpyDeviceToHost, st));
    SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
    if (t > 0) {
      run = (prev - r <= tol) ? run + 1 : 0;
      if (run >= patience) break;
    }
    prev = r;
  }
  if (iters_run_host) *iters_run_host = done;
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_solve(const symnmf_matrix* A, int64_t n, float* W, float* H, int32_t k,
                                      double alpha, int32_t mode, int32_t precision, int64_t s, double tau,
                                      uint64_t seed, const float* U, const double* lambda, int32_t l,
                                      int32_t max_iters, double tol, int32_t patience, int32_t refine,
                                      int32_t* iters_host, double* resid_host, void* ws, size_t* ws_bytes,
                                      cudaStream_t st) {
  // NEXT-2/3 driver: `mode` iterations until the P:1086 stopping rule, then (refine = 1, the
  // Iterative Refinement of P:557-563 / P:1088) EXACT iterations on the full A until the same
  // rule.  Both phases reuse one workspace (the first solver is destroyed before the second).
  if (!A || max_iters < 1 || patience < 1 || !(tol >= 0.0) || (refine && bad_matrix(A))) return SYMNMF_ERR_ARG;
  const int32_t prec2 = (A && !bad_matrix(A) && A->kind == SYMNMF_CSR) ? SYMNMF_FP32 : precision;
  size_t b1 = 0, b2 = 0;
  symnmf_status r = symnmf_solver_create(nullptr, A, n, W, H, k, alpha, mode, precision, s, tau, seed, 0, max_iters,
                                         U, lambda, l, 1, nullptr, &b1, st);
  if (r != SYMNMF_OK) return r;
  if (refine) {
    r = symnmf_solver_create(nullptr, A, n, W, H, k, alpha, SYMNMF_EXACT | (mode & SYMNMF_RULE_BPP), prec2, 0, 1.0,
                             seed, 0, max_iters, nullptr, nullptr, 0, 1, nullptr, &b2, st);
    if (r != SYMNMF_OK) return r;
  }
  bool q;
  r = ws_protocol(ws, ws_bytes, std::max(b1, b2), &q);
  if (r != SYMNMF_OK || q) return r;
  int32_t ran[2] = {0, 0};
  for (int phase = 0; phase < (refine ? 2 : 1); ++phase) {
    symnmf_solver* S = nullptr;
    size_t bytes = *ws_bytes;
    r = phase == 0 ? symnmf_solver_create(&S, A, n, W, H, k, alpha, mode, precision, s, tau, seed, 0, max_iters, U,
                                          lambda, l, 1, ws, &bytes, st)
                   : symnmf_solver_create(&S, A, n, W, H, k, alpha, SYMNMF_EXACT | (mode & SYMNMF_RULE_BPP), prec2, 0,
                                          1.0, seed, 0, max_iters, nullptr, nullptr, 0, 1, ws, &bytes, st);
    if (r != SYMNMF_OK) return r;
    r = symnmf_solver_run_until(S, max_iters, tol, patience, &ran[phase], st);
    if (r == SYMNMF_OK)
      r = symnmf_solver_stats(S, nullptr, nullptr, resid_host ? resid_host + (size_t)phase * max_iters : nullptr, st);
    symnmf_solver_destroy(S);
    if (r != SYMNMF_OK) return r;
  }
  if (iters_host) { iters_host[0] = ran[0]; iters_host[1] = ran[1]; }
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_solver_pgrad(symnmf_solver* S, double* pgrad_host, cudaStream_t st) {
  if (!S || !pgrad_host || !S->with_resid) return SYMNMF_ERR_ARG;
  const int32_t m = std::min(S->iters_done, S->max_iters);
  if (m > 0)
    SYMNMF_CUDA_TRY(cudaMemcpyAsync(pgrad_host, S->pgrad, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_solver_last_plan(const symnmf_solver* S, float* lev_out, int32_t* uniq_idx_out,
                                                 double* uniq_w_out, int64_t* counts_out, double* mass_out,
                                                 cudaStream_t st) {
  if (!S || S->mode != SYMNMF_LVS || !lev_out || !uniq_idx_out || !uniq_w_out || !counts_out || !mass_out)
    return SYMNMF_ERR_ARG;
  const size_t n = (size_t)S->n;
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(lev_out, S->lev, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(uniq_idx_out, S->plan.uniq_idx, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(uniq_w_out, S->plan.uniq_w, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(counts_out, S->plan.counts, sizeof(int64_t) * 4, cudaMemcpyDeviceToDevice, st));
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(mass_out, S->plan.mass, sizeof(double) * 2, cudaMemcpyDeviceToDevice, st));
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_solver_plan_history(const symnmf_solver* S, int32_t t, int32_t side, float* lev_out,
                                                    int32_t* uniq_idx_out, double* uniq_w_out, int64_t* counts_out,
                                                    double* mass_out, cudaStream_t st) {
  if (!S || !S->record || !lev_out || !uniq_idx_out || !uniq_w_out || !counts_out || !mass_out) return SYMNMF_ERR_ARG;
  if (t < 0 || t >= std::min(S->iters_done, S->max_iters) || (side != 0 && side != 1)) return SYMNMF_ERR_ARG;
  const size_t h = (size_t)2 * t + side, n = (size_t)S->n, cap = (size_t)S->plan.cap;
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(lev_out, S->hlev + h * n, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(uniq_idx_out, S->huniq + h * cap, sizeof(int32_t) * cap, cudaMemcpyDeviceToDevice, st));
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(uniq_w_out, S->hw + h * cap, sizeof(double) * cap, cudaMemcpyDeviceToDevice, st));
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(counts_out, S->hcounts + h * 4, sizeof(int64_t) * 4, cudaMemcpyDeviceToDevice, st));
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(mass_out, S->hmass + h * 2, sizeof(double) * 2, cudaMemcpyDeviceToDevice, st));
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_solver_stats(symnmf_solver* S, int32_t* iters_done_host, symnmf_half_stats* stats_host,
                                             double* resid_host, cudaStream_t st) {
  if (!S) return SYMNMF_ERR_ARG;
  const int32_t m = std::min(S->iters_done, S->max_iters);
  int32_t status = 0;
  SYMNMF_CUDA_TRY(cudaMemcpyAsync(&status, S->status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (stats_host && m > 0)
    SYMNMF_CUDA_TRY(cudaMemcpyAsync(stats_host, S->stats, sizeof(symnmf_half_stats) * 2 * m, cudaMemcpyDeviceToHost, st));
  if (resid_host && m > 0)
    SYMNMF_CUDA_TRY(cudaMemcpyAsync(resid_host, S->resid, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
  if (iters_done_host) *iters_done_host = S->iters_done;
  return (symnmf_status)status;
}

extern "C" symnmf_status symnmf_solver_destroy(symnmf_solver* S) {
  if (!S) return SYMNMF_ERR_ARG;
  release_solver_resources(*S);
  delete S;
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_solver_profile(symnmf_solver* S, int32_t iters, int32_t cap,
                                               char (*names_host)[48], float* ms_host, int32_t* count_host,
                                               cudaStream_t st) {
  if (!S || iters < 1 || cap < 1 || !names_host || !ms_host || !count_host) return SYMNMF_ERR_ARG;
  symnmf_solver::Prof prof;
  prof.n = 0;
  for (int i = 0; i <= symnmf_solver::Prof::kMax; ++i) SYMNMF_CUDA_TRY(cudaEventCreate(&prof.ev[i]));
  std::vector<double> acc;
  int sites = 0;
  for (int it = 0; it < iters; ++it) {
    // keep the device busy while the host enqueues the instrumented iteration
    spin_kernel<<<1, 1, 0, st>>>(200000);
    prof.n = 0;
    cudaEventRecord(prof.ev[0], st);
    S->prof = &prof;
    const bool ok = enqueue_iteration(*S, st);
    S->prof = nullptr;
    if (!ok) break;
    SYMNMF_CUDA_TRY(cudaStreamSynchronize(st));
    sites = prof.n;
    acc.resize(sites, 0.0);
    for (int i = 0; i < sites; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, prof.ev[i], prof.ev[i + 1]);
      acc[i] += ms;
    }
  }
  S->iters_done += iters;
  const int m = std::min(sites, (int)cap);
  for (int i = 0; i < m; ++i) {
    std::snprintf(names_host[i], 48, "%s", prof.name[i]);
    ms_host[i] = (float)(acc[i] / iters);
  }
  *count_host = m;
  for (int i = 0; i <= symnmf_solver::Prof::kMax; ++i) cudaEventDestroy(prof.ev[i]);
  return finish();
}

extern "C" symnmf_status symnmf_solver_graph_nodes(const symnmf_solver* S, int32_t* kernels_host,
                                                   int32_t* memsets_host) {
  if (!S || !S->graph) return SYMNMF_ERR_ARG;
  size_t nn = 0;
  SYMNMF_CUDA_TRY(cudaGraphGetNodes(S->graph, nullptr, &nn));
  cudaGraphNode_t* nodes = new (std::nothrow) cudaGraphNode_t[nn ? nn : 1];
  if (!nodes) return SYMNMF_ERR_ARG;
  if (cudaGraphGetNodes(S->graph, nodes, &nn) != cudaSuccess) { delete[] nodes; return SYMNMF_ERR_CUDA; }
  int32_t kc = 0, mc = 0;
  for (size_t i = 0; i < nn; ++i) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nodes[i], &t) != cudaSuccess) continue;
    if (t == cudaGraphNodeTypeKernel) ++kc;
    if (t == cudaGraphNodeTypeMemset) ++mc;
  }
  delete[] nodes;
  if (kernels_host) *kernels_host = kc;
  if (memsets_host) *memsets_host = mc;
  return SYMNMF_OK;
}

extern "C" symnmf_status symnmf_iterate(const symnmf_matrix* A, int64_t n, float* W, float* H, int32_t k, double alpha,
                                        int32_t mode, int32_t precision, int64_t s, double tau, uint64_t seed,
                                        int32_t first_iter, int32_t iters, const float* U, const double* lambda,
                                        int32_t l, symnmf_half_stats* stats_host, double* resid_host, void* ws,
                                        size_t* ws_bytes, cudaStream_t st) {
  if (iters < 1) return SYMNMF_ERR_ARG;
  symnmf_solver* S = nullptr;
  symnmf_status r = symnmf_solver_create(&S, A, n, W, H, k, alpha, mode, precision, s, tau, seed, first_iter, iters, U,
                                         lambda, l, resid_host ? 1 : 0, ws, ws_bytes, st);
  if (r != SYMNMF_OK || !ws) return r;
  r = symnmf_solver_run(S, iters, st);
  if (r == SYMNMF_OK) r = symnmf_solver_stats(S, nullptr, stats_host, resid_host, st);
  symnmf_solver_destroy(S);
  return r;
}
