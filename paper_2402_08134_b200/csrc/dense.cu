// Dense SIMT products (precision SYMNMF_FP32):
//  (a10) Y = A F for dense A -- the fp32 reference-precision path and
//        the product for widths the tensor-core kernel does not cover;
//  (a9)  Y_s = A[U,:]^T (omega o F[U,:]) (sampled rows of A gathered
//        row by row: with symmetry A[U,:]^T = A[:,U], Z28).
// Accumulation: fp32 FMAs over a K tile, flushed into fp64 registers every
// 256 (product) / 32 (sampled) terms, so the long-K sums stay well inside the
// 1e-5 fp32 tolerance.  Split-K over gridDim.y with fp32 atomics into a
// zeroed Y when one wave would leave SMs idle.
#include "kernels.cuh"

namespace symnmf {

constexpr int DBM = 128;  // rows per CTA
constexpr int DBK = 32;   // K tile
constexpr int DTH = 256;

template <int KP, int TX, int CPT>
__global__ void __launch_bounds__(DTH) dense_ah_simt(const float* __restrict__ A, int64_t lda, int64_t n,
                                                     const float* __restrict__ F, int64_t ldf, int k,
                                                     float* __restrict__ Y, int64_t ldy, int64_t kchunk, int atomic,
                                                     const int32_t* __restrict__ status) {
  constexpr int TY = DTH / TX;
  constexpr int RM = DBM / TY;
  __shared__ float sA[DBK][DBM + 1];
  __shared__ __align__(16) float sF[DBK][KP];
  if (dev_failed(status)) return;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int64_t m0 = (int64_t)blockIdx.x * DBM;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk, kend = min64(n, kbeg + kchunk);
  float acc[RM][CPT];
  double acc64[RM][CPT];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < CPT; ++j) { acc[i][j] = 0.f; acc64[i][j] = 0.0; }
  int tiles_since = 0;
  for (int64_t k0 = kbeg; k0 < kend; k0 += DBK) {
    __syncthreads();
    for (int e = tid; e < DBM * DBK; e += DTH) {
      const int r = e / DBK, c = e - r * DBK;
      const int64_t gr = m0 + r, gc = k0 + c;
      sA[c][r] = (gr < n && gc < kend) ? A[gr * lda + gc] : 0.f;
    }
    for (int e = tid; e < DBK * KP; e += DTH) {
      const int r = e / KP, c = e - r * KP;
      const int64_t gr = k0 + r;
      sF[r][c] = (gr < kend && c < k) ? F[gr * ldf + c] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < DBK; ++kk) {
      float a[RM], b[CPT];
#pragma unroll
      for (int i = 0; i < RM; ++i) a[i] = sA[kk][ty + TY * i];
#pragma unroll
      for (int j = 0; j < CPT; ++j) b[j] = sF[kk][tx * CPT + j];
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < CPT; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (++tiles_since == 8) {
      tiles_since = 0;
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < CPT; ++j) { acc64[i][j] += (double)acc[i][j]; acc[i][j] = 0.f; }
    }
  }
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int64_t gr = m0 + ty + TY * i;
    if (gr >= n) continue;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = tx * CPT + j;
      if (c >= k) continue;
      const float v = (float)(acc64[i][j] + (double)acc[i][j]);
      if (atomic) atomicAdd(Y + gr * ldy + c, v);
      else Y[gr * ldy + c] = v;
    }
  }
}

template <int KP, int TX, int CPT>
static void launch_dense_t(const float* A, int64_t lda, int64_t n, const float* F, int64_t ldf, int k, float* Y,
                           int64_t ldy, const int32_t* status, cudaStream_t st) {
  const int64_t mt = (n + DBM - 1) / DBM;
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>(16, (148 * 4 + mt - 1) / mt));
  int64_t kchunk = (n + splits - 1) / splits;
  kchunk = (kchunk + DBK - 1) / DBK * DBK;
  splits = (n + kchunk - 1) / kchunk;
  if (splits > 1) cudaMemset2DAsync(Y, sizeof(float) * ldy, 0, sizeof(float) * k, n, st);
  dim3 grid((unsigned)mt, (unsigned)splits);
  dense_ah_simt<KP, TX, CPT><<<grid, DTH, 0, st>>>(A, lda, n, F, ldf, k, Y, ldy, kchunk, splits > 1 ? 1 : 0, status);
}

void launch_dense_ah_simt(const float* A, int64_t lda, int64_t n, const float* F, int64_t ldf, int k, float* Y,
                          int64_t ldy, const int32_t* status, cudaStream_t st) {
  if (k <= 8) launch_dense_t<8, 2, 4>(A, lda, n, F, ldf, k, Y, ldy, status, st);
  else if (k <= 16) launch_dense_t<16, 4, 4>(A, lda, n, F, ldf, k, Y, ldy, status, st);
  else if (k <= 32) launch_dense_t<32, 8, 4>(A, lda, n, F, ldf, k, Y, ldy, status, st);
  else if (k <= 64) launch_dense_t<64, 16, 4>(A, lda, n, F, ldf, k, Y, ldy, status, st);
  else if (k <= 80) launch_dense_t<80, 16, 5>(A, lda, n, F, ldf, k, Y, ldy, status, st);
  else launch_dense_t<96, 16, 6>(A, lda, n, F, ldf, k, Y, ldy, status, st);
}

// ---------------------------------------------------------------- sampled dense
// Thread = output row c (a column of A[U,:]); the CTA walks the sampled rows
// U in chunks of 32, staging omega_u F[U_u, :] in shared memory, reading
// A[U_u, c0 .. c0+127] coalesced.  gridDim.y splits U (atomics into zeroed Y).
template <int KP>
__global__ void __launch_bounds__(128) sampled_dense_kernel(const float* __restrict__ A, int64_t lda, int64_t n,
                                                            const float* __restrict__ F, int k,
                                                            const int32_t* __restrict__ uniq,
                                                            const double* __restrict__ w,
                                                            const int64_t* __restrict__ n_uniq_dev,
                                                            float* __restrict__ Y, const int32_t* __restrict__ status) {
  __shared__ __align__(16) float sFw[32][KP];
  __shared__ int64_t sRow[32];
  if (dev_failed(status)) return;
  const int tid = threadIdx.x;
  const int64_t c = (int64_t)blockIdx.x * 128 + tid;
  const int64_t nu = *n_uniq_dev;
  const int64_t per = (nu + gridDim.y - 1) / gridDim.y;
  const int64_t u0 = (int64_t)blockIdx.y * per, u1 = min(nu, u0 + per);
  float acc[KP];
  double acc64[KP];
#pragma unroll
  for (int j = 0; j < KP; ++j) { acc[j] = 0.f; acc64[j] = 0.0; }
  for (int64_t ub = u0; ub < u1; ub += 32) {
    const int cnt = (int)min64(32, u1 - ub);
    __syncthreads();
    if (tid < 32) sRow[tid] = tid < cnt ? (int64_t)uniq[ub + tid] : 0;
    __syncthreads();
    for (int e = tid; e < 32 * KP; e += 128) {
      const int r = e / KP, j = e - r * KP;
      sFw[r][j] = (r < cnt && j < k) ? (float)w[ub + r] * F[sRow[r] * k + j] : 0.f;
    }
    __syncthreads();
    if (c < n) {
      float a[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) a[r] = r < cnt ? __ldg(A + sRow[r] * lda + c) : 0.f;
#pragma unroll
      for (int r = 0; r < 32; ++r)
#pragma unroll
        for (int j = 0; j < KP; ++j) acc[j] = fmaf(a[r], sFw[r][j], acc[j]);
#pragma unroll
      for (int j = 0; j < KP; ++j) { acc64[j] += (double)acc[j]; acc[j] = 0.f; }
    }
  }
  if (c < n) {
    const bool atomic = gridDim.y > 1;
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      if (j >= k) break;
      const float v = (float)acc64[j];
      if (atomic) atomicAdd(Y + c * k + j, v);
      else Y[c * k + j] = v;
    }
  }
}

template <int KP>
static void launch_sd_t(const float* A, int64_t lda, int64_t n, const float* F, int k, const int32_t* uniq,
                        const double* w, const int64_t* nu, int64_t cap, float* Y, const int32_t* status,
                        cudaStream_t st) {
  const int64_t cb = (n + 127) / 128;
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>((148 * 8 + cb - 1) / cb, (cap + 127) / 128));
  if (splits > 1) cudaMemsetAsync(Y, 0, sizeof(float) * n * k, st);
  sampled_dense_kernel<KP><<<dim3((unsigned)cb, (unsigned)splits), 128, 0, st>>>(A, lda, n, F, k, uniq, w, nu, Y,
                                                                                 status);
}

void launch_sampled_dense(const float* A, int64_t lda, int64_t n, const float* F, int k, const int32_t* uniq,
                          const double* w, const int64_t* n_uniq_dev, int64_t cap, float* Y, const int32_t* status,
                          cudaStream_t st) {
  switch (kpad(k)) {
    case 8: launch_sd_t<8>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, Y, status, st); break;
    case 16: launch_sd_t<16>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, Y, status, st); break;
    case 32: launch_sd_t<32>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, Y, status, st); break;
    default: launch_sd_t<64>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, Y, status, st); break;
  }
}

}  // namespace symnmf
