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
// Y_s[c, :] = sum_u A[U_u, c] (omega_u F[U_u, :])  (A[U,:]^T = A[:,U] by symmetry, Z28).
// CTA tile: 128 output rows c x KP columns; thread = 4 rows c (one float4 of each gathered row of
// A) x JB columns.  The CTA's range of U (indices and weights) is loaded into shared memory
// once; the gathered SDU x 128 slabs of A and the SDU raw rows F[U_u, :] then stream through an
// SDS-stage cp.async ring, so no load on the critical path depends on another; omega_u scales
// the staged F rows once per stage.  fp32 FMAs, flushed into fp64 registers every stage.  gridDim.y splits U
// (fp32 atomics into a zeroed Y) so that the grid fills the SMs.
constexpr int SDC = 128;    // output rows per CTA
constexpr int SDS = 4;      // pipeline stages
constexpr int SDUMAX = 2048;   // U entries per CTA (indices + weights in shared memory)

template <int KP, int JB, int SDU>   // SDU sampled rows per stage
struct SdSmem {
  static constexpr size_t a = 0;                                              // float [SDS][SDU][SDC]
  static constexpr size_t f = a + sizeof(float) * SDS * SDU * SDC;            // float [SDS][SDU][KP]
  static constexpr size_t row = f + sizeof(float) * SDS * SDU * KP;           // int64 [SDUMAX]
  static constexpr size_t w = row + sizeof(int64_t) * SDUMAX;                 // float [SDUMAX]
  static constexpr size_t bytes = w + sizeof(float) * SDUMAX;
};

template <int KP, int JB, int SDU>
__global__ void __launch_bounds__(32 * (KP / JB), 2) sampled_dense_v3(const float* __restrict__ A, int64_t lda, int64_t n,
                                                                  const float* __restrict__ F, int k,
                                                                  const int32_t* __restrict__ uniq,
                                                                  const double* __restrict__ w,
                                                                  const int64_t* __restrict__ n_uniq_dev,
                                                                  float* __restrict__ Y, int vec,
                                                                  const int32_t* __restrict__ status) {
  using L = SdSmem<KP, JB, SDU>;
  constexpr int NT = 32 * (KP / JB);
  extern __shared__ __align__(16) unsigned char sds[];
  float* sA = reinterpret_cast<float*>(sds + L::a);
  float* sF = reinterpret_cast<float*>(sds + L::f);
  int64_t* sRow = reinterpret_cast<int64_t*>(sds + L::row);
  float* sW = reinterpret_cast<float*>(sds + L::w);
  if (dev_failed(status)) return;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * SDC;
  const int64_t nu = *n_uniq_dev;
  const int64_t per = ((nu + gridDim.y - 1) / gridDim.y + SDU - 1) / SDU * SDU;
  const int64_t u0 = (int64_t)blockIdx.y * per, u1 = min64(nu, u0 + per);
  if (u0 >= u1) return;
  float acc[4][JB];
  double acc64[4][JB];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < JB; ++j) { acc[i][j] = 0.f; acc64[i][j] = 0.0; }
  // the CTA's U range in chunks of SDUMAX entries (indices + weights staged once per chunk)
  for (int64_t cu0 = u0; cu0 < u1; cu0 += SDUMAX) {
    const int cnt = (int)min64(SDUMAX, u1 - cu0);
    __syncthreads();
    for (int e = tid; e < ((cnt + SDU - 1) / SDU) * SDU; e += NT) {
      const bool ok = e < cnt;
      sRow[e] = ok ? (int64_t)__ldg(uniq + cu0 + e) : -1;
      sW[e] = ok ? (float)__ldg(w + cu0 + e) : 0.f;
    }
    __syncthreads();
    const int nst = (cnt + SDU - 1) / SDU;
    auto issue = [&](int s) {
      if (s < nst) {
        const int buf = s % SDS;
        float* a = sA + (size_t)buf * SDU * SDC;
        for (int e = tid; e < SDU * (SDC / 4); e += NT) {
          const int r = e / (SDC / 4), q = e - r * (SDC / 4);
          const int64_t row = sRow[s * SDU + r];
          const int64_t c = c0 + 4 * q;
          float* dst = a + r * SDC + 4 * q;
          if (vec) {
            const bool ok = row >= 0 && c < n;
            cp_async16(dst, ok ? (const void*)(A + row * lda + c) : (const void*)A, ok);
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) dst[t] = (row >= 0 && c + t < n) ? __ldg(A + row * lda + c + t) : 0.f;
          }
        }
        float* f = sF + (size_t)buf * SDU * KP;
        if (k == KP) {
          for (int e = tid; e < SDU * (KP / 4); e += NT) {
            const int r = e / (KP / 4), q = e - r * (KP / 4);
            const int64_t row = sRow[s * SDU + r];
            cp_async16(f + r * KP + 4 * q, row >= 0 ? (const void*)(F + row * KP + 4 * q) : (const void*)F, row >= 0);
          }
        } else {
          for (int e = tid; e < SDU * KP; e += NT) {
            const int r = e / KP, j = e - r * KP;
            const int64_t row = sRow[s * SDU + r];
            f[r * KP + j] = (row >= 0 && j < k) ? __ldg(F + row * k + j) : 0.f;
          }
        }
      }
      cp_async_commit();   // (possibly empty) group per stage keeps the wait count uniform
    };
#pragma unroll
    for (int s = 0; s < SDS - 1; ++s) issue(s);
    for (int s = 0; s < nst; ++s) {
      issue(s + SDS - 1);
      cp_async_wait<SDS - 1>();
      __syncthreads();
      const int buf = s % SDS;
      const float* a = sA + (size_t)buf * SDU * SDC;
      float* fs = sF + (size_t)buf * SDU * KP;
      for (int e = tid; e < SDU * KP; e += NT) fs[e] *= sW[s * SDU + e / KP];   // omega_u F[U_u, :], once
      __syncthreads();
      const float* f = fs;
#pragma unroll 4
      for (int r = 0; r < SDU; ++r) {
        const float4 a4 = *reinterpret_cast<const float4*>(a + r * SDC + 4 * tx);
        float fv[JB];
#pragma unroll
        for (int j = 0; j < JB; j += 4) {
          const float4 v = *reinterpret_cast<const float4*>(f + r * KP + ty * JB + j);
          fv[j] = v.x; fv[j + 1] = v.y; fv[j + 2] = v.z; fv[j + 3] = v.w;
        }
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < JB; ++j) acc[i][j] = fmaf(av[i], fv[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < JB; ++j) { acc64[i][j] += (double)acc[i][j]; acc[i][j] = 0.f; }
      __syncthreads();   // buffer `buf` is refilled by a later issue()
    }
    cp_async_wait<0>();
  }
  const bool atomic = gridDim.y > 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t c = c0 + 4 * tx + i;
    if (c >= n) continue;
#pragma unroll
    for (int j = 0; j < JB; ++j) {
      const int jj = ty * JB + j;
      if (jj >= k) continue;
      const float v = (float)acc64[i][j];
      if (atomic) atomicAdd(Y + c * k + jj, v);
      else Y[c * k + jj] = v;
    }
  }
}

template <int KP, int JB, int SDU = (KP == 64 ? 16 : 32)>
static void launch_sd_t(const float* A, int64_t lda, int64_t n, const float* F, int k, const int32_t* uniq,
                        const double* w, const int64_t* nu, int64_t cap, float* Y, const int32_t* status,
                        cudaStream_t st) {
  using L = SdSmem<KP, JB, SDU>;
  const int64_t cb = (n + SDC - 1) / SDC;
  cudaFuncSetAttribute(sampled_dense_v3<KP, JB, SDU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sampled_dense_v3<KP, JB, SDU>, 32 * (KP / JB), L::bytes);
  const int64_t slots = 148 * (int64_t)std::max(1, occ);
  // U splits: whole waves of CTAs (the sampled rows are the long K dimension), at most what the
  // expected |U| <= min(cap, n) keeps busy with >= 4 stages per CTA
  int64_t splits = 1;
  double best = 0.0;
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(16, (cap + 4 * SDU - 1) / (4 * SDU)));
  for (int64_t sp = 1; sp <= smax; ++sp) {
    const int64_t ctas = cb * sp, waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots) * (1.0 - 0.01 * (double)sp);
    if (eff > best + 1e-9) { best = eff; splits = sp; }
  }
  if (splits > 1) cudaMemsetAsync(Y, 0, sizeof(float) * n * k, st);
  const int vec = (lda % 4 == 0 && n % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) ? 1 : 0;
  sampled_dense_v3<KP, JB, SDU><<<dim3((unsigned)cb, (unsigned)splits), 32 * (KP / JB), L::bytes, st>>>(
      A, lda, n, F, k, uniq, w, nu, Y, vec, status);
}

void launch_sampled_dense(const float* A, int64_t lda, int64_t n, const float* F, int k, const int32_t* uniq,
                          const double* w, const int64_t* n_uniq_dev, int64_t cap, float* Y, const int32_t* status,
                          cudaStream_t st) {
  switch (kpad(k)) {
    case 8: launch_sd_t<8, 4>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, Y, status, st); break;
    case 16: launch_sd_t<16, 4>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, Y, status, st); break;
    case 32: launch_sd_t<32, 4>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, Y, status, st); break;
    default: launch_sd_t<64, 8>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, Y, status, st); break;
  }
}

}  // namespace symnmf
