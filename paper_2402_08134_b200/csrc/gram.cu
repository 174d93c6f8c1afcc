// (a1) Gram F^T F, (a8) weighted sampled Gram, the cross products U^T F / Q^T Z of
// the LAI path, and (a2) the one-CTA fp64 Cholesky + triangular inverse of
// CholeskyQR.
//
// Layout: F is n x k fp32 row-major; a CTA stages GTR rows in shared memory
// (coalesced: a tile of consecutive rows is one contiguous run of k*GTR
// floats), each thread owns 4x4 register blocks of the k x k output (upper
// blocks only when symmetric), accumulates a tile in fp32 and flushes into
// fp64 registers every ~64 rows, then the CTA writes one fp64 partial; a
// one-CTA finalize sums the partials in fixed order (deterministic).
#include "kernels.cuh"

namespace symnmf {

constexpr int GT = 256;   // threads per CTA
constexpr int GTR = 32;   // rows per staged tile

__device__ __forceinline__ void pair_to_blocks(int p, int nba, int nbb, int sym, int& ai, int& bi) {
  if (!sym) { ai = p / nbb; bi = p - ai * nbb; return; }
  int a = 0, rem = p;
  while (rem >= nba - a) { rem -= nba - a; ++a; }
  ai = a; bi = a + rem;
}

template <int PPT, bool F64P>
__global__ void __launch_bounds__(GT) cross_gram_partial(
    const float* __restrict__ A, int64_t lda, int ka, const float* __restrict__ B, int64_t ldb, int kb, int sym,
    int64_t nrows, const int64_t* __restrict__ nrows_dev, const int32_t* __restrict__ gather,
    const double* __restrict__ wts, double* __restrict__ partial, const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smraw[];
  if (dev_failed(status)) return;
  const int tid = threadIdx.x;
  const int nba = (ka + 3) >> 2, nbb = (kb + 3) >> 2;
  const int pairs = sym ? nba * (nba + 1) / 2 : nba * nbb;
  const int sta = nba * 4 + 4, stb = nbb * 4 + 4;
  float* sa = reinterpret_cast<float*>(smraw);
  float* sb = sym ? sa : sa + GTR * sta;
  float* sw = sa + GTR * sta + (sym ? 0 : GTR * stb);
  const int64_t nr = nrows_dev ? *nrows_dev : nrows;
  const int64_t tiles = (nr + GTR - 1) / GTR;
  const int64_t tpc = (tiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = blockIdx.x * tpc, t1 = min(tiles, t0 + tpc);

  int RG, g, p0;
  if (pairs <= GT) { RG = GT / pairs; g = tid / pairs; p0 = tid - g * pairs; }
  else { RG = 1; g = 0; p0 = tid; }
  const bool active = g < RG;
  int ai[PPT], bi[PPT];
  bool pv[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int p = p0 + q * GT;
    pv[q] = active && p < pairs && (q == 0 || pairs > GT);
    if (pv[q]) pair_to_blocks(p, nba, nbb, sym, ai[q], bi[q]); else { ai[q] = 0; bi[q] = 0; }
  }
  float acc[PPT][16];
  double acc64[PPT][16];
#pragma unroll
  for (int q = 0; q < PPT; ++q)
#pragma unroll
    for (int e = 0; e < 16; ++e) { acc[q][e] = 0.f; acc64[q][e] = 0.0; }
  const int rows_per_tile = (GTR + RG - 1) / RG;
  int since_flush = 0;

  for (int64_t t = t0; t < t1; ++t) {
    __syncthreads();
    const int64_t rbase = t * GTR;
    const int wa = nba * 4;
    for (int e = tid; e < GTR * wa; e += GT) {
      const int r = e / wa, c = e - r * wa;
      const int64_t idx = rbase + r;
      float v = 0.f;
      if (c < ka && idx < nr) {
        const int64_t row = gather ? (int64_t)gather[idx] : idx;
        v = A[row * lda + c];
      }
      sa[r * sta + c] = v;
    }
    if (!sym) {
      const int wb = nbb * 4;
      for (int e = tid; e < GTR * wb; e += GT) {
        const int r = e / wb, c = e - r * wb;
        const int64_t idx = rbase + r;
        float v = 0.f;
        if (c < kb && idx < nr) {
          const int64_t row = gather ? (int64_t)gather[idx] : idx;
          v = B[row * ldb + c];
        }
        sb[r * stb + c] = v;
      }
    }
    if (tid < GTR) {
      const int64_t idx = rbase + tid;
      sw[tid] = idx < nr ? (wts ? (float)wts[idx] : 1.f) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      if (!pv[q]) continue;
      for (int r = g; r < GTR; r += RG) {
        const float w = sw[r];
        const float4 a4 = *reinterpret_cast<const float4*>(sa + r * sta + 4 * ai[q]);
        const float4 b4 = *reinterpret_cast<const float4*>(sb + r * stb + 4 * bi[q]);
        if constexpr (F64P) {   // exact products (fp32 inputs), fp64 sums: Grams whose small
                                // eigenvalues matter (CholeskyQR of the range finder's sketches)
          const double a[4] = {(double)a4.x * w, (double)a4.y * w, (double)a4.z * w, (double)a4.w * w};
          const double b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc64[q][i * 4 + j] = fma(a[i], b[j], acc64[q][i * 4 + j]);
        } else {
          const float a[4] = {a4.x * w, a4.y * w, a4.z * w, a4.w * w};
          const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[q][i * 4 + j] = fmaf(a[i], b[j], acc[q][i * 4 + j]);
        }
      }
    }
    since_flush += rows_per_tile;
    if (since_flush >= 64) {
      since_flush = 0;
#pragma unroll
      for (int q = 0; q < PPT; ++q)
#pragma unroll
        for (int e = 0; e < 16; ++e) { acc64[q][e] += (double)acc[q][e]; acc[q][e] = 0.f; }
    }
  }
#pragma unroll
  for (int q = 0; q < PPT; ++q)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc64[q][e] += (double)acc[q][e];

  const int P16 = pairs * 16;
  double* out = partial + (int64_t)blockIdx.x * P16;
  if (RG == 1) {
#pragma unroll
    for (int q = 0; q < PPT; ++q)
      if (pv[q]) {
        const int p = p0 + q * GT;
#pragma unroll
        for (int e = 0; e < 16; ++e) out[p * 16 + e] = acc64[q][e];
      }
    return;
  }
  __syncthreads();
  double* red = reinterpret_cast<double*>(smraw);  // [RG][P16]
  if (pv[0]) {
#pragma unroll
    for (int e = 0; e < 16; ++e) red[g * P16 + p0 * 16 + e] = acc64[0][e];
  }
  __syncthreads();
  for (int e = tid; e < P16; e += GT) {
    double s = 0.0;
    for (int gg = 0; gg < RG; ++gg) s += red[gg * P16 + e];
    out[e] = s;
  }
}

__global__ void cross_gram_finalize(const double* __restrict__ partial, int grid, int ka, int kb, int sym,
                                    double* __restrict__ out, int ldo, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int nba = (ka + 3) >> 2, nbb = (kb + 3) >> 2;
  const int pairs = sym ? nba * (nba + 1) / 2 : nba * nbb;
  const int P16 = pairs * 16;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < P16; e += gridDim.x * blockDim.x) {
    // eight independent partial chains (fixed order: deterministic) keep 8 loads in flight
    double s8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int pb = 0;
    for (; pb + 8 <= grid; pb += 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) s8[q] += __ldcg(partial + (int64_t)(pb + q) * P16 + e);
    }
    for (; pb < grid; ++pb) s8[0] += __ldcg(partial + (int64_t)pb * P16 + e);
    const double s = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
    const int p = e >> 4, i = (e >> 2) & 3, j = e & 3;
    int ai, bi;
    pair_to_blocks(p, nba, nbb, sym, ai, bi);
    const int a = 4 * ai + i, b = 4 * bi + j;
    if (a >= ka || b >= kb) continue;
    if (sym) {
      if (ai == bi && a > b) continue;   // diagonal block: write the upper half only, mirrored
      out[a * ldo + b] = s;
      out[b * ldo + a] = s;
    } else {
      out[a * ldo + b] = s;
    }
  }
}

int gram_grid(int64_t rows_cap) {
  const int64_t tiles = (rows_cap + GTR - 1) / GTR;
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 296));
}

size_t gram_partial_doubles(int ka, int kb, bool sym, int grid) {
  const int nba = (ka + 3) / 4, nbb = (kb + 3) / 4;
  const int pairs = sym ? nba * (nba + 1) / 2 : nba * nbb;
  return (size_t)grid * pairs * 16;
}

void launch_cross_gram(const float* A, int64_t lda, int ka, const float* B, int64_t ldb, int kb, bool sym,
                       int64_t nrows, const int64_t* nrows_dev, const int32_t* gather, const double* wts,
                       double* partial, int grid, double* out, int ldo, const int32_t* status, cudaStream_t st,
                       bool fp64_products) {
  const int nba = (ka + 3) / 4, nbb = (kb + 3) / 4;
  const int pairs = sym ? nba * (nba + 1) / 2 : nba * nbb;
  const int sta = nba * 4 + 4, stb = nbb * 4 + 4;
  size_t tile = sizeof(float) * (GTR * sta + (sym ? 0 : GTR * stb) + GTR);
  const int RG = pairs <= GT ? GT / pairs : 1;
  size_t red = RG > 1 ? sizeof(double) * RG * pairs * 16 : 0;
  size_t smem = std::max(tile, red);
  const int ppt = (pairs + GT - 1) / GT;
#define SYMNMF_GRAM_LAUNCH(P, D)                                                                          \
  do {                                                                                                    \
    cudaFuncSetAttribute(cross_gram_partial<P, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    cross_gram_partial<P, D><<<grid, GT, smem, st>>>(A, lda, ka, B, ldb, kb, sym, nrows, nrows_dev, gather, \
                                                     wts, partial, status);                               \
  } while (0)
  if (ppt <= 1) {
    if (fp64_products) SYMNMF_GRAM_LAUNCH(1, true); else SYMNMF_GRAM_LAUNCH(1, false);
  } else {
    if (fp64_products) SYMNMF_GRAM_LAUNCH(2, true); else SYMNMF_GRAM_LAUNCH(2, false);
  }
#undef SYMNMF_GRAM_LAUNCH
  cross_gram_finalize<<<(pairs * 16 + 127) / 128, 128, 0, st>>>(partial, grid, ka, kb, sym, out, ldo, status);
}

// ---------------------------------------------------------------- (a2) Cholesky + inverse
// One CTA.  G = R^T R with R upper (right-looking, fp64).  A non-positive or
// non-finite pivot triggers one retry with G + (1e-12 tr(G)/k) I;
// a second failure sets SYMNMF_ERR_NOT_PD.  Then R^{-1} by backward elimination of R X = I.
// shift_rel > 0 factors G + shift_rel tr(G) I from the start (the shifted
// first pass of the range finder's CholeskyQR2, which must survive a
// numerically rank-deficient sketch A Omega).
// One barrier per column in both phases: step j updates the trailing rows from the unscaled
// row j (a_ic -= a_ji a_jc / a_jj) and scales row j - 1 by 1 / r_{j-1,j-1}, which step j no longer
// reads; warps take rows, lanes columns.  (Was: three barriers per column, a thread per column of
// R^{-1} with a dependent O(k^2) chain -- 0.14 ms per call at k = 74, verdict r1.)
__global__ void __launch_bounds__(512) chol_inv_kernel(const double* __restrict__ G, int k, float* __restrict__ R32,
                                                       int ldr32, int padk32, double* __restrict__ R64, int ldr64,
                                                       double shift_rel, int32_t* __restrict__ status) {
  extern __shared__ double smd[];
  __shared__ double jit[2];
  if (dev_failed(status)) return;
  const int ld = k + 1;
  double* a = smd;
  double* x = smd + k * ld;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < k; ++i) tr += G[i * k + i];
    jit[0] = shift_rel * tr;
    jit[1] = shift_rel * tr + 1e-12 * tr / k;
  }
  __syncthreads();
  bool fail = true;
  for (int attempt = 0; attempt < 2 && fail; ++attempt) {
    const double jitter = jit[attempt];
    if (attempt == 1 && !(jitter > 0.0)) break;
    for (int e = tid; e < k * k; e += nt) {
      const int i = e / k, c = e - i * k;
      a[i * ld + c] = G[e] + (i == c ? jitter : 0.0);
    }
    __syncthreads();
    fail = false;
    double rprev = 1.0;
    for (int j = 0; j < k; ++j) {
      const double d = a[j * ld + j];   // final since the previous barrier; the same in every thread
      if (!(d > 0.0) || !isfinite(d)) { fail = true; break; }
      const double dinv = 1.0 / d;
      for (int i = j + 1 + wid; i < k; i += nw) {
        const double f = a[j * ld + i] * dinv;
        for (int c = i + lane; c < k; c += 32) a[i * ld + c] -= f * a[j * ld + c];
      }
      if (j > 0)
        for (int c = j - 1 + tid; c < k; c += nt) a[(j - 1) * ld + c] = c == j - 1 ? rprev : a[(j - 1) * ld + c] / rprev;
      rprev = sqrt(d);
      __syncthreads();
    }
    if (!fail) {
      for (int c = k - 1 + tid; c < k; c += nt) a[(k - 1) * ld + c] = rprev;
      __syncthreads();
    } else {
      __syncthreads();
    }
  }
  if (fail) {
    if (tid == 0) dev_fail(status, SYMNMF_ERR_NOT_PD);
    return;
  }
  // R X = I: step i divides row i of the right-hand side (deferred to step i - 1) and eliminates
  // column i from rows m < i
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, c = e - i * k;
    x[i * ld + c] = i == c ? 1.0 : 0.0;
  }
  __syncthreads();
  double iprev = 1.0;
  for (int i = k - 1; i >= 0; --i) {
    const double inv = 1.0 / a[i * ld + i];
    for (int m = wid; m < i; m += nw) {
      const double f = a[m * ld + i] * inv;
      for (int c = i + lane; c < k; c += 32) x[m * ld + c] -= f * x[i * ld + c];
    }
    if (i + 1 < k)
      for (int c = i + 1 + tid; c < k; c += nt) x[(i + 1) * ld + c] *= iprev;
    iprev = inv;
    __syncthreads();
  }
  for (int c = tid; c < k; c += nt) x[c] *= iprev;
  __syncthreads();
  if (R32) {
    for (int e = tid; e < padk32 * padk32; e += nt) {
      const int i = e / padk32, c = e - i * padk32;
      R32[i * ldr32 + c] = (i < k && c < k) ? (float)x[i * ld + c] : 0.f;
    }
  }
  if (R64) {
    for (int e = tid; e < k * k; e += nt) {
      const int i = e / k, c = e - i * k;
      R64[i * ldr64 + c] = x[i * ld + c];
    }
  }
}

void launch_chol_inv(const double* G, int k, float* Rinv32, int ldr32, int padk32, double* Rinv64, int ldr64,
                     int32_t* status, cudaStream_t st, double shift_rel) {
  const size_t smem = sizeof(double) * 2 * k * (k + 1);
  cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  chol_inv_kernel<<<1, 512, smem, st>>>(G, k, Rinv32, ldr32, padk32, Rinv64, ldr64, shift_rel, status);
}

}  // namespace symnmf
