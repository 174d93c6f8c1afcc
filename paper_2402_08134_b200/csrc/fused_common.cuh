// Device helpers shared by the fused solver kernels (fused.cu) and the persistent
// row-tile kernels (tile.cu): last-CTA detection, the fp64 warp Cholesky
// of CholeskyQR, register-blocked Gram partials and the
// last-CTA Gram finalize.  Included by .cu files only.
#pragma once
#include "kernels.cuh"

namespace symnmf {

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ bool arrive_last(unsigned int* counter) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0;
  }
  return last;
}

// One warp: fp64 Cholesky a = R^T R (upper, in place, ld = k + 1) of G + jitter I with one
// retry, then x = R^{-1}.  Returns nonzero on failure.
__device__ inline int warp_chol_inv(double* a, double* x, const double* G, int k, double shift_rel, bool inverse = true) {
  const int lane = threadIdx.x & 31, ld = k + 1;
  // G -> shared memory once (independent loads), trace from shared memory
  for (int e = lane; e < k * k; e += 32) {
    const int i = e / k, c = e - i * k;
    x[i * ld + c] = G[e];
  }
  __syncwarp();
  double tr = 0.0;
  for (int i = 0; i < k; ++i) tr += x[i * ld + i];
  int fail = 1;
  for (int attempt = 0; attempt < 2 && fail; ++attempt) {
    double jitter = shift_rel * tr + (attempt ? 1e-12 * tr / k : 0.0);
    if (attempt && !(jitter > 0.0)) break;
    for (int e = lane; e < k * ld; e += 32) {
      const int i = e / ld, c = e - i * ld;
      if (c < k) a[e] = x[e] + (i == c ? jitter : 0.0);
    }
    __syncwarp();
    fail = 0;
    for (int j = 0; j < k; ++j) {
      const double d = a[j * ld + j];
      if (!(d > 0.0) || !isfinite(d)) { fail = 1; break; }
      const double r = sqrt(d), rinv = 1.0 / r;
      __syncwarp();
      for (int c = j + 1 + lane; c < k; c += 32) a[j * ld + c] *= rinv;
      if (lane == 0) a[j * ld + j] = r;
      __syncwarp();
      for (int i = j + 1 + lane; i < k; i += 32) {      // lane-parallel rows of the trailing update
        const double aji = a[j * ld + i];
        for (int c = i; c < k; ++c) a[i * ld + c] = fma(-aji, a[j * ld + c], a[i * ld + c]);
      }
      __syncwarp();
    }
    __syncwarp();
  }
  if (fail) return 1;
  if (!inverse) return 0;
  for (int c = lane; c < k; c += 32) {
    x[c * ld + c] = 1.0 / a[c * ld + c];
    for (int i = c - 1; i >= 0; --i) {
      double s = 0.0;
      for (int j = i + 1; j <= c; ++j) s = fma(a[i * ld + j], x[j * ld + c], s);
      x[i * ld + c] = -s / a[i * ld + i];
    }
    for (int i = c + 1; i < k; ++i) x[i * ld + c] = 0.0;
  }
  __syncwarp();
  return 0;
}

// 1/sqrt(d) in fp64 without the long-latency fp64 sqrt and divide sequences: fp32 MUFU
// estimate refined by two Newton steps (relative error ~1e-16 for normal d).
__device__ __forceinline__ double rsqrt_fp64(double d) {
  if (!(d > 1e-30 && d < 1e30)) return 1.0 / sqrt(d);   // outside the fp32 estimate's safe range
  double y = (double)rsqrtf((float)d);
  const double h = 0.5 * d;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// One warp, k <= KP <= 32: fp64 Cholesky G + jitter I = R^T R held in registers, lane c owning
// column c (R[i][c], i <= c).  Step j broadcasts R[j][i] from lane i with compile-time shuffle
// sources, so there is no shared memory traffic and no barrier.  Padding columns c >= k carry
// the identity.  Writes R (fp32, KP x KP upper, zero padded) and rd = 1 / diag(R).
// One factorisation pass over b (fully unrolled: every register index is a compile-time
// constant, no break, so b stays in registers).  Returns nonzero if a pivot was not positive.
template <int KP>
__device__ __forceinline__ int chol_col_pass(double (&b)[KP], int lane, double& myr) {
  int fail = 0;
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    const double d = __shfl_sync(0xffffffffu, b[j], j);
    fail |= (!(d > 0.0) || !isfinite(d)) ? 1 : 0;
    const double dd = fail ? 1.0 : d;
    const double rinv = rsqrt_fp64(dd), r = dd * rinv;
    if (lane == j) { b[j] = r; myr = r; }
    else if (lane > j) b[j] *= rinv;                          // R[j][lane]
    // constant trip count (i > j as a predicate): unrolls whatever order the compiler unrolls
    // the two loops in, so b[] stays in registers (with `i = j + 1` bounds, the BPP kernel's
    // copy kept b[] in local memory)
#pragma unroll
    for (int i = 1; i < KP; ++i) {
      if (i <= j) continue;
      const double rji = __shfl_sync(0xffffffffu, b[j], i);   // R[j][i] from lane i
      if (lane >= i) b[i] = fma(-rji, b[j], b[i]);            // A[i][lane] -= R[j][i] R[j][lane]
    }
  }
  return fail;
}

template <int KP>
__device__ inline int warp_chol_col(const double* G, int k, double shift_rel, float* R32, float* rd32) {
  static_assert(KP <= 32, "one column per lane");
  const int lane = threadIdx.x & 31;
  double b[KP];   // column `lane` of G (re-read from G for the retry: keeps register use at KP doubles)
  const double dl = lane < k ? G[lane * k + lane] : 0.0;
  const double tr = warp_sum(dl);
  double myr = 1.0;
  double jitter = shift_rel * tr;
#pragma unroll
  for (int i = 0; i < KP; ++i)
    b[i] = ((lane < k && i < k) ? G[i * k + lane] : (i == lane ? 1.0 : 0.0)) + ((i == lane && lane < k) ? jitter : 0.0);
  int fail = chol_col_pass<KP>(b, lane, myr);
  if (fail) {                                   // one retry with 1e-12 tr(G)/k on the diagonal
    jitter += 1e-12 * tr / k;
    if (!(jitter > 0.0)) return 1;
#pragma unroll
    for (int i = 0; i < KP; ++i)
      b[i] = ((lane < k && i < k) ? G[i * k + lane] : (i == lane ? 1.0 : 0.0)) + ((i == lane && lane < k) ? jitter : 0.0);
    fail = chol_col_pass<KP>(b, lane, myr);
  }
  if (fail) return 1;
  if (lane < KP) {
#pragma unroll
    for (int i = 0; i < KP; ++i) R32[i * KP + lane] = (i <= lane && lane < k) ? (float)b[i] : 0.f;
    rd32[lane] = lane < k ? (float)(1.0 / myr) : 0.f;
  }
  return 0;
}

// Per-thread share of a k x k Gram accumulated from row tiles in shared memory:
// one upper 4x4 block (ai <= bi) per thread, row groups g = t / pairs.
struct GramThread {
  int ai, bi, g, RG, p;
  bool active;
  float acc[16];
  double acc64[16];
  int since;
  __device__ void init(int t, int nthreads, int nb) {
    const int pairs = nb * (nb + 1) / 2;
    RG = nthreads / pairs;
    g = t / pairs;
    p = t - g * pairs;
    active = g < RG;
    int a = 0, rem = p;
    while (rem >= nb - a) { rem -= nb - a; ++a; }
    ai = a; bi = a + rem;
#pragma unroll
    for (int e = 0; e < 16; ++e) { acc[e] = 0.f; acc64[e] = 0.0; }
    since = 0;
  }
  // rows r of s (row stride `stride` floats, 16B aligned), optional fp32 row weights w
  __device__ void accumulate(const float* s, int stride, int rows, const float* w) {
    if (!active) return;
    for (int r = g; r < rows; r += RG) {
      const float4 a4 = *reinterpret_cast<const float4*>(s + r * stride + 4 * ai);
      const float4 b4 = *reinterpret_cast<const float4*>(s + r * stride + 4 * bi);
      const float wr = w ? w[r] : 1.f;
      const float a[4] = {a4.x * wr, a4.y * wr, a4.z * wr, a4.w * wr};
      const float2 b01 = make_float2(b4.x, b4.y), b23 = make_float2(b4.z, b4.w);
#pragma unroll
      for (int i = 0; i < 4; ++i) {   // packed FFMA2 over column pairs
        float2 p0 = make_float2(acc[i * 4], acc[i * 4 + 1]), p1 = make_float2(acc[i * 4 + 2], acc[i * 4 + 3]);
        p0 = ffma2(make_float2(a[i], a[i]), b01, p0);
        p1 = ffma2(make_float2(a[i], a[i]), b23, p1);
        acc[i * 4] = p0.x; acc[i * 4 + 1] = p0.y; acc[i * 4 + 2] = p1.x; acc[i * 4 + 3] = p1.y;
      }
    }
    since += (rows + RG - 1) / RG;
    if (since >= 64) flush();
  }
  __device__ void flush() {
#pragma unroll
    for (int e = 0; e < 16; ++e) { acc64[e] += (double)acc[e]; acc[e] = 0.f; }
    since = 0;
  }
  // CTA-cooperative commit: reduce the row groups in shared memory (fixed order), then one
  // fp64 red.add per Gram entry and CTA into replica blockIdx % kGramReplicas of the global
  // accumulator (k x k upper triangle per replica): bounded same-address contention.
  // `red` needs RG * pairs * 16 doubles (<= 32 KB); all threads of the CTA must call.
  __device__ void commit(double* Gacc, int k, double* red) {
    flush();
    const int nb = (k + 3) >> 2, pairs = nb * (nb + 1) / 2, P16 = pairs * 16;
    __syncthreads();
    if (active) {
#pragma unroll
      for (int e = 0; e < 16; ++e) red[g * P16 + p * 16 + e] = acc64[e];
    }
    __syncthreads();
    double* rep = Gacc + (size_t)(blockIdx.x % kGramReplicas) * k * k;
    for (int idx = threadIdx.x; idx < P16; idx += blockDim.x) {
      double s = 0.0;
      for (int gg = 0; gg < RG; ++gg) s += red[gg * P16 + idx];
      const int pp = idx >> 4, i = (idx >> 2) & 3, j = idx & 3;
      int a0 = 0, rem = pp;
      while (rem >= nb - a0) { rem -= nb - a0; ++a0; }
      const int a = 4 * a0 + i, b = 4 * (a0 + rem) + j;
      if (a < k && b < k && a <= b && s != 0.0) atomicAdd(rep + a * k + b, s);
    }
  }
};

// Last CTA: G_out (mirrored, fp64) <- sum of the accumulator replicas, replicas <- 0;
// optional Cholesky -> R^{-1} fp32 (KP x KP).
// Rf32 (nullable): CholeskyQR factor of G, R upper (KP x KP fp32) followed by 1 / diag(R) (KP).
template <int KP>
__device__ inline void finalize_gram(double* Gacc, double* Gout, int k, float* Rf32, double* sm_a, double* sm_x,
                              int32_t* status) {
  const int kk = k * k;
  for (int e = threadIdx.x; e < kk; e += blockDim.x) {
    const int a = e / k, b = e - a * k;
    if (a > b) continue;
    double v[kGramReplicas];
#pragma unroll
    for (int r = 0; r < kGramReplicas; ++r) v[r] = __ldcg(Gacc + (size_t)r * kk + e);
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < kGramReplicas; ++r) s += v[r];
    Gout[a * k + b] = s;
    Gout[b * k + a] = s;
#pragma unroll
    for (int r = 0; r < kGramReplicas; ++r) Gacc[(size_t)r * kk + e] = 0.0;
  }
  __syncthreads();
  if (!Rf32) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x < 32) {
    int fail;
    if constexpr (KP <= 16) {   // register form; wider factors use shared memory (register budget of the host kernel)
      fail = warp_chol_col<KP>(Gout, k, 0.0, Rf32, Rf32 + KP * KP);
    } else {
      fail = warp_chol_inv(sm_a, sm_x, Gout, k, 0.0, /*inverse=*/false);
      if (!fail) {
        for (int e = threadIdx.x; e < KP * KP; e += 32) {
          const int i = e / KP, c = e - i * KP;
          Rf32[e] = (i <= c && c < k) ? (float)sm_a[i * (k + 1) + c] : 0.f;
        }
        for (int c = threadIdx.x; c < KP; c += 32) Rf32[KP * KP + c] = c < k ? (float)(1.0 / sm_a[c * (k + 1) + c]) : 0.f;
      }
    }
    if (fail && threadIdx.x == 0) dev_fail(status, SYMNMF_ERR_NOT_PD);
  }
}

}  // namespace symnmf
