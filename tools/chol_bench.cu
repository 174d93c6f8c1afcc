// Microbenchmark: cycles of candidate k x k Cholesky formulations for the last-CTA step.
#include <cstdio>
#include "../paper_2402_08134_b200/csrc/fused.cu"
using namespace symnmf;

template <int KP, typename T>
__device__ int chol_col_t(const double* G, int k, float* R32) {   // register, lane = column, type T
  const int lane = threadIdx.x & 31;
  T b[KP];
#pragma unroll
  for (int i = 0; i < KP; ++i) b[i] = (lane < k && i < k) ? (T)G[i * k + lane] : (T)(i == lane ? 1 : 0);
  int fail = 0;
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    const T d = __shfl_sync(0xffffffffu, b[j], j);
    if (!(d > T(0))) { fail = 1; break; }
    T rinv;
    if constexpr (sizeof(T) == 4) rinv = rsqrtf(d); else rinv = rsqrt_fp64(d);
    const T r = d * rinv;
    if (lane == j) b[j] = r; else if (lane > j) b[j] *= rinv;
#pragma unroll
    for (int i = j + 1; i < KP; ++i) {
      const T rji = __shfl_sync(0xffffffffu, b[j], i);
      if (lane >= i) b[i] = fma(-rji, b[j], b[i]);
    }
  }
  if (lane < KP)
    for (int i = 0; i < KP; ++i) R32[i * KP + lane] = (float)b[i];
  return fail;
}

// whole CTA, fp64, smem, right-looking
__device__ int chol_cta(const double* G, int k, double* a, float* R32) {
  const int t = threadIdx.x, ld = k + 1;
  __shared__ int fail;
  for (int e = t; e < k * k; e += blockDim.x) a[(e / k) * ld + e % k] = G[e];
  if (t == 0) fail = 0;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    const double d = a[j * ld + j];
    if (!(d > 0.0)) { if (t == 0) fail = 1; break; }
    const double rinv = rsqrt_fp64(d);
    // scale row j (c > j) and update trailing (i, c) with i <= c, both using scaled values
    const int m = k - j - 1;
    for (int e = t; e < m; e += blockDim.x) a[j * ld + j + 1 + e] *= rinv;
    __syncthreads();
    for (int e = t; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e / m, c = j + 1 + e % m;
      if (i <= c) a[i * ld + c] = fma(-a[j * ld + i], a[j * ld + c], a[i * ld + c]);
    }
    if (t == 0) a[j * ld + j] = d * rinv;
    __syncthreads();
  }
  return fail;
}

template <int KP>
__global__ void bench(const double* G, int k, float* R, long long* cyc, int variant) {
  __shared__ double a[64 * 65];
  long long t0 = clock64();
  int f = 0;
  for (int rep = 0; rep < 10; ++rep) {
    if (variant == 0) f += warp_chol_col<KP>(G, k, 0.0, R, R + KP * KP);
    else if (variant == 1) f += chol_col_t<KP, float>(G, k, R);
    else if (variant == 2) f += chol_col_t<KP, double>(G, k, R);
    else f += chol_cta(G, k, a, R);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 10; cyc[1] = f; }
}
int main() {
  const int k = 16;
  double hG[32 * 32];
  for (int kk : {16, 32}) {
    for (int i = 0; i < kk; ++i) for (int j = 0; j < kk; ++j) hG[i * kk + j] = (i == j ? kk + 1.0 : 1.0 / (1 + i + j));
    double* G; float* R; long long* c;
    cudaMalloc(&G, sizeof(hG)); cudaMalloc(&R, 4 * 64 * 65); cudaMalloc(&c, 16);
    cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
    const char* names[] = {"warp_chol_col(fp64,rsqrt+2NR)", "reg fp32", "reg fp64", "cta smem fp64 (256 thr)"};
    for (int v = 0; v < 4; ++v) {
      if (kk == 16) bench<16><<<1, v == 3 ? 256 : 32>>>(G, kk, R, c, v);
      else bench<32><<<1, v == 3 ? 256 : 32>>>(G, kk, R, c, v);
      long long hc[2]; cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
      printf("k=%d %-32s %8lld cycles (fail=%lld)\n", kk, names[v], hc[0], hc[1]);
    }
  }
  (void)k;
  return 0;
}
