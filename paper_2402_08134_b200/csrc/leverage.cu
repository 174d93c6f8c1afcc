// (a3) Leverage scores l_i = ||f_i R^{-1}||^2 (Eq. 2.10; Alg. LvS-SymNMF
// lines "Solve H R^{-1} = Q_H", "p_H[i] = ||Q_H[i,:]||^2").
// R^{-1} (upper, fp32, KP x KP zero padded) sits in shared memory; a CTA
// stages 128 consecutive rows of F (one contiguous run) with coalesced loads
// and every thread forms q = f_i R^{-1} for its row in registers.
#include "kernels.cuh"

namespace symnmf {

template <int KP>
__global__ void __launch_bounds__(128) leverage_kernel(const float* __restrict__ F, int64_t n, int k,
                                                       const float* __restrict__ Rinv, float* __restrict__ lev,
                                                       const int32_t* __restrict__ status) {
  __shared__ __align__(16) float sR[KP * KP];
  extern __shared__ float sF[];
  if (dev_failed(status)) return;
  const int tid = threadIdx.x;
  for (int e = tid; e < KP * KP; e += 128) sR[e] = Rinv[e];
  const int stride = k | 1;
  for (int64_t base = (int64_t)blockIdx.x * 128; base < n; base += (int64_t)gridDim.x * 128) {
    __syncthreads();
    const int cnt = (int)min64(128, n - base);
    const float* src = F + base * k;
    for (int e = tid; e < cnt * k; e += 128) {
      const int r = e / k, c = e - r * k;
      sF[r * stride + c] = src[e];
    }
    __syncthreads();
    if (tid < cnt) {
      float f[KP];
#pragma unroll
      for (int a = 0; a < KP; ++a) f[a] = a < k ? sF[tid * stride + a] : 0.f;
      float l = 0.f;
#pragma unroll
      for (int c = 0; c < KP; ++c) {
        float q = 0.f;
#pragma unroll
        for (int a = 0; a <= c; ++a) q = fmaf(f[a], sR[a * KP + c], q);
        l = fmaf(q, q, l);
      }
      lev[base + tid] = l;
    }
  }
}

template <int KP>
static void launch_lev_t(const float* F, int64_t n, int k, const float* Rinv, float* lev, const int32_t* status,
                         cudaStream_t st) {
  const size_t smem = sizeof(float) * 128 * (k | 1);
  cudaFuncSetAttribute(leverage_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t blocks = std::min<int64_t>((n + 127) / 128, 148 * 8);
  leverage_kernel<KP><<<(int)std::max<int64_t>(blocks, 1), 128, smem, st>>>(F, n, k, Rinv, lev, status);
}

void launch_leverage(const float* F, int64_t n, int k, const float* Rinv32, float* lev, const int32_t* status,
                     cudaStream_t st) {
  switch (kpad(k)) {
    case 8: launch_lev_t<8>(F, n, k, Rinv32, lev, status, st); break;
    case 16: launch_lev_t<16>(F, n, k, Rinv32, lev, status, st); break;
    case 32: launch_lev_t<32>(F, n, k, Rinv32, lev, status, st); break;
    default: launch_lev_t<64>(F, n, k, Rinv32, lev, status, st); break;
  }
}

}  // namespace symnmf
