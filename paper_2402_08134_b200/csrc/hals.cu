// (a11) Efficient symmetric HALS sweep, Eq. 2.6 with the Update(G + alpha I,
// Y + alpha F^T) shape of Alg. LvS-SymNMF / LAI-SymNMF:
//   for every row r, i = 0..k-1 in order (Gauss-Seidel over the columns, Z9):
//     x_ri <- max(0, (Y_ri + alpha F_ri - sum_{j != i} x_rj G_ji) / (G_ii + alpha))
// Rows are independent, so the column sweep of the paper becomes a per-row
// register loop.  A warp stages 32 consecutive rows (one contiguous run of 32k
// floats) of B = Y + alpha F and X through shared memory with coalesced loads
// (odd row stride: conflict-free per-row reads), each lane updates one row in
// registers, and the warp writes X back coalesced.  G (+ alpha on the
// diagonal) lives in shared memory as fp32; column i of G is read as float4
// broadcasts.
#include "kernels.cuh"

namespace symnmf {

constexpr int HW = 4;   // warps per CTA

template <int KP>
__global__ void __launch_bounds__(HW * 32) hals_sweep_kernel(const double* __restrict__ G,
                                                             const float* __restrict__ Y,
                                                             const float* __restrict__ F, float* __restrict__ X,
                                                             int64_t n, int k, double alpha,
                                                             const int32_t* __restrict__ status) {
  __shared__ __align__(16) float sG[KP * KP];   // sG[i*KP + j] = G[j][i] (G symmetric), 0 on the diagonal
  __shared__ float sInv[KP];
  __shared__ int sOk[KP];
  extern __shared__ float smw[];
  if (dev_failed(status)) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < KP * KP; e += HW * 32) {
    const int i = e / KP, j = e - i * KP;
    sG[e] = (i < k && j < k && i != j) ? (float)G[j * k + i] : 0.f;
  }
  for (int i = tid; i < KP; i += HW * 32) {
    const double den = i < k ? G[i * k + i] + alpha : 0.0;
    sOk[i] = den > 0.0;
    sInv[i] = den > 0.0 ? (float)(1.0 / den) : 0.f;
  }
  __syncthreads();
  const int stride = k | 1;
  float* sB = smw + wid * 2 * 32 * stride;
  float* sX = sB + 32 * stride;
  const float a32 = (float)alpha;
  const int64_t nwarps = (int64_t)gridDim.x * HW;
  for (int64_t base = ((int64_t)blockIdx.x * HW + wid) * 32; base < n; base += nwarps * 32) {
    const int cnt = (int)min64(32, n - base);
    const int64_t g0 = base * k;
    for (int e = lane; e < cnt * k; e += 32) {
      const int r = e / k, c = e - r * k;
      sB[r * stride + c] = fmaf(a32, F[g0 + e], Y[g0 + e]);
      sX[r * stride + c] = X[g0 + e];
    }
    __syncwarp();
    if (lane < cnt) {
      float x[KP], b[KP];
#pragma unroll
      for (int j = 0; j < KP; ++j) {
        x[j] = j < k ? sX[lane * stride + j] : 0.f;
        b[j] = j < k ? sB[lane * stride + j] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        if (i < k) {
          float s = b[i];
#pragma unroll
          for (int j = 0; j < KP; j += 4) {
            const float4 g = *reinterpret_cast<const float4*>(sG + i * KP + j);
            s = fmaf(-x[j], g.x, s);
            s = fmaf(-x[j + 1], g.y, s);
            s = fmaf(-x[j + 2], g.z, s);
            s = fmaf(-x[j + 3], g.w, s);
          }
          if (sOk[i]) x[i] = fmaxf(0.f, s * sInv[i]);
        }
      }
#pragma unroll
      for (int j = 0; j < KP; ++j)
        if (j < k) sX[lane * stride + j] = x[j];
    }
    __syncwarp();
    for (int e = lane; e < cnt * k; e += 32) {
      const int r = e / k, c = e - r * k;
      X[g0 + e] = sX[r * stride + c];
    }
    __syncwarp();
  }
}

template <int KP>
static void launch_hals_t(const double* G, const float* Y, const float* F, float* X, int64_t n, int k, double alpha,
                          const int32_t* status, cudaStream_t st) {
  const size_t smem = sizeof(float) * HW * 2 * 32 * (k | 1);
  cudaFuncSetAttribute(hals_sweep_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + HW * 32 - 1) / (HW * 32), 148 * 8));
  hals_sweep_kernel<KP><<<(unsigned)blocks, HW * 32, smem, st>>>(G, Y, F, X, n, k, alpha, status);
}

void launch_hals_sweep(const double* G, const float* Y, const float* F, float* X, int64_t n, int k, double alpha,
                       const int32_t* status, cudaStream_t st) {
  switch (kpad(k)) {
    case 8: launch_hals_t<8>(G, Y, F, X, n, k, alpha, status, st); break;
    case 16: launch_hals_t<16>(G, Y, F, X, n, k, alpha, status, st); break;
    case 32: launch_hals_t<32>(G, Y, F, X, n, k, alpha, status, st); break;
    default: launch_hals_t<64>(G, Y, F, X, n, k, alpha, status, st); break;
  }
}

}  // namespace symnmf
