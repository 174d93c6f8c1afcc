// (a12) Pieces of Alg. RRF / Alg. Apx-EVD and (a13)
// the LAI product U (Lambda (U^T F)):
//  - Gaussian Omega by Box-Muller on Philox4x32-10 (reading Z18),
//  - row-apply of a small matrix (Q = Y R^{-1}, U = Q V, Y = U M),
//  - one-CTA parallel-order cyclic Jacobi eigensolver for T = Q^T A Q (fp64).
#include "kernels.cuh"

namespace symnmf {

__global__ void gaussian_kernel(int64_t total, uint64_t seed, float* __restrict__ Om) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * p >= total) return;
  const uint4 x = philox4x32_10(make_uint4((uint32_t)p, (uint32_t)((uint64_t)p >> 32), 0u, 1u),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const double u1 = ((double)x.x + 0.5) * 2.3283064365386963e-10;   // 2^-32
  const double u2 = ((double)x.y + 0.5) * 2.3283064365386963e-10;
  const double rho = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.141592653589793 * u2;
  Om[2 * p] = (float)(rho * cos(ang));
  if (2 * p + 1 < total) Om[2 * p + 1] = (float)(rho * sin(ang));
}

void launch_gaussian(int64_t n, int l, uint64_t seed, float* Omega, cudaStream_t st) {
  const int64_t total = n * l, pairs = (total + 1) / 2;
  gaussian_kernel<<<(unsigned)((pairs + 255) / 256), 256, 0, st>>>(total, seed, Omega);
}

// ---------------------------------------------------------------- row apply
constexpr int RW = 4;   // warps per CTA

template <typename MT>
__global__ void __launch_bounds__(RW * 32) rowapply_kernel(const float* __restrict__ X, int64_t ldx, int64_t n, int ka,
                                                           const MT* __restrict__ M, int kb, float* __restrict__ Y,
                                                           int64_t ldy, const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smr[];
  if (dev_failed(status)) return;
  const int kbp = (kb + 31) & ~31;
  MT* sM = reinterpret_cast<MT*>(smr);
  const int sx = ka | 1, sy = kb | 1;
  float* wbase = reinterpret_cast<float*>(smr + sizeof(MT) * ka * kbp);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  float* sX = wbase + wid * 32 * (sx + sy);
  float* sY = sX + 32 * sx;
  for (int e = tid; e < ka * kbp; e += RW * 32) {
    const int a = e / kbp, b = e - a * kbp;
    sM[e] = b < kb ? M[a * kb + b] : MT(0);
  }
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * RW;
  for (int64_t base = ((int64_t)blockIdx.x * RW + wid) * 32; base < n; base += nwarps * 32) {
    const int cnt = (int)min64(32, n - base);
    for (int e = lane; e < cnt * ka; e += 32) {
      const int r = e / ka, c = e - r * ka;
      sX[r * sx + c] = X[(base + r) * ldx + c];
    }
    __syncwarp();
    if (lane < cnt) {
      for (int cb = 0; cb < kbp; cb += 32) {
        MT acc[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) acc[b] = MT(0);
        for (int a = 0; a < ka; ++a) {
          const MT xa = (MT)sX[lane * sx + a];
          const MT* mrow = sM + a * kbp + cb;
#pragma unroll
          for (int b = 0; b < 32; ++b) acc[b] += xa * mrow[b];
        }
#pragma unroll
        for (int b = 0; b < 32; ++b)
          if (cb + b < kb) sY[lane * sy + cb + b] = (float)acc[b];
      }
    }
    __syncwarp();
    for (int e = lane; e < cnt * kb; e += 32) {
      const int r = e / kb, c = e - r * kb;
      Y[(base + r) * ldy + c] = sY[r * sy + c];
    }
    __syncwarp();
  }
}

template <typename MT>
static void launch_rowapply_t(const float* X, int64_t ldx, int64_t n, int ka, const MT* M, int kb, float* Y,
                              int64_t ldy, const int32_t* status, cudaStream_t st) {
  const int kbp = (kb + 31) & ~31;
  const size_t smem = sizeof(MT) * ka * kbp + sizeof(float) * RW * 32 * ((ka | 1) + (kb | 1));
  cudaFuncSetAttribute(rowapply_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + RW * 32 - 1) / (RW * 32), 148 * 4));
  rowapply_kernel<MT><<<(unsigned)blocks, RW * 32, smem, st>>>(X, ldx, n, ka, M, kb, Y, ldy, status);
}

void launch_rowapply32(const float* X, int64_t ldx, int64_t n, int ka, const float* M, int kb, float* Y, int64_t ldy,
                       const int32_t* status, cudaStream_t st) {
  launch_rowapply_t<float>(X, ldx, n, ka, M, kb, Y, ldy, status, st);
}
void launch_rowapply64(const float* X, int64_t ldx, int64_t n, int ka, const double* M, int kb, float* Y,
                       int64_t ldy, const int32_t* status, cudaStream_t st) {
  launch_rowapply_t<double>(X, ldx, n, ka, M, kb, Y, ldy, status, st);
}

__global__ void scale_rows_kernel(const double* __restrict__ Z, int l, int k, const double* __restrict__ lam,
                                  float* __restrict__ M, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < l * k; e += gridDim.x * blockDim.x)
    M[e] = (float)(lam[e / k] * Z[e]);
}
void launch_scale_rows(const double* Z, int l, int k, const double* lambda, float* M32, const int32_t* status,
                       cudaStream_t st) {
  scale_rows_kernel<<<(l * k + 255) / 256, 256, 0, st>>>(Z, l, k, lambda, M32, status);
}

__global__ void symmetrize_kernel(double* T, int l) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < l * l; e += gridDim.x * blockDim.x) {
    const int i = e / l, j = e - i * l;
    if (i < j) {
      const double v = 0.5 * (T[i * l + j] + T[j * l + i]);
      T[i * l + j] = v;
      T[j * l + i] = v;
    }
  }
}
void launch_symmetrize(double* T, int l, cudaStream_t st) { symmetrize_kernel<<<(l * l + 255) / 256, 256, 0, st>>>(T, l); }

// ---------------------------------------------------------------- Jacobi EVD
// Brent-Luk round-robin ordering: each of the m-1 steps of a sweep applies
// m/2 disjoint rotations at once (rows, then columns and V).
__device__ __forceinline__ int rr_index(int pos, int step, int m) {
  return pos == 0 ? 0 : ((pos - 1 + step) % (m - 1)) + 1;
}

__global__ void __launch_bounds__(256) jacobi_kernel(const double* __restrict__ Tin, int l, double* __restrict__ Vout,
                                                     double* __restrict__ lam, int32_t* __restrict__ status) {
  extern __shared__ double sj[];
  __shared__ double cs[kMaxL / 2 + 1], sn[kMaxL / 2 + 1];
  __shared__ int pi_[kMaxL / 2 + 1], pj_[kMaxL / 2 + 1];
  __shared__ double red[32];
  __shared__ int done;
  __shared__ int order[kMaxL];
  if (dev_failed(status)) return;
  const int ld = l + 1, tid = threadIdx.x, nt = blockDim.x;
  double* T = sj;
  double* V = sj + l * ld;
  for (int e = tid; e < l * l; e += nt) {
    const int i = e / l, j = e - i * l;
    T[i * ld + j] = Tin[e];
    V[i * ld + j] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  const int m = l + (l & 1), half = m / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < l * l; e += nt) {
      const int i = e / l, j = e - i * l;
      const double v = T[i * ld + j];
      tot += v * v;
      if (i < j) off += v * v;
    }
    off = block_sum(off, red);
    tot = block_sum(tot, red);
    if (tid == 0) done = !(off > 1e-30 * tot);
    __syncthreads();
    if (done) break;
    for (int step = 0; step < m - 1; ++step) {
      if (tid < half) {
        int i = rr_index(tid, step, m), j = rr_index(m - 1 - tid, step, m);
        if (i > j) { const int t = i; i = j; j = t; }
        double c = 1.0, s = 0.0;
        if (j < l) {
          const double tij = T[i * ld + j];
          if (tij != 0.0) {
            const double th = (T[j * ld + j] - T[i * ld + i]) / (2.0 * tij);
            const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
          }
        }
        cs[tid] = c; sn[tid] = s; pi_[tid] = i; pj_[tid] = j < l ? j : -1;
      }
      __syncthreads();
      for (int e = tid; e < half * l; e += nt) {
        const int p = e / l, col = e - p * l;
        const int i = pi_[p], j = pj_[p];
        if (j < 0 || sn[p] == 0.0) continue;
        const double c = cs[p], s = sn[p];
        const double ti = T[i * ld + col], tj = T[j * ld + col];
        T[i * ld + col] = c * ti - s * tj;
        T[j * ld + col] = s * ti + c * tj;
      }
      __syncthreads();
      for (int e = tid; e < half * l; e += nt) {
        const int p = e / l, r = e - p * l;
        const int i = pi_[p], j = pj_[p];
        if (j < 0 || sn[p] == 0.0) continue;
        const double c = cs[p], s = sn[p];
        const double ti = T[r * ld + i], tj = T[r * ld + j];
        T[r * ld + i] = c * ti - s * tj;
        T[r * ld + j] = s * ti + c * tj;
        const double vi = V[r * ld + i], vj = V[r * ld + j];
        V[r * ld + i] = c * vi - s * vj;
        V[r * ld + j] = s * vi + c * vj;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {   // stable selection by |lambda| descending (Z17)
    for (int i = 0; i < l; ++i) order[i] = i;
    for (int a = 0; a < l; ++a) {
      int best = a;
      for (int b = a + 1; b < l; ++b)
        if (fabs(T[order[b] * ld + order[b]]) > fabs(T[order[best] * ld + order[best]])) best = b;
      const int t = order[best];
      for (int b = best; b > a; --b) order[b] = order[b - 1];
      order[a] = t;
    }
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += nt) {
    const int r = e / l, c = e - r * l;
    Vout[r * l + c] = V[r * ld + order[c]];
  }
  for (int c = tid; c < l; c += nt) lam[c] = T[order[c] * ld + order[c]];
}

void launch_jacobi_evd(double* T, int l, double* V, double* lambda, int32_t* status, cudaStream_t st) {
  const size_t smem = sizeof(double) * 2 * l * (l + 1);
  cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  jacobi_kernel<<<1, 256, smem, st>>>(T, l, V, lambda, status);
}

}  // namespace symnmf
