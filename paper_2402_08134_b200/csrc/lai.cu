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
// Y = X M (X n x ka fp32, M ka x kb in MT = float or double, Y n x kb fp32, MT accumulation).
// Persistent CTAs of 8 warps; M staged once per CTA in shared memory (ka rounded up to 4, zero
// padded).  A warp owns 8 rows at a time (staged in its own shared-memory slice, 4 values of a row
// per broadcast LDS.128); lane j computes columns cb*32 + j of the 8 rows, so M is read
// conflict-free and Y is stored coalesced.  (Was: lane = row, 4 warps per SM at 133 KB of shared
// memory per CTA -- 0.29 ms per fp64 apply at n = 60,000, l = 74; verdict r1.)
constexpr int RW = 8;    // warps per CTA
constexpr int RR = 8;    // rows per warp step

template <typename MT, int NCB>
__global__ void __launch_bounds__(RW * 32) rowapply_kernel(const float* __restrict__ X, int64_t ldx, int64_t n, int ka,
                                                           const MT* __restrict__ M, int kb, float* __restrict__ Y,
                                                           int64_t ldy, const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smr[];
  if (dev_failed(status)) return;
  constexpr int KBP = NCB * 32;
  const int ka4 = (ka + 3) & ~3;
  MT* sM = reinterpret_cast<MT*>(smr);                                   // [ka4][KBP]
  float* sXall = reinterpret_cast<float*>(smr + sizeof(MT) * ka4 * KBP);  // [RW][RR][ka4]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  float* sX = sXall + wid * RR * ka4;
  for (int e = tid; e < ka4 * KBP; e += RW * 32) {
    const int a = e / KBP, b = e - a * KBP;
    sM[e] = (a < ka && b < kb) ? M[a * kb + b] : MT(0);
  }
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * RW;
  for (int64_t base = ((int64_t)blockIdx.x * RW + wid) * RR; base < n; base += nwarps * RR) {
    const int cnt = (int)min64(RR, n - base);
    for (int e = lane; e < RR * ka4; e += 32) {
      const int r = e / ka4, c = e - r * ka4;
      sX[e] = (r < cnt && c < ka) ? X[(base + r) * ldx + c] : 0.f;
    }
    __syncwarp();
    MT acc[RR][NCB];
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
      for (int q = 0; q < NCB; ++q) acc[r][q] = MT(0);
    for (int a = 0; a < ka4; a += 4) {
      MT m[4][NCB];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int q = 0; q < NCB; ++q) m[t][q] = sM[(a + t) * KBP + q * 32 + lane];
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const float4 x = *reinterpret_cast<const float4*>(sX + r * ka4 + a);
        const MT xv[4] = {(MT)x.x, (MT)x.y, (MT)x.z, (MT)x.w};
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int q = 0; q < NCB; ++q) acc[r][q] += xv[t] * m[t][q];
      }
    }
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
      for (int q = 0; q < NCB; ++q) {
        const int col = q * 32 + lane;
        if (r < cnt && col < kb) Y[(base + r) * ldy + col] = (float)acc[r][q];
      }
    __syncwarp();
  }
}

template <typename MT, int NCB>
static void launch_rowapply_n(const float* X, int64_t ldx, int64_t n, int ka, const MT* M, int kb, float* Y,
                              int64_t ldy, const int32_t* status, cudaStream_t st) {
  const int ka4 = (ka + 3) & ~3;
  const size_t smem = sizeof(MT) * ka4 * NCB * 32 + sizeof(float) * RW * RR * ka4;
  cudaFuncSetAttribute(rowapply_kernel<MT, NCB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rowapply_kernel<MT, NCB>, RW * 32, smem);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + RW * RR - 1) / (RW * RR), 148 * std::max(1, occ)));
  rowapply_kernel<MT, NCB><<<(unsigned)blocks, RW * 32, smem, st>>>(X, ldx, n, ka, M, kb, Y, ldy, status);
}

template <typename MT>
static void launch_rowapply_t(const float* X, int64_t ldx, int64_t n, int ka, const MT* M, int kb, float* Y,
                              int64_t ldy, const int32_t* status, cudaStream_t st) {
  if (kb <= 32) launch_rowapply_n<MT, 1>(X, ldx, n, ka, M, kb, Y, ldy, status, st);
  else if (kb <= 64) launch_rowapply_n<MT, 2>(X, ldx, n, ka, M, kb, Y, ldy, status, st);
  else launch_rowapply_n<MT, 3>(X, ldx, n, ka, M, kb, Y, ldy, status, st);
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

__global__ void __launch_bounds__(1024) jacobi_kernel(const double* __restrict__ Tin, int l, double* __restrict__ Vout,
                                                     double* __restrict__ lam, int32_t* __restrict__ status) {
  extern __shared__ double sj[];
  __shared__ double cs[kMaxL / 2 + 1], sn[kMaxL / 2 + 1];
  __shared__ int pi_[kMaxL / 2 + 1], pj_[kMaxL / 2 + 1];
  __shared__ double red[32];
  __shared__ int done;
  __shared__ int order[kMaxL];
  if (dev_failed(status)) return;
  const int ld = l + 1, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
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
      // rows i, j of T for every pair: warp w takes pairs w, w + nw, ..., lanes the columns
      for (int p = wid; p < half; p += nw) {
        const int i = pi_[p], j = pj_[p];
        if (j < 0 || sn[p] == 0.0) continue;
        const double c = cs[p], s = sn[p];
        for (int col = lane; col < l; col += 32) {
          const double ti = T[i * ld + col], tj = T[j * ld + col];
          T[i * ld + col] = c * ti - s * tj;
          T[j * ld + col] = s * ti + c * tj;
        }
      }
      __syncthreads();
      // columns i, j of T and of V
      for (int p = wid; p < half; p += nw) {
        const int i = pi_[p], j = pj_[p];
        if (j < 0 || sn[p] == 0.0) continue;
        const double c = cs[p], s = sn[p];
        for (int r = lane; r < l; r += 32) {
          const double ti = T[r * ld + i], tj = T[r * ld + j];
          T[r * ld + i] = c * ti - s * tj;
          T[r * ld + j] = s * ti + c * tj;
          const double vi = V[r * ld + i], vj = V[r * ld + j];
          V[r * ld + i] = c * vi - s * vj;
          V[r * ld + j] = s * vi + c * vj;
        }
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
  jacobi_kernel<<<1, 1024, smem, st>>>(T, l, V, lambda, status);
}

}  // namespace symnmf
