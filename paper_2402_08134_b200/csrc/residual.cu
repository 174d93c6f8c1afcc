// (a15) Normalised residual ||A - H H^T||_F / ||A||_F (Eq. 2.2).
// Dense: the direct definition, sum_ij (A_ij - h_i . h_j)^2 with fp64 accumulation.
// CSR: the trace identity of App. C.2, ||A||^2 - 2 tr(H^T (A H)) + ||H^T H||^2,
// every sum in fp64 (fixed-order, deterministic combine).
#include "kernels.cuh"

namespace symnmf {

constexpr int RB_ROWS = 32, RB_COLS = 128;

template <int KP>
__global__ void __launch_bounds__(256) resid_dense_partial(const float* __restrict__ A, int64_t lda, int64_t n,
                                                           const float* __restrict__ H, int k,
                                                           double* __restrict__ partial,
                                                           const int32_t* __restrict__ status) {
  __shared__ float sHr[RB_ROWS][KP];
  __shared__ float sHc[RB_COLS][KP + 1];
  __shared__ double red[32];
  if (dev_failed(status)) return;
  const int tid = threadIdx.x, tc = tid & (RB_COLS - 1), tr = tid >> 7;
  double d2 = 0.0, a2 = 0.0;
  const int64_t rtiles = (n + RB_ROWS - 1) / RB_ROWS;
  for (int64_t rt = blockIdx.x; rt < rtiles; rt += gridDim.x) {
    const int64_t r0 = rt * RB_ROWS;
    __syncthreads();
    for (int e = tid; e < RB_ROWS * KP; e += 256) {
      const int r = e / KP, a = e - r * KP;
      sHr[r][a] = (r0 + r < n && a < k) ? H[(r0 + r) * k + a] : 0.f;
    }
    for (int64_t c0 = 0; c0 < n; c0 += RB_COLS) {
      __syncthreads();
      for (int e = tid; e < RB_COLS * KP; e += 256) {
        const int c = e / KP, a = e - c * KP;
        sHc[c][a] = (c0 + c < n && a < k) ? H[(c0 + c) * k + a] : 0.f;
      }
      __syncthreads();
      const int64_t c = c0 + tc;
      if (c < n) {
        for (int r = tr; r < RB_ROWS; r += 2) {
          if (r0 + r >= n) break;
          float dot = 0.f;
#pragma unroll
          for (int a = 0; a < KP; ++a) dot = fmaf(sHr[r][a], sHc[tc][a], dot);
          const double av = (double)A[(r0 + r) * lda + c];
          const double d = av - (double)dot;
          d2 += d * d;
          a2 += av * av;
        }
      }
    }
  }
  d2 = block_sum(d2, red);
  a2 = block_sum(a2, red);
  if (tid == 0) { partial[2 * blockIdx.x] = d2; partial[2 * blockIdx.x + 1] = a2; }
}

__global__ void resid_dense_final(const double* __restrict__ partial, int grid, double* __restrict__ out,
                                  const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  if (threadIdx.x != 0) return;
  double d2 = 0.0, a2 = 0.0;
  for (int b = 0; b < grid; ++b) { d2 += partial[2 * b]; a2 += partial[2 * b + 1]; }
  out[0] = sqrt(d2) / sqrt(a2);
  out[1] = a2;
  out[2] = nan("");
  out[3] = nan("");
}

__global__ void __launch_bounds__(256) resid_csr_partial(const float* __restrict__ val, int64_t nnz,
                                                         const float* __restrict__ H, const float* __restrict__ AH,
                                                         int64_t nk, double* __restrict__ partial,
                                                         const int32_t* __restrict__ status) {
  __shared__ double red[32];
  if (dev_failed(status)) return;
  double a2 = 0.0, tr = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += stride) {
    const double v = val[e];
    a2 += v * v;
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nk; e += stride)
    tr += (double)H[e] * (double)AH[e];
  a2 = block_sum(a2, red);
  tr = block_sum(tr, red);
  if (threadIdx.x == 0) { partial[2 * blockIdx.x] = a2; partial[2 * blockIdx.x + 1] = tr; }
}

__global__ void resid_csr_final(const double* __restrict__ partial, int grid, const double* __restrict__ G, int k,
                                double* __restrict__ out, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  if (threadIdx.x != 0) return;
  double a2 = 0.0, tr = 0.0, g2 = 0.0;
  for (int b = 0; b < grid; ++b) { a2 += partial[2 * b]; tr += partial[2 * b + 1]; }
  for (int e = 0; e < k * k; ++e) g2 += G[e] * G[e];
  const double r2 = a2 - 2.0 * tr + g2;
  out[0] = sqrt(r2 > 0.0 ? r2 : 0.0) / sqrt(a2);
  out[1] = a2;
  out[2] = tr;
  out[3] = g2;
}

// NEXT-3: projected-gradient norm of the SymNMF objective (App. D):
// grad = 4 (H (H^T H) - A H), computed per entry in fp64 from the fp32 H, AH and
// the fp64 Gram; the KKT mask keeps grad_ij if grad_ij < 0 or H_ij > 0.
// partial[2b] = sum of masked grad^2, partial[2b+1] = sum of grad^2 over block b's rows.
template <int KP>
__global__ void __launch_bounds__(256) pgrad_partial(const float* __restrict__ H, const float* __restrict__ AH,
                                                     const double* __restrict__ G, int64_t n, int k,
                                                     double* __restrict__ partial, const int32_t* __restrict__ status) {
  __shared__ double sG[KP * KP];
  __shared__ double red[32];
  if (dev_failed(status)) return;
  for (int e = threadIdx.x; e < KP * KP; e += blockDim.x) {
    const int a = e / KP, b = e - a * KP;
    sG[e] = (a < k && b < k) ? G[a * k + b] : 0.0;
  }
  __syncthreads();
  double p2 = 0.0, g2 = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double h[KP];
#pragma unroll
    for (int a = 0; a < KP; ++a) h[a] = a < k ? (double)H[r * k + a] : 0.0;
#pragma unroll 1
    for (int j = 0; j < k; ++j) {
      double hg = 0.0;
#pragma unroll
      for (int a = 0; a < KP; ++a) hg = fma(h[a], sG[a * KP + j], hg);
      const double g = 4.0 * (hg - (double)AH[r * k + j]);
      g2 += g * g;
      if (g < 0.0 || H[r * k + j] > 0.f) p2 += g * g;   // KKT mask
    }
  }
  p2 = block_sum(p2, red);
  g2 = block_sum(g2, red);
  if (threadIdx.x == 0) { partial[2 * blockIdx.x] = p2; partial[2 * blockIdx.x + 1] = g2; }
}

__global__ void pgrad_final(const double* __restrict__ partial, int grid, double* __restrict__ out,
                            const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  if (threadIdx.x != 0) return;
  double p2 = 0.0, g2 = 0.0;
  for (int b = 0; b < grid; ++b) { p2 += partial[2 * b]; g2 += partial[2 * b + 1]; }
  out[0] = sqrt(p2);
  out[1] = sqrt(g2);
}

int pgrad_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 4)); }

void launch_pgrad(const float* H, const float* AH, const double* G, int64_t n, int k, double* partial, int grid,
                  double* out, const int32_t* status, cudaStream_t st) {
  switch (kpad(k)) {
    case 8: pgrad_partial<8><<<grid, 256, 0, st>>>(H, AH, G, n, k, partial, status); break;
    case 16: pgrad_partial<16><<<grid, 256, 0, st>>>(H, AH, G, n, k, partial, status); break;
    case 32: pgrad_partial<32><<<grid, 256, 0, st>>>(H, AH, G, n, k, partial, status); break;
    default: pgrad_partial<64><<<grid, 256, 0, st>>>(H, AH, G, n, k, partial, status); break;
  }
  pgrad_final<<<1, 32, 0, st>>>(partial, grid, out, status);
}

// Sum of squares of a rows x cols fp32 block with leading dimension ld, fp64 accumulation
// (||A||_F^2 and ||B||_F^2 of Ada-RRF's residual trick).  partial[b] per block,
// out[0] = fixed-order sum of the partials.
__global__ void __launch_bounds__(256) sumsq_partial(const float* __restrict__ X, int64_t rows, int64_t cols,
                                                     int64_t ld, double* __restrict__ partial,
                                                     const int32_t* __restrict__ status) {
  __shared__ double red[32];
  if (dev_failed(status)) return;
  double s = 0.0;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    const double v = (double)X[r * ld + c];
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void sumsq_final(const double* __restrict__ partial, int grid, double* __restrict__ out,
                            const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int b = 0; b < grid; ++b) s += partial[b];
  out[0] = s;
}

int sumsq_grid() { return 148 * 8; }

void launch_sumsq(const float* X, int64_t rows, int64_t cols, int64_t ld, double* partial, double* out,
                  const int32_t* status, cudaStream_t st) {
  sumsq_partial<<<sumsq_grid(), 256, 0, st>>>(X, rows, cols, ld, partial, status);
  sumsq_final<<<1, 32, 0, st>>>(partial, sumsq_grid(), out, status);
}

int residual_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + RB_ROWS - 1) / RB_ROWS, 148 * 4));
}

void launch_residual(const symnmf_matrix& A, const float* H, int k, const float* AH, const double* G,
                     double* partial, int grid, double* out, const int32_t* status, cudaStream_t st) {
  if (A.kind == SYMNMF_DENSE) {
    switch (kpad(k)) {
      case 8: resid_dense_partial<8><<<grid, 256, 0, st>>>(A.val, A.lda, A.n, H, k, partial, status); break;
      case 16: resid_dense_partial<16><<<grid, 256, 0, st>>>(A.val, A.lda, A.n, H, k, partial, status); break;
      case 32: resid_dense_partial<32><<<grid, 256, 0, st>>>(A.val, A.lda, A.n, H, k, partial, status); break;
      default: resid_dense_partial<64><<<grid, 256, 0, st>>>(A.val, A.lda, A.n, H, k, partial, status); break;
    }
    resid_dense_final<<<1, 32, 0, st>>>(partial, grid, out, status);
  } else {
    resid_csr_partial<<<grid, 256, 0, st>>>(A.val, A.nnz, H, AH, A.n * k, partial, status);
    resid_csr_final<<<1, 32, 0, st>>>(partial, grid, G, k, out, status);
  }
}

}  // namespace symnmf
