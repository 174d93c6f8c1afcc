// NEXT-1: Update(G + alpha I, Y + alpha F^T) by exact per-row NLS -- the ANLS update the paper
// uses with block principal pivoting (App. G; Kim & Park's full exchange with
// the backup rule, cited but not restated by the paper):
//   row r:  min_{x >= 0} x^T Gh x - 2 b^T x,   Gh = G + alpha I,  b = Y_r + alpha F_r.
// One warp per row; lane c owns variables c and c + 32 (k <= 64).  Each pivoting step solves only
// the passive-set system Gh_FF x_F = b_F: the passive indices are compacted (ballot + popc), the
// |F| x |F| system is gathered from Gh (shared by the CTA, fp64, padded rows) into the warp's own
// shared-memory block, factored by a lane-per-row Cholesky and solved by two substitutions -- so a
// step costs O(|F|^2) lane work instead of a k x k refactorisation, and SymNMF rows have small
// passive sets.  The dual y = Gh x - b of the active variables reads Gh's rows at the |F| passive
// columns.  The pivoting starts from the support of one HALS sweep of the row (see below).
// Optionally re-zeroes Y (the LvS scatter target) after reading it.
#include "fused_common.cuh"

namespace symnmf {

constexpr int kBppMaxIt = 256;    // pivoting steps per row before the row is reported

template <int KP>
struct BppL {
  static constexpr int WPB = KP <= 32 ? 8 : 2;        // warps (rows in flight) per CTA
  static constexpr int GS = KP + 1;                   // padded row stride of Gh / M (doubles)
  static constexpr size_t g = 0;                                          // Gh  [KP][GS]
  static constexpr size_t m = g + sizeof(double) * KP * GS;               // M   [WPB][KP][GS]
  static constexpr size_t v = m + sizeof(double) * WPB * KP * GS;         // rhs / z / x [WPB][3][KP]
  static constexpr size_t idx = v + sizeof(double) * WPB * 3 * KP;        // passive list [WPB][KP]
  static constexpr size_t bytes = idx + sizeof(int) * WPB * KP;
};

template <int KP>
__global__ void __launch_bounds__(BppL<KP>::WPB * 32) bpp_rows(const double* __restrict__ G, float* __restrict__ Y,
                                                                const float* __restrict__ F, float* __restrict__ X,
                                                                int64_t n, int k, double alpha, int zeroY,
                                                                int32_t* __restrict__ nonconv, int32_t* status) {
  using L = BppL<KP>;
  constexpr int GS = L::GS, H = KP > 32 ? 2 : 1;    // variables per lane
  extern __shared__ __align__(16) unsigned char smb[];
  double* sG = reinterpret_cast<double*>(smb + L::g);
  if (dev_failed(status)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* M = reinterpret_cast<double*>(smb + L::m) + (size_t)wid * KP * GS;
  double* rhs = reinterpret_cast<double*>(smb + L::v) + (size_t)wid * 3 * KP;
  double* zz = rhs + KP;
  double* xs = zz + KP;
  int* idx = reinterpret_cast<int*>(smb + L::idx) + wid * KP;
  for (int e = threadIdx.x; e < KP * KP; e += blockDim.x) {
    const int i = e / KP, j = e - i * KP;
    sG[i * GS + j] = (i < k && j < k) ? G[i * k + j] + (i == j ? alpha : 0.0) : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  const int64_t nw = (int64_t)gridDim.x * L::WPB;
  for (int64_t r = (int64_t)blockIdx.x * L::WPB + wid; r < n; r += nw) {
    double bh[H], x[H], y[H];
    bool inF[H], act[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int v = lane + 32 * h;
      act[h] = v < k;
      bh[h] = act[h] ? (double)Y[r * k + v] + alpha * (double)F[r * k + v] : 0.0;
      x[h] = act[h] ? (double)X[r * k + v] : 0.0;
    }
    // Initial passive set: the support of one Gauss-Seidel (HALS) sweep of this row from the current
    // X -- usually close to the NNLS support, so the pivoting starts from a small system.
    // BPP converges to the unique NLS solution from any initial passive set (the backup rule
    // guarantees termination), so the start changes the work, not the result.
    for (int i = 0; i < k; ++i) {
      double part = 0.0;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int v = lane + 32 * h;
        if (act[h] && v != i) part = fma(sG[i * GS + v], x[h], part);
      }
      const double sum = warp_sum(part);
      const double xi = fmax(0.0, (__shfl_sync(0xffffffffu, bh[i >> 5], i & 31) - sum) / sG[i * GS + i]);
      if ((i & 31) == lane) x[i >> 5] = xi;
    }
    bool fail = false;
    unsigned Fm[H];
    int pos[H], nf = 0;
    // x_F = Gh_FF^{-1} b_F on the passive set, y = Gh x - b on the active set
    auto solve = [&]() {
      int base = 0;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        Fm[h] = __ballot_sync(0xffffffffu, inF[h]);
        pos[h] = base + __popc(Fm[h] & ((1u << lane) - 1u));
        if (inF[h]) {
          idx[pos[h]] = lane + 32 * h;
          rhs[pos[h]] = bh[h];
        }
        base += __popc(Fm[h]);
      }
      nf = base;
      __syncwarp();
      for (int e = lane; e < nf * nf; e += 32) {   // M = Gh_FF (lower part)
        const int a = e / nf, c = e - a * nf;
        if (c <= a) M[a * GS + c] = sG[idx[a] * GS + idx[c]];
      }
      __syncwarp();
      for (int j = 0; j < nf; ++j) {               // Cholesky M = L L^T, lane-per-row updates
        const double d = M[j * GS + j];
        if (!(d > 0.0) || !isfinite(d)) { fail = true; return; }
        const double rj = sqrt(d), rinv = 1.0 / rj;
        __syncwarp();
        for (int a = j + 1 + lane; a < nf; a += 32) M[a * GS + j] *= rinv;
        if (lane == 0) M[j * GS + j] = rj;
        __syncwarp();
        for (int a = j + 1 + lane; a < nf; a += 32) {
          const double laj = M[a * GS + j];
          for (int c = j + 1; c <= a; ++c) M[a * GS + c] = fma(-laj, M[c * GS + j], M[a * GS + c]);
        }
        __syncwarp();
      }
      for (int a = lane; a < nf; a += 32) zz[a] = rhs[a];   // forward L z = rhs
      __syncwarp();
      for (int j = 0; j < nf; ++j) {
        const double zj = zz[j] / M[j * GS + j];
        __syncwarp();
        if (lane == 0) zz[j] = zj;
        for (int a = j + 1 + lane; a < nf; a += 32) zz[a] = fma(-M[a * GS + j], zj, zz[a]);
        __syncwarp();
      }
      for (int j = nf - 1; j >= 0; --j) {                   // backward L^T x = z
        const double xj = zz[j] / M[j * GS + j];
        __syncwarp();
        if (lane == 0) xs[j] = xj;
        for (int a = lane; a < j; a += 32) zz[a] = fma(-M[j * GS + a], xj, zz[a]);
        __syncwarp();
      }
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int v = lane + 32 * h;
        if (inF[h]) {
          x[h] = xs[pos[h]];
          y[h] = 0.0;
        } else {
          x[h] = 0.0;
          double yy = -bh[h];
          if (act[h])
            for (int q = 0; q < nf; ++q) yy = fma(sG[v * GS + idx[q]], xs[q], yy);
          y[h] = yy;
        }
      }
      __syncwarp();
    };
#pragma unroll
    for (int h = 0; h < H; ++h) inF[h] = act[h] && x[h] > 0.0;
    solve();
    int ninf = k + 1, p = 3, it = 0;
    for (; it < kBppMaxIt && !fail; ++it) {
      unsigned V[H];
      int nv = 0;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        V[h] = __ballot_sync(0xffffffffu, act[h] && (inF[h] ? x[h] < 0.0 : y[h] < 0.0));
        nv += __popc(V[h]);
      }
      if (nv == 0) break;
      if (nv < ninf) { ninf = nv; p = 3; }        // full exchange while the infeasible set shrinks
      else if (p >= 1) { --p; }                   // ... or up to 3 times without progress
      else {                                      // backup rule: exchange only max(V)
        int hmax = H - 1;
        while (hmax > 0 && !V[hmax]) --hmax;
        const unsigned top = 1u << (31 - __clz(V[hmax]));
#pragma unroll
        for (int h = 0; h < H; ++h) V[h] = h == hmax ? top : 0u;
      }
#pragma unroll
      for (int h = 0; h < H; ++h)
        if ((V[h] >> lane) & 1u) inF[h] = !inF[h];
      solve();
    }
    if (fail) {                                   // Gh_FF not SPD (alpha = 0 and rank-deficient G)
      if (lane == 0) dev_fail(status, SYMNMF_ERR_NOT_PD);
      it = kBppMaxIt;
    }
    if (it >= kBppMaxIt && lane == 0) atomicAdd(nonconv, 1);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int v = lane + 32 * h;
      if (act[h]) {
        X[r * k + v] = (float)(x[h] > 0.0 ? x[h] : 0.0);
        if (zeroY) Y[r * k + v] = 0.f;
      }
    }
  }
}

bool bpp_supported(int k) { return k >= 1 && k <= 64; }

template <int KP>
static void launch_bpp_t(const double* G, float* Y, const float* F, float* X, int64_t n, int k, double alpha,
                         bool zeroY, int32_t* nonconv, int32_t* status, cudaStream_t st) {
  using L = BppL<KP>;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + L::WPB - 1) / L::WPB, 148 * 8));
  cudaFuncSetAttribute(bpp_rows<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes);
  launch_pdl(bpp_rows<KP>, grid, L::WPB * 32, L::bytes, st, G, Y, F, X, n, k, alpha, zeroY ? 1 : 0, nonconv, status);
}

void launch_bpp(const double* G, float* Y, const float* F, float* X, int64_t n, int k, double alpha, bool zeroY,
                int32_t* nonconv, int32_t* status, cudaStream_t st) {
  switch (kpad(k)) {
    case 8: launch_bpp_t<8>(G, Y, F, X, n, k, alpha, zeroY, nonconv, status, st); break;
    case 16: launch_bpp_t<16>(G, Y, F, X, n, k, alpha, zeroY, nonconv, status, st); break;
    case 32: launch_bpp_t<32>(G, Y, F, X, n, k, alpha, zeroY, nonconv, status, st); break;
    default: launch_bpp_t<64>(G, Y, F, X, n, k, alpha, zeroY, nonconv, status, st); break;
  }
}

}  // namespace symnmf
