// NEXT-1: Update(G + alpha I, Y + alpha F^T) by exact per-row NLS -- the ANLS update the paper
// uses with block principal pivoting (App. G; Kim & Park's full exchange with
// the backup rule, cited but not restated by the paper):
//   row r:  min_{x >= 0} x^T Gh x - 2 b^T x,   Gh = G + alpha I,  b = Y_r + alpha F_r.
// One warp per row, lane c <-> variable c (k <= 32).  Each pivoting step factors the passive-set
// system in fp64 registers: the lane-per-column Cholesky (chol_col_pass) of Gh with the active
// rows / columns replaced by the identity and a zero right-hand side there, so x_active = 0 falls
// out of the same solve; forward substitution broadcasts z_j lane by lane, back substitution
// reduces row j of R over the lanes holding it; the dual y = Gh x - b uses Gh from shared memory.
// Optionally re-zeroes Y (the LvS scatter target) after reading it.
#include "fused_common.cuh"

namespace symnmf {

constexpr int BT = 256;           // 8 warps, one row each at a time
constexpr int kBppMaxIt = 256;    // pivoting steps per row before the row is reported

template <int KP>
__global__ void __launch_bounds__(BT, 1) bpp_rows(const double* __restrict__ G, float* __restrict__ Y,
                                                  const float* __restrict__ F, float* __restrict__ X, int64_t n, int k,
                                                  double alpha, int zeroY, int32_t* __restrict__ nonconv,
                                                  int32_t* status) {
  __shared__ double sG[KP * KP];   // Gh padded with the identity
  if (dev_failed(status)) return;
  for (int e = threadIdx.x; e < KP * KP; e += BT) {
    const int i = e / KP, j = e - i * KP;
    sG[e] = (i < k && j < k) ? G[i * k + j] + (i == j ? alpha : 0.0) : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const bool act = lane < k;
  const int64_t nw = (int64_t)gridDim.x * (BT / 32);
  for (int64_t r = (int64_t)blockIdx.x * (BT / 32) + (threadIdx.x >> 5); r < n; r += nw) {
    const double bh = act ? (double)Y[r * k + lane] + alpha * (double)F[r * k + lane] : 0.0;
    // cold start (F empty, x = 0, y = -b): measured faster than starting from the support of the
    // replaced factor, which the sampled LvS problems move from one half to the next
    bool inF = false;
    double x = 0.0, y = -bh;
    int ninf = k + 1, p = 3, it = 0;
    for (; it < kBppMaxIt; ++it) {
      const bool inf = act && (inF ? x < 0.0 : y < 0.0);
      unsigned V = __ballot_sync(0xffffffffu, inf);
      if (!V) break;
      const int nv = __popc(V);
      if (nv < ninf) { ninf = nv; p = 3; }        // full exchange while the infeasible set shrinks
      else if (p >= 1) { --p; }                   // ... or up to 3 times without progress
      else V = 1u << (31 - __clz(V));             // backup rule: exchange only max(V)
      if ((V >> lane) & 1u) inF = !inF;
      const unsigned Fm = __ballot_sync(0xffffffffu, inF);
      // passive-set system: column `lane` of Gh_FF, identity elsewhere
      double b[KP];
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        const bool fi = (Fm >> i) & 1u;
        b[i] = (lane < KP && fi && inF) ? sG[i * KP + lane] : (i == lane ? 1.0 : 0.0);
      }
      double myr = 1.0;
      if (chol_col_pass<KP>(b, lane, myr)) {      // Gh_FF not SPD (alpha = 0 and rank-deficient G)
        if (lane == 0) dev_fail(status, SYMNMF_ERR_NOT_PD);
        it = kBppMaxIt;
        break;
      }
      // R^T z = rhs (forward), R x = z (backward); R column `lane` in b[0..lane]
      double acc = inF ? bh : 0.0, z = 0.0;
#pragma unroll
      for (int j = 0; j < KP; ++j) {
        const double zj = __shfl_sync(0xffffffffu, lane == j ? acc / myr : 0.0, j);
        if (lane == j) z = zj;
        else if (lane > j) acc = fma(-b[j], zj, acc);
      }
      double xv = 0.0;
#pragma unroll
      for (int j = KP - 1; j >= 0; --j) {
        const double s = warp_sum(lane > j && lane < KP ? b[j] * xv : 0.0);   // sum_{i>j} R[j][i] x_i
        if (lane == j) xv = (z - s) / myr;
      }
      x = inF ? xv : 0.0;
      double yy = -bh;
#pragma unroll
      for (int j = 0; j < KP; ++j) {
        const double xj = __shfl_sync(0xffffffffu, x, j);
        if (lane < KP) yy = fma(sG[j * KP + lane], xj, yy);   // Gh symmetric: row j, lane-contiguous
      }
      y = inF ? 0.0 : yy;
    }
    if (it >= kBppMaxIt && lane == 0) atomicAdd(nonconv, 1);
    if (act) {
      X[r * k + lane] = (float)(x > 0.0 ? x : 0.0);
      if (zeroY) Y[r * k + lane] = 0.f;
    }
  }
}

bool bpp_supported(int k) { return k <= 32; }

void launch_bpp(const double* G, float* Y, const float* F, float* X, int64_t n, int k, double alpha, bool zeroY,
                int32_t* nonconv, int32_t* status, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + BT / 32 - 1) / (BT / 32), 148 * 8));
#define SYMNMF_BPP(KP) \
  launch_pdl(bpp_rows<KP>, grid, BT, 0, st, G, Y, F, X, n, k, alpha, zeroY ? 1 : 0, nonconv, status)
  switch (kpad(k)) {
    case 8: SYMNMF_BPP(8); break;
    case 16: SYMNMF_BPP(16); break;
    default: SYMNMF_BPP(32); break;
  }
#undef SYMNMF_BPP
}

}  // namespace symnmf
