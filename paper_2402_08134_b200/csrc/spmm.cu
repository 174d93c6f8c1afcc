// (a10) Exact CSR product Y = A F and (a9) the sampled CSR product
// Y_s = sum_{i in U} omega_i A[i,:]^T f_i (by symmetry
// row i of A equals column i).
//
// Exact: a group of k/4 lanes owns one row; each lane keeps a float4 slice of
// the output row and streams the row's (col, val) pairs with 4-way unrolled
// independent gathers of F rows (128-bit loads).  Sampled: one warp per
// sampled row; groups of k/4 lanes scatter-add omega_i a_ic f_i into row c of
// Y_s with 128-bit vector atomics (red.global.add.v4.f32).
#include <cstdlib>
#include "kernels.cuh"

namespace symnmf {

template <int LPR>   // lanes per row = k / 4
__global__ void __launch_bounds__(256) spmm_csr_v4(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                                   const float* __restrict__ val, int64_t n,
                                                   const float4* __restrict__ F4, float4* __restrict__ Y4,
                                                   const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int li = threadIdx.x % LPR;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t r = gtid / LPR; r < n; r += ngroups) {
    const int64_t e0 = rowptr[r], e1 = rowptr[r + 1];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t e = e0;
    for (; e + 4 <= e1; e += 4) {
      int c[4];
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { c[u] = __ldg(col + e + u); v[u] = __ldg(val + e + u); }
      float4 f[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) f[u] = __ldg(F4 + (int64_t)c[u] * LPR + li);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x = fmaf(v[u], f[u].x, acc.x); acc.y = fmaf(v[u], f[u].y, acc.y);
        acc.z = fmaf(v[u], f[u].z, acc.z); acc.w = fmaf(v[u], f[u].w, acc.w);
      }
    }
    for (; e < e1; ++e) {
      const int c = __ldg(col + e);
      const float v = __ldg(val + e);
      const float4 f = __ldg(F4 + (int64_t)c * LPR + li);
      acc.x = fmaf(v, f.x, acc.x); acc.y = fmaf(v, f.y, acc.y);
      acc.z = fmaf(v, f.z, acc.z); acc.w = fmaf(v, f.w, acc.w);
    }
    Y4[r * LPR + li] = acc;
  }
}

// Generic k (k % 4 != 0): one warp per row, lane j owns columns j and j + 32.
__global__ void __launch_bounds__(256) spmm_csr_scalar(const int64_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ col, const float* __restrict__ val,
                                                       int64_t n, const float* __restrict__ F, int k,
                                                       float* __restrict__ Y, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    float a0 = 0.f, a1 = 0.f;
    for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
      const int64_t c = __ldg(col + e);
      const float v = __ldg(val + e);
      if (lane < k) a0 = fmaf(v, __ldg(F + c * k + lane), a0);
      if (lane + 32 < k) a1 = fmaf(v, __ldg(F + c * k + lane + 32), a1);
    }
    if (lane < k) Y[r * k + lane] = a0;
    if (lane + 32 < k) Y[r * k + lane + 32] = a1;
  }
}

// Y slice per scatter pass (L2 is 126 MB); SYMNMF_SCATTER_SLICE_MB overrides (symnmf.h).
// Measured on c4 (Y = 256 MB), LvS it/s by slice: 48 MB 425, 64 MB 433, 86 MB 435, 128 MB 427,
// 256 MB (one pass) 400 -- every pass rescans the sampled nonzeros, so fewer passes win until the
// slice stops fitting in L2 next to the streamed rows of A.
static bool scatter_shfl();
static bool scatter_merge();
// Rows of Y per destination-range pass.  Passes launched one by one: 86 MB (43/64/86/128 MB: 0.47/0.35/
// 0.35/0.39 ms per c4 half).  Passes merged into one launch (k in {16, 32, 64}): 48 MB -- two adjacent
// slices fit L2 while the tail of a pass overlaps the head of the next (86/64/52/43/32 MB:
// 0.309/0.291/0.287/0.290/0.309 ms).
static int64_t scatter_slice_bytes(int k) {
  const char* e = getenv("SYMNMF_SCATTER_SLICE_MB");
  const int64_t mb = e ? atoll(e) : 0;
  if (mb > 0) return mb << 20;
  const bool merged = (k == 16 || k == 32 || k == 64) && scatter_shfl() && scatter_merge();
  return (merged ? 48ll : 86ll) << 20;   // c4 with 2 warps per row and pass: 48 MB (6 passes) 0.276, 52-60 MB (5) 0.282 ms
}

// Warps per sampled row of the scatter; SYMNMF_SCATTER_SPLIT overrides (symnmf.h).
static int scatter_split(int k) {
  const char* e = getenv("SYMNMF_SCATTER_SPLIT");
  const int v = e ? atoi(e) : 0;
  // c4 LvS it/s by split, three 86 MB passes launched one by one: 1 565, 2 583, 4 614, 8 598, 16 545;
  // five merged 52 MB passes (a row's per-pass segment is shorter): 1 728, 2 738, 3 738, 4 731, 8 653
  if (v > 0) return std::min(v, 64);
  return (k == 16 || k == 32 || k == 64) && scatter_shfl() && scatter_merge() ? 2 : 4;
}

// Coalesced + shuffled entry loads in the scatter (sampled_csr_v4s, the default for k in {16, 32, 64}
// when the pass bounds are precomputed or there is one pass); SYMNMF_SCATTER_SHFL=0 restores the
// broadcast loads.  c4 LvS: 662 / 664 vs 675 / 675 it/s (scatter 0.350-0.360 vs 0.345-0.347 ms per half).
static bool scatter_shfl() {
  const char* e = getenv("SYMNMF_SCATTER_SHFL");
  return !e || atoi(e) != 0;
}

// All destination passes of the shuffled scatter in one launch (block range p = pass p), the default;
// SYMNMF_SCATTER_MERGE=0 launches them one by one.  c4: scatter 0.345 -> 0.308 ms per half, LvS 675 -> 711 it/s.
static bool scatter_merge() {
  const char* e = getenv("SYMNMF_SCATTER_MERGE");
  return !e || atoi(e) != 0;
}

static int grid_for(int64_t work_threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work_threads + 255) / 256, 148 * 16));
}

void launch_spmm_csr(const symnmf_matrix& A, const float* F, int k, float* Y, const int32_t* status, cudaStream_t st) {
  const int64_t n = A.n;
  if (k % 4 == 0) {
    const int lpr = k / 4;
    const int grid = grid_for(n * lpr);
    const float4* F4 = reinterpret_cast<const float4*>(F);
    float4* Y4 = reinterpret_cast<float4*>(Y);
    switch (lpr) {
      case 1: launch_pdl(spmm_csr_v4<1>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, n, F4, Y4, status); return;
      case 2: launch_pdl(spmm_csr_v4<2>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, n, F4, Y4, status); return;
      case 4: launch_pdl(spmm_csr_v4<4>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, n, F4, Y4, status); return;
      case 8: launch_pdl(spmm_csr_v4<8>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, n, F4, Y4, status); return;
      case 16: launch_pdl(spmm_csr_v4<16>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, n, F4, Y4, status); return;
      default: break;
    }
  }
  launch_pdl(spmm_csr_scalar, grid_for(n * 32), 256, 0, st, A.rowptr, A.colidx, A.val, n, F, k, Y, status);
}

// ---------------------------------------------------------------- sampled (scatter) product
// One warp per (sampled row u, part): the row's nonzeros in this pass's destination range are cut
// into `split` contiguous parts, so a hub row (10^4 nonzeros at c4) is spread over several warps
// instead of serialising one; each lane keeps SC_UNROLL entry loads in flight ahead of its vector
// atomics (the per-step load -> red dependency bound the single-warp walk: ncu r2, long_scoreboard
// 22 cycles per issued instruction, 20% warps active).
constexpr int SC_UNROLL = 8;

template <int LPR>
__global__ void __launch_bounds__(256) sampled_csr_v4(const int64_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ col, const float* __restrict__ val,
                                                      const float4* __restrict__ F4, const int32_t* __restrict__ uniq,
                                                      const double* __restrict__ w,
                                                      const int64_t* __restrict__ n_uniq_dev, float4* __restrict__ Y4,
                                                      int32_t c_lo, int32_t c_hi, int ranged, int split,
                                                      const int32_t* __restrict__ ppos, int pass, int64_t n,
                                                      const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  constexpr int NPW = 32 / LPR;   // nonzeros per warp step
  const int lane = threadIdx.x & 31, sub = lane / LPR, li = lane % LPR;
  const int64_t nu = *n_uniq_dev;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nu * split; t += nw) {
    const int64_t u = t / split;
    const int part = (int)(t - u * split);
    const int64_t i = uniq[u];
    int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
    if (ranged && ppos) {   // the pass boundaries of row i, found once per A (sampled_pass_bounds)
      const int64_t base = e0;
      if (pass > 0) e0 = base + ppos[(int64_t)(pass - 1) * n + i];
      if (ppos[(int64_t)pass * n + i] >= 0) e1 = base + ppos[(int64_t)pass * n + i];
    } else if (ranged) {   // this pass's destination range [c_lo, c_hi): a sub-range of the sorted row
      int64_t a = e0, b = e1;
      while (a < b) { const int64_t m = (a + b) >> 1; if (__ldg(col + m) < c_lo) a = m + 1; else b = m; }
      int64_t c = a, d = e1;
      while (c < d) { const int64_t m = (c + d) >> 1; if (__ldg(col + m) < c_hi) c = m + 1; else d = m; }
      e0 = a; e1 = c;
    }
    const int64_t len = e1 - e0;
    const int64_t p0 = e0 + len * part / split, p1 = e0 + len * (part + 1) / split;
    if (p0 >= p1) continue;
    const float om = (float)w[u];
    float4 f = __ldg(F4 + i * LPR + li);
    f.x *= om; f.y *= om; f.z *= om; f.w *= om;
    for (int64_t e = p0 + sub; e < p1; e += NPW * SC_UNROLL) {
      int cc[SC_UNROLL];
      float aa[SC_UNROLL];
#pragma unroll
      for (int j = 0; j < SC_UNROLL; ++j) {
        const int64_t ej = e + (int64_t)j * NPW;
        const bool ok = ej < p1;
        cc[j] = ok ? __ldg(col + ej) : -1;
        aa[j] = ok ? __ldg(val + ej) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < SC_UNROLL; ++j)
        if (cc[j] >= 0)
          atomicAdd(Y4 + (int64_t)cc[j] * LPR + li, make_float4(aa[j] * f.x, aa[j] * f.y, aa[j] * f.z, aa[j] * f.w));
    }
  }
}

// Default for k in {16, 32, 64} (SYMNMF_SCATTER_SHFL=0 disables): the warp loads 32 consecutive entries of its part coalesced (one
// col and one val load per lane instead of 8 broadcast loads per lane group), the next 32 before this
// batch's atomics, and the lane groups take their entries by shuffle.
template <int LPR>
__global__ void __launch_bounds__(256) sampled_csr_v4s(
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, const float* __restrict__ val,
    const float4* __restrict__ F4, const int32_t* __restrict__ uniq, const double* __restrict__ w,
    const int64_t* __restrict__ n_uniq_dev, float4* __restrict__ Y4, int split, const int32_t* __restrict__ ppos,
    int pass, int merged, int64_t n, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  constexpr int NPW = 32 / LPR;   // nonzeros per warp step
  const int lane = threadIdx.x & 31, sub = lane / LPR, li = lane % LPR;
  const int64_t nu = *n_uniq_dev;
  // merged > 1: one launch for all `merged` destination passes, block range p of the grid working on
  // pass p -- CTAs are dispatched in block order, so the passes still run one after the other (each
  // slice of Y L2-resident while its atomics land), but the tail of a pass overlaps the head of the next
  const int gpp = merged > 1 ? gridDim.x / merged : gridDim.x;
  if (merged > 1) pass = blockIdx.x / gpp;
  const int64_t nw = ((int64_t)gpp * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)(blockIdx.x - pass * (merged > 1 ? gpp : 0)) * blockDim.x + threadIdx.x) >> 5;
       t < nu * split; t += nw) {
    const int64_t u = t / split;
    const int part = (int)(t - u * split);
    const int64_t i = uniq[u];
    int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
    if (ppos) {   // the pass boundaries of row i, found once per A (sampled_pass_bounds)
      const int64_t base = e0;
      if (pass > 0) e0 = base + ppos[(int64_t)(pass - 1) * n + i];
      if (ppos[(int64_t)pass * n + i] >= 0) e1 = base + ppos[(int64_t)pass * n + i];
    }
    const int64_t len = e1 - e0;
    const int64_t p0 = e0 + len * part / split, p1 = e0 + len * (part + 1) / split;
    if (p0 >= p1) continue;
    int cl = -1;
    float al = 0.f;
    if (p0 + lane < p1) { cl = __ldg(col + p0 + lane); al = __ldg(val + p0 + lane); }
    const float om = (float)w[u];
    float4 f = __ldg(F4 + i * LPR + li);
    f.x *= om; f.y *= om; f.z *= om; f.w *= om;
    for (int64_t e = p0; e < p1; e += 32) {
      const int cc = cl;
      const float ac = al;
      cl = -1; al = 0.f;
      if (e + 32 + lane < p1) { cl = __ldg(col + e + 32 + lane); al = __ldg(val + e + 32 + lane); }
#pragma unroll
      for (int j = 0; j < LPR; ++j) {
        const int c = __shfl_sync(0xffffffffu, cc, sub + j * NPW);
        const float a = __shfl_sync(0xffffffffu, ac, sub + j * NPW);
        if (c >= 0) atomicAdd(Y4 + (int64_t)c * LPR + li, make_float4(a * f.x, a * f.y, a * f.z, a * f.w));
      }
    }
  }
}

__global__ void __launch_bounds__(256) sampled_csr_scalar(const int64_t* __restrict__ rowptr,
                                                          const int32_t* __restrict__ col,
                                                          const float* __restrict__ val, const float* __restrict__ F,
                                                          int k, const int32_t* __restrict__ uniq,
                                                          const double* __restrict__ w,
                                                          const int64_t* __restrict__ n_uniq_dev,
                                                          float* __restrict__ Y, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int lane = threadIdx.x & 31;
  const int64_t nu = *n_uniq_dev;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nu; u += nw) {
    const int64_t i = uniq[u];
    const float om = (float)w[u];
    const float f0 = lane < k ? om * F[i * k + lane] : 0.f;
    const float f1 = lane + 32 < k ? om * F[i * k + lane + 32] : 0.f;
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int64_t c = __ldg(col + e);
      const float a = __ldg(val + e);
      if (lane < k) atomicAdd(Y + c * k + lane, a * f0);
      if (lane + 32 < k) atomicAdd(Y + c * k + lane + 32, a * f1);
    }
  }
}

void launch_sampled_csr(const symnmf_matrix& A, const float* F, int k, const int32_t* uniq, const double* w,
                        const int64_t* n_uniq_dev, int64_t cap, float* Y, const int32_t* status, cudaStream_t st) {
  cudaMemsetAsync(Y, 0, sizeof(float) * (size_t)A.n * k, st);
  launch_sampled_csr_nozero(A, F, k, uniq, w, n_uniq_dev, cap, Y, status, st);
}

// Destination-range passes of the scatter for this A and k (>= 1).
int sampled_csr_passes(int64_t n, int k) {
  const int64_t ybytes = (int64_t)sizeof(float) * n * k;
  const int64_t slice = scatter_slice_bytes(k);
  return (int)std::max<int64_t>(1, (ybytes + slice - 1) / slice);
}

// ppos[p][i] (p < passes - 1) = offset within row i of its first entry with column >= the start of
// pass p + 1 (row columns sorted); the last pass ends at the row end (ppos row passes - 1 = -1).
// Once per A: the scatter then reads a row's in-range sub-range instead of binary-searching it in
// every pass (two dependent log2(deg) load chains per warp and pass, measured ~1/3 of the c4 scatter).
__global__ void sampled_pass_bounds_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                           int64_t n, int passes, int32_t* __restrict__ ppos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
  int64_t a = e0;
  for (int p = 0; p < passes; ++p) {
    if (p == passes - 1) { ppos[(int64_t)p * n + i] = -1; break; }
    const int32_t hi = (int32_t)(n * (p + 1) / passes);
    int64_t b = e1;
    while (a < b) { const int64_t m = (a + b) >> 1; if (col[m] < hi) a = m + 1; else b = m; }
    ppos[(int64_t)p * n + i] = (int32_t)(a - e0);
  }
}

void launch_sampled_pass_bounds(const symnmf_matrix& A, int k, int32_t* ppos, cudaStream_t st) {
  const int passes = sampled_csr_passes(A.n, k);
  if (passes > 1 && A.n > 0)
    sampled_pass_bounds_kernel<<<(unsigned)((A.n + 255) / 256), 256, 0, st>>>(A.rowptr, A.colidx, A.n, passes, ppos);
}

void launch_sampled_csr_nozero(const symnmf_matrix& A, const float* F, int k, const int32_t* uniq, const double* w,
                               const int64_t* n_uniq_dev, int64_t cap, float* Y, const int32_t* status,
                               cudaStream_t st, const int32_t* ppos) {
  const int grid = grid_for(std::max<int64_t>(cap, 1) * 32);
  if (k % 4 == 0) {
    const float4* F4 = reinterpret_cast<const float4*>(F);
    float4* Y4 = reinterpret_cast<float4*>(Y);
    // Destination-range passes: each pass scatters only into rows [c_lo, c_hi) of Y, a slice
    // small enough to stay resident in L2 (126 MB) while the pass's vector atomics land on it,
    // instead of read-modify-writes of random 128-byte lines of a Y larger than L2.
    const int passes = sampled_csr_passes(A.n, k);
    const int split = scatter_split(k);
    const bool shfl = scatter_shfl();
    for (int p = 0; p < passes; ++p) {
      const int32_t lo = (int32_t)(A.n * p / passes), hi = (int32_t)(A.n * (p + 1) / passes);
      const int ranged = passes > 1;
      if (shfl && (!ranged || ppos) && (k == 16 || k == 32 || k == 64)) {
        const int32_t* pp = ranged ? ppos : nullptr;
        const int merged = ranged && scatter_merge() ? passes : 1;
        const int g = grid * merged;   // 6 / 8 / 12 / 16 CTAs per SM and pass: 0.297 / 0.290 / 0.288 / 0.288 ms
        if (k == 16) launch_pdl(sampled_csr_v4s<4>, g, 256, 0, st, A.rowptr, A.colidx, A.val, F4, uniq, w, n_uniq_dev, Y4, split, pp, p, merged, A.n, status);
        else if (k == 32) launch_pdl(sampled_csr_v4s<8>, g, 256, 0, st, A.rowptr, A.colidx, A.val, F4, uniq, w, n_uniq_dev, Y4, split, pp, p, merged, A.n, status);
        else launch_pdl(sampled_csr_v4s<16>, g, 256, 0, st, A.rowptr, A.colidx, A.val, F4, uniq, w, n_uniq_dev, Y4, split, pp, p, merged, A.n, status);
        if (merged > 1) break;
        continue;
      }
      switch (k / 4) {
        case 1: launch_pdl(sampled_csr_v4<1>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, F4, uniq, w, n_uniq_dev, Y4, lo, hi, ranged, split, ppos, p, A.n, status); break;
        case 2: launch_pdl(sampled_csr_v4<2>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, F4, uniq, w, n_uniq_dev, Y4, lo, hi, ranged, split, ppos, p, A.n, status); break;
        case 4: launch_pdl(sampled_csr_v4<4>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, F4, uniq, w, n_uniq_dev, Y4, lo, hi, ranged, split, ppos, p, A.n, status); break;
        case 8: launch_pdl(sampled_csr_v4<8>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, F4, uniq, w, n_uniq_dev, Y4, lo, hi, ranged, split, ppos, p, A.n, status); break;
        case 16: launch_pdl(sampled_csr_v4<16>, grid, 256, 0, st, A.rowptr, A.colidx, A.val, F4, uniq, w, n_uniq_dev, Y4, lo, hi, ranged, split, ppos, p, A.n, status); break;
        default: break;
      }
    }
    if (k / 4 <= 16 && (k / 4 & (k / 4 - 1)) == 0) return;
  }
  launch_pdl(sampled_csr_scalar, grid, 256, 0, st, A.rowptr, A.colidx, A.val, F, k, uniq, w, n_uniq_dev, Y, status);
}


}  // namespace symnmf
