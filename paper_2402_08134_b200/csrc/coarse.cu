// (a9) The sampled CSR product Y_s = sum_{i in U} omega_i A[i,:]^T f_i
// for large graphs, as a two-level sort of the sampled nonzeros by destination row (row i of A is
// column i; reading Z28) instead of float atomics into Y_s:
//
//   plan_row_sums/write  pre[t] = sum_{t' < t} nnz(u_t') over the plan's rows, rb[t] = rowptr[u_t] -
//                        pre[t]: entry j of the concatenated sampled rows is nonzero rb[t] + j of A
//   coarse_count         per CTA a shared-memory histogram of the entries' coarse buckets (CB
//                        consecutive destination rows each), added into the global bucket counts
//   coarse_scan          bucket starts (one CTA); cursors = starts, counts re-zeroed
//   coarse_scatter       the same entries again: each CTA reserves its run in every bucket with one
//                        atomic per (CTA, bucket), then writes (t, row in bucket) and a_e into it
//   coarse_rows          one CTA per bucket: a shared-memory counting sort of its entries by
//                        destination row, then nnz-balanced slices over them (a hub destination is
//                        spread over lane groups), each row accumulated in registers from the
//                        gather table Z[t] = omega_t f_{u_t} (|U| x 4k bytes, L2 resident) and
//                        written once; rows shared by slices are combined in slice order; rows
//                        without a sampled neighbour are written as 0.
// Every row of Y_s is written exactly once, with no atomics on floating-point data.  The order of
// the terms inside a row follows shared-memory integer atomics (it may differ from run to run), so
// Y_s is compared by tolerance, as every other GPU product sum (reading Z29).
#include "kernels.cuh"

namespace symnmf {

constexpr int kPlanTile = 1024;      // plan rows per CTA of the plan-row scan (256 threads x 4)
constexpr int kEntChunk = 2048;      // sampled nonzeros per warp chunk (64 per lane)
constexpr int kEntUnroll = 8;        // independent entries in flight per lane
constexpr int kCoarseMaxBuckets = 8192;

// ---------------------------------------------------------------- plan-row offsets (two passes)
__device__ __forceinline__ void plan_row_lens(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ uniq,
                                              int64_t nu, int64_t t0, int64_t (&start)[4], int64_t (&len)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t t = t0 + q;
    if (t < nu) {
      const int64_t u = uniq[t];
      start[q] = rowptr[u];
      len[q] = rowptr[u + 1] - start[q];
    } else {
      start[q] = 0;
      len[q] = 0;
    }
  }
}

__global__ void __launch_bounds__(256) plan_row_sums(const int64_t* __restrict__ rowptr,
                                                     const int32_t* __restrict__ uniq,
                                                     const int64_t* __restrict__ n_uniq_dev,
                                                     int64_t* __restrict__ tsum, int64_t* __restrict__ pre,
                                                     unsigned int* counter, const int32_t* __restrict__ status) {
  __shared__ int64_t sh[33];
  __shared__ bool last;
  if (dev_failed(status)) return;
  const int64_t nu = *n_uniq_dev;
  const int64_t nt = (nu + kPlanTile - 1) / kPlanTile;
  if ((int64_t)blockIdx.x < nt) {
    int64_t start[4], len[4];
    plan_row_lens(rowptr, uniq, nu, (int64_t)blockIdx.x * kPlanTile + threadIdx.x * 4, start, len);
    const int64_t s = block_sum(len[0] + len[1] + len[2] + len[3], sh);
    if (threadIdx.x == 0) tsum[blockIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) *counter = 0;
  int64_t run = 0;
  for (int64_t base = 0; base < nt; base += 256) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nt ? __ldcg(tsum + i) : 0;
    int64_t tot;
    const int64_t e = block_excl_scan(v, sh, &tot);
    if (i < nt) tsum[i] = run + e;
    run += tot;
  }
  if (threadIdx.x == 0) pre[nu] = run;
}

__global__ void __launch_bounds__(256) plan_row_write(const int64_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ uniq,
                                                      const int64_t* __restrict__ n_uniq_dev,
                                                      const int64_t* __restrict__ tsum, int64_t* __restrict__ pre,
                                                      int64_t* __restrict__ rb, const int32_t* __restrict__ status) {
  __shared__ int64_t sh[33];
  if (dev_failed(status)) return;
  const int64_t nu = *n_uniq_dev;
  if ((int64_t)blockIdx.x * kPlanTile >= nu) return;
  const int64_t t0 = (int64_t)blockIdx.x * kPlanTile + threadIdx.x * 4;
  int64_t start[4], len[4];
  plan_row_lens(rowptr, uniq, nu, t0, start, len);
  int64_t p = block_excl_scan(len[0] + len[1] + len[2] + len[3], sh, (int64_t*)nullptr) + tsum[blockIdx.x];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (t0 + q < nu) {
      pre[t0 + q] = p;
      rb[t0 + q] = start[q] - p;
    }
    p += len[q];
  }
}

// Largest t in [lo, hi] with pre[t] <= j (pre non-decreasing, pre[lo] <= j).
__device__ __forceinline__ int64_t row_of_entry(const int64_t* __restrict__ pre, int64_t lo, int64_t hi, int64_t j) {
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(pre + mid) <= j) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// The same search by a whole warp in 32-ary steps.  Largest t < cnt with pre[t] <= j.
__device__ __forceinline__ int64_t warp_row_of_entry(const int64_t* __restrict__ pre, int64_t cnt, int64_t j,
                                                     int lane) {
  int64_t lo = 0, len = cnt;
  while (len > 1) {
    const int64_t step = (len + 31) / 32;
    const int64_t p = lo + (int64_t)lane * step;
    const bool le = p < lo + len && __ldg(pre + p) <= j;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    const int last = 31 - __clz(m);
    lo += (int64_t)last * step;
    len = min64(step, len - (int64_t)last * step);
  }
  return lo;
}

// Visit every sampled nonzero in nnz-balanced warp chunks: fn(t, e) with t the plan slot (-1: none)
// and e the nonzero of A.  The chunk -> warp assignment depends only on the grid, so two calls in
// kernels of the same grid visit the same entries in the same CTA.
template <class Fn>
__device__ __forceinline__ void for_sampled_nonzeros(const int64_t* __restrict__ pre, const int64_t* __restrict__ rb,
                                                     int64_t nu, Fn&& fn) {
  const int lane = threadIdx.x & 31;
  const int64_t total = pre[nu];
  const int64_t nchunks = (total + kEntChunk - 1) / kEntChunk;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t ch = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < nchunks; ch += nw) {
    const int64_t j0 = ch * kEntChunk, j1 = min64(total, j0 + kEntChunk);
    const int64_t thi = warp_row_of_entry(pre, nu, j1 - 1, lane);
    int64_t tcur = warp_row_of_entry(pre, thi + 1, j0, lane);
    for (int64_t jb = j0; jb < j1; jb += 32 * kEntUnroll) {
      int64_t t[kEntUnroll], e[kEntUnroll];
#pragma unroll
      for (int u = 0; u < kEntUnroll; ++u) {
        const int64_t j = jb + 32 * u + lane;
        t[u] = j < j1 ? row_of_entry(pre, tcur, thi, j) : -1;
        e[u] = t[u] >= 0 ? __ldg(rb + t[u]) + j : 0;
      }
      fn(t, e);
      const int64_t jl = min64(j1, jb + 32 * kEntUnroll) - 1;
      tcur = row_of_entry(pre, tcur, thi, jl);
    }
  }
}

// ---------------------------------------------------------------- coarse partition
__global__ void __launch_bounds__(256) coarse_count(const int32_t* __restrict__ col, const int64_t* __restrict__ pre,
                                                    const int64_t* __restrict__ rb,
                                                    const int64_t* __restrict__ n_uniq_dev, int nb, int lb,
                                                    int32_t* __restrict__ gcnt, const int32_t* __restrict__ status) {
  extern __shared__ int32_t hist[];
  if (dev_failed(status)) return;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int64_t nu = *n_uniq_dev;
  if (nu > 0) {
    for_sampled_nonzeros(pre, rb, nu, [&](const int64_t (&t)[kEntUnroll], const int64_t (&e)[kEntUnroll]) {
      int32_t c[kEntUnroll];
#pragma unroll
      for (int u = 0; u < kEntUnroll; ++u) c[u] = t[u] >= 0 ? __ldg(col + e[u]) : 0;
#pragma unroll
      for (int u = 0; u < kEntUnroll; ++u)
        if (t[u] >= 0) atomicAdd(hist + (c[u] >> lb), 1);
    });
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (hist[b]) atomicAdd(gcnt + b, hist[b]);
}

__global__ void __launch_bounds__(1024) coarse_scan(int32_t* __restrict__ gcnt, int nb, int32_t* __restrict__ gstart,
                                                    int32_t* __restrict__ cursor, const int32_t* __restrict__ status) {
  __shared__ int32_t sh[33];
  if (dev_failed(status)) return;
  int32_t run = 0;
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const int32_t v = i < nb ? gcnt[i] : 0;
    int32_t tot;
    const int32_t e = block_excl_scan(v, sh, &tot);
    if (i < nb) {
      gstart[i] = run + e;
      cursor[i] = run + e;
      gcnt[i] = 0;   // counts zero for the next plan
    }
    run += tot;
  }
  if (threadIdx.x == 0) gstart[nb] = run;
}

__global__ void __launch_bounds__(256) coarse_scatter(const int32_t* __restrict__ col, const float* __restrict__ val,
                                                      const int64_t* __restrict__ pre, const int64_t* __restrict__ rb,
                                                      const int64_t* __restrict__ n_uniq_dev, int nb, int lb,
                                                      int32_t* __restrict__ cursor, int2* __restrict__ key,
                                                      float* __restrict__ kval, const int32_t* __restrict__ status) {
  extern __shared__ int32_t sm[];
  int32_t* hist = sm;        // [nb] counts, then the CTA's next slot per bucket
  int32_t* base = sm + nb;   // [nb] the CTA's run in each bucket
  if (dev_failed(status)) return;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int64_t nu = *n_uniq_dev;
  if (nu <= 0) return;
  for_sampled_nonzeros(pre, rb, nu, [&](const int64_t (&t)[kEntUnroll], const int64_t (&e)[kEntUnroll]) {
    int32_t c[kEntUnroll];
#pragma unroll
    for (int u = 0; u < kEntUnroll; ++u) c[u] = t[u] >= 0 ? __ldg(col + e[u]) : 0;
#pragma unroll
    for (int u = 0; u < kEntUnroll; ++u)
      if (t[u] >= 0) atomicAdd(hist + (c[u] >> lb), 1);
  });
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const int32_t h = hist[b];
    base[b] = h ? atomicAdd(cursor + b, h) : 0;
    hist[b] = 0;
  }
  __syncthreads();
  const int32_t cmask = (1 << lb) - 1;
  for_sampled_nonzeros(pre, rb, nu, [&](const int64_t (&t)[kEntUnroll], const int64_t (&e)[kEntUnroll]) {
    int32_t c[kEntUnroll];
    float a[kEntUnroll];
#pragma unroll
    for (int u = 0; u < kEntUnroll; ++u) {
      c[u] = t[u] >= 0 ? __ldg(col + e[u]) : 0;
      a[u] = t[u] >= 0 ? __ldcs(val + e[u]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kEntUnroll; ++u) {
      if (t[u] >= 0) {
        const int b = c[u] >> lb;
        const int32_t p = base[b] + atomicAdd(hist + b, 1);
        key[p] = make_int2((int32_t)t[u], c[u] & cmask);
        kval[p] = a[u];
      }
    }
  });
}

// ---------------------------------------------------------------- per-bucket rows
template <int KP>
struct CoarseRowsSmem {
  static constexpr int NSL = (256 / 32) * (32 / (KP / 4));   // lane groups = slices
  static constexpr int NC = 2 * NSL;                         // carry slots
};

__device__ __forceinline__ int row_of_off(const int32_t* sOff, int rows, int e) {   // sOff[r] <= e < sOff[r+1]
  int lo = 0, hi = rows - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sOff[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int KP>
__global__ void __launch_bounds__(256) coarse_rows(const int32_t* __restrict__ gstart, int64_t n, int lb,
                                                   const int2* __restrict__ key, const float* __restrict__ kval,
                                                   int2* __restrict__ sorted, const float4* __restrict__ Z4,
                                                   float4* __restrict__ Y4, const int32_t* __restrict__ status) {
  using L = CoarseRowsSmem<KP>;
  constexpr int LPR = KP / 4, NG = 32 / LPR;
  extern __shared__ __align__(16) unsigned char smc[];
  const int CB = 1 << lb;
  int32_t* sOff = reinterpret_cast<int32_t*>(smc);            // [CB + 1]
  int32_t* sCur = sOff + CB + 1;                              // [CB]
  float4* sC = reinterpret_cast<float4*>(smc + ((sizeof(int32_t) * (2 * CB + 1) + 15) & ~size_t(15)));   // [NC][LPR]
  int32_t* sCr = reinterpret_cast<int32_t*>(sC + L::NC * LPR);   // [NC]
  __shared__ int32_t sh[33];
  if (dev_failed(status)) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, grp = lane / LPR, li = lane % LPR;
  const int64_t b = blockIdx.x;
  const int64_t r0 = b << lb;
  const int rows = (int)min64(CB, n - r0);
  const int32_t e0 = gstart[b], m = gstart[b + 1] - e0;
  // 1. counting sort of the bucket's entries by destination row (shared-memory integer atomics)
  for (int r = tid; r < CB; r += 256) sCur[r] = 0;
  __syncthreads();
  for (int e = tid; e < m; e += 256) atomicAdd(sCur + key[e0 + e].y, 1);
  __syncthreads();
  {
    const int per = CB / 256;   // CB is a multiple of 256
    int32_t loc = 0;
    for (int q = 0; q < per; ++q) loc += sCur[tid * per + q];
    int32_t tot;
    int32_t run = block_excl_scan(loc, sh, &tot);
    for (int q = 0; q < per; ++q) {
      const int r = tid * per + q;
      const int32_t c = sCur[r];
      sOff[r] = run;
      run += c;
    }
    if (tid == 0) sOff[CB] = tot;
  }
  __syncthreads();
  for (int r = tid; r < CB; r += 256) sCur[r] = sOff[r];
  __syncthreads();
  for (int e = tid; e < m; e += 256) {
    const int2 kk = key[e0 + e];
    const int32_t p = atomicAdd(sCur + kk.y, 1);
    sorted[e0 + p] = make_int2(kk.x, __float_as_int(kval[e0 + e]));
  }
  for (int c = tid; c < L::NC; c += 256) sCr[c] = -1;
  __syncthreads();
  // 2. nnz-balanced slices over the sorted entries; interior rows written, first / last carried
  {
    const int sl = wid * NG + grp;
    const int Ls = (m + L::NSL - 1) / L::NSL;
    const int s0 = min(m, sl * Ls), s1 = min(m, s0 + Ls);
    if (s0 < s1) {
      const int rfirst = row_of_off(sOff, rows, s0), rlast = row_of_off(sOff, rows, s1 - 1);
      int row = rfirst, rend = sOff[rfirst + 1];
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      auto put = [&](int r, float4 v) {
        if (r == rfirst || r == rlast) sC[(2 * sl + (r == rfirst ? 0 : 1)) * LPR + li] = v;
        else Y4[(r0 + r) * LPR + li] = v;                   // interior: this slice owns the row
      };
      if (li == 0) { sCr[2 * sl] = rfirst; sCr[2 * sl + 1] = rlast != rfirst ? rlast : -1; }
      constexpr int U = 8;
      for (int e = s0; e < s1; e += U) {
        int2 en[U];
        float4 z[U];
#pragma unroll
        for (int u = 0; u < U; ++u) en[u] = (e + u < s1) ? sorted[e0 + e + u] : make_int2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u)
          z[u] = (e + u < s1) ? __ldg(Z4 + (int64_t)en[u].x * LPR + li) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = e + u;
          if (j < s1) {
            if (j >= rend) {
              put(row, acc);
              acc = make_float4(0.f, 0.f, 0.f, 0.f);
              do { ++row; rend = sOff[row + 1]; } while (rend <= j);   // skips rows without entries
            }
            const float a = __int_as_float(en[u].y);
            acc.x = fmaf(a, z[u].x, acc.x); acc.y = fmaf(a, z[u].y, acc.y);
            acc.z = fmaf(a, z[u].z, acc.z); acc.w = fmaf(a, z[u].w, acc.w);
          }
        }
      }
      put(row, acc);
    }
  }
  __syncthreads();
  // 3. carried rows: runs of equal rows (consecutive slots) summed in slice order, written once
  for (int e = tid; e < L::NC * LPR; e += 256) {
    const int c = e / LPR, q = e - c * LPR;
    const int r = sCr[c];
    if (r < 0) continue;
    int prev = c - 1;
    while (prev >= 0 && sCr[prev] < 0) --prev;
    if (prev >= 0 && sCr[prev] == r) continue;   // not the head of its run
    float4 s = sC[c * LPR + q];
    for (int c2 = c + 1; c2 < L::NC; ++c2) {
      const int r2 = sCr[c2];
      if (r2 < 0) continue;
      if (r2 != r) break;
      const float4 v = sC[c2 * LPR + q];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    Y4[(r0 + r) * LPR + q] = s;
  }
  // 4. rows without a sampled neighbour
  for (int e = tid; e < rows * LPR; e += 256) {
    const int r = e / LPR, q = e - r * LPR;
    if (sOff[r] == sOff[r + 1]) Y4[(r0 + r) * LPR + q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// ---------------------------------------------------------------- host side
int coarse_lb(int64_t n) {   // log2 of the rows per coarse bucket: >= 10, <= kCoarseMaxBuckets buckets
  int lb = 10;
  while ((((n + (1ll << lb) - 1) >> lb) > kCoarseMaxBuckets) && lb < 12) ++lb;
  return (((n + (1ll << lb) - 1) >> lb) > kCoarseMaxBuckets) ? -1 : lb;
}

bool coarse_supported(int64_t n, int64_t nnz, int k) {
  return coarse_lb(n) >= 0 && nnz < (int64_t)INT32_MAX && (k == 8 || k == 16 || k == 32 || k == 64);
}

void coarse_layout(Carver& c, int64_t n, int64_t nnz, int64_t cap, CoarseWs* w) {
  const int lb = coarse_lb(n);
  w->lb = lb;
  w->nb = (int)((n + (1ll << lb) - 1) >> lb);
  w->cap = cap;
  w->ptsum = c.take<int64_t>((size_t)(cap + kPlanTile - 1) / kPlanTile + 4);
  w->pre = c.take<int64_t>((size_t)cap + 1);
  w->rb = c.take<int64_t>((size_t)cap + 1);
  w->gcnt = c.take<int32_t>((size_t)w->nb + 1);
  w->gstart = c.take<int32_t>((size_t)w->nb + 1);
  w->cursor = c.take<int32_t>((size_t)w->nb + 1);
  w->key = c.take<int2>((size_t)nnz);
  w->kval = c.take<float>((size_t)nnz);
  w->sorted = c.take<int2>((size_t)nnz);
}

static int coarse_grid(int64_t nnz) {
  const int64_t warps = (nnz + kEntChunk - 1) / kEntChunk;
  return (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 148 * 8));
}

template <int KP>
static void coarse_rows_t(const CoarseWs& w, int64_t n, const float* Z, float* Y, const int32_t* status,
                          cudaStream_t st) {
  using L = CoarseRowsSmem<KP>;
  const int CB = 1 << w.lb;
  const size_t smem = ((sizeof(int32_t) * (2 * CB + 1) + 15) & ~size_t(15)) + sizeof(float4) * L::NC * (KP / 4) +
                      sizeof(int32_t) * L::NC;
  cudaFuncSetAttribute(coarse_rows<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(coarse_rows<KP>, w.nb, 256, smem, st, w.gstart, n, w.lb, w.key, w.kval, w.sorted,
             reinterpret_cast<const float4*>(Z), reinterpret_cast<float4*>(Y), status);
}

void launch_coarse_partition(const symnmf_matrix& A, const int32_t* uniq, const int64_t* n_uniq_dev,
                             const CoarseWs& w, unsigned int* counter, int32_t* status, cudaStream_t st) {
  const int ptiles = (int)std::max<int64_t>(1, (w.cap + kPlanTile - 1) / kPlanTile);
  launch_pdl(plan_row_sums, ptiles, 256, 0, st, A.rowptr, uniq, n_uniq_dev, w.ptsum, w.pre, counter, status);
  launch_pdl(plan_row_write, ptiles, 256, 0, st, A.rowptr, uniq, n_uniq_dev, w.ptsum, w.pre, w.rb, status);
  const int grid = coarse_grid(A.nnz);
  const size_t hs = sizeof(int32_t) * w.nb;
  cudaFuncSetAttribute(coarse_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs);
  cudaFuncSetAttribute(coarse_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * hs));
  launch_pdl(coarse_count, grid, 256, hs, st, A.colidx, w.pre, w.rb, n_uniq_dev, w.nb, w.lb, w.gcnt, status);
  launch_pdl(coarse_scan, 1, 1024, 0, st, w.gcnt, w.nb, w.gstart, w.cursor, status);
  launch_pdl(coarse_scatter, grid, 256, 2 * hs, st, A.colidx, A.val, w.pre, w.rb, n_uniq_dev, w.nb, w.lb, w.cursor,
             w.key, w.kval, status);
}

void launch_coarse_rows(const CoarseWs& w, int64_t n, const float* Z, int k, float* Y, int32_t* status,
                        cudaStream_t st) {
  switch (k) {
    case 8: coarse_rows_t<8>(w, n, Z, Y, status, st); break;
    case 16: coarse_rows_t<16>(w, n, Z, Y, status, st); break;
    case 32: coarse_rows_t<32>(w, n, Z, Y, status, st); break;
    default: coarse_rows_t<64>(w, n, Z, Y, status, st); break;
  }
}

}  // namespace symnmf
