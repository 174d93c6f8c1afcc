// (a9) The sampled CSR product Y_s = sum_{i in U} omega_i A[i,:]^T f_i
// in destination-bucketed form: the sampled rows' nonzeros are counting-sorted by their column
// (= the destination row of Y_s, since row i of A is column i), so the HALS sweep that
// consumes Y_s can pull each destination row's terms from one contiguous bucket and Y_s never
// exists in HBM.  Steps (all on the solver's stream, after the plan):
//
//   plan_row_*        pre[t] = sum_{t' < t} nnz(u_t') over the plan's unique rows (two passes), and
//                     rb[t] = rowptr[u_t] - pre[t], so entry j of the concatenated sampled rows is
//                     nonzero e = rb[t] + j of A for the t with pre[t] <= j < pre[t+1].
//   bucket_count      slot[e] = atomicAdd(&cnt[col[e]], 1) for every sampled nonzero e: the count
//                     of each bucket and the entry's place in it (nnz-balanced warp chunks, so a
//                     hub row is spread over many warps).
//   bucket_scan_*     off = exclusive scan of cnt (two passes: tile sums + last-CTA scan of the
//                     tile sums, then the tiles), cnt re-zeroed for the next plan.
//   bucket_fill       ent[off[c] + slot[e]] = (t, a_e): the bucket entries.
//   bucket_pull       Y_s[r] = sum over bucket r of a_e Z[t_e], Z[t] = omega_t f_{u_t} (the sampled
//                     Gram kernel writes Z); or, fused, the row-tile sweep of tile.cu reads the buckets.
//
// The order of the entries inside a bucket follows the atomics (run to run it may differ), so the
// fp32 sum of a bucket is compared by tolerance, like every other GPU product sum (reading Z29).
#include "kernels.cuh"

namespace symnmf {

constexpr int kBucketChunk = 2048;   // sampled nonzeros per warp chunk (64 per lane)
constexpr int kBucketUnroll = 8;     // independent entries in flight per lane

// ---------------------------------------------------------------- plan_row_offsets (two passes)
constexpr int kPlanTile = 1024;   // plan rows per CTA (256 threads x 4)

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
                                                      int64_t* __restrict__ rb, int32_t* __restrict__ slot_of,
                                                      const int32_t* __restrict__ status) {
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
      if (slot_of) slot_of[uniq[t0 + q]] = (int32_t)(t0 + q);
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

// The same search by a whole warp: 32-ary steps (each lane probes one split point), so a chunk's
// bounds cost ~log32(nu) dependent loads instead of log2(nu).  Largest t < cnt with pre[t] <= j.
__device__ __forceinline__ int64_t warp_row_of_entry(const int64_t* __restrict__ pre, int64_t cnt, int64_t j,
                                                     int lane) {
  int64_t lo = 0, len = cnt;                          // answer in [lo, lo + len)
  while (len > 1) {
    const int64_t step = (len + 31) / 32;
    const int64_t p = lo + (int64_t)lane * step;      // lane probes the start of its segment
    const bool le = p < lo + len && __ldg(pre + p) <= j;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    const int last = 31 - __clz(m);                   // the last segment whose start is <= j (lane 0 always)
    lo += (int64_t)last * step;
    len = min64(step, len - (int64_t)last * step);
  }
  return lo;
}

// Visit every sampled nonzero in nnz-balanced warp chunks: fn(t, e) with t the plan slot and e the
// nonzero of A.  Each lane keeps kBucketUnroll entries in flight.
template <class Fn>
__device__ __forceinline__ void for_sampled_nonzeros(const int64_t* __restrict__ pre, const int64_t* __restrict__ rb,
                                                     int64_t nu, Fn&& fn) {
  const int lane = threadIdx.x & 31;
  const int64_t total = pre[nu];
  const int64_t nchunks = (total + kBucketChunk - 1) / kBucketChunk;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t ch = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < nchunks; ch += nw) {
    const int64_t j0 = ch * kBucketChunk, j1 = min64(total, j0 + kBucketChunk);
    const int64_t thi = warp_row_of_entry(pre, nu, j1 - 1, lane);
    int64_t tcur = warp_row_of_entry(pre, thi + 1, j0, lane);
    for (int64_t jb = j0; jb < j1; jb += 32 * kBucketUnroll) {
      int64_t t[kBucketUnroll], e[kBucketUnroll];
#pragma unroll
      for (int u = 0; u < kBucketUnroll; ++u) {
        const int64_t j = jb + 32 * u + lane;
        t[u] = j < j1 ? row_of_entry(pre, tcur, thi, j) : -1;
        e[u] = t[u] >= 0 ? __ldg(rb + t[u]) + j : 0;
      }
      fn(t, e);
      // the group's last entry's row starts the next group's search
      const int64_t jl = min64(j1, jb + 32 * kBucketUnroll) - 1;
      tcur = row_of_entry(pre, tcur, thi, jl);
    }
  }
}

__global__ void __launch_bounds__(256) bucket_count(const int32_t* __restrict__ col, const int64_t* __restrict__ pre,
                                                    const int64_t* __restrict__ rb,
                                                    const int64_t* __restrict__ n_uniq_dev, int32_t* __restrict__ cnt,
                                                    int32_t* __restrict__ slot, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t nu = *n_uniq_dev;
  if (nu <= 0) return;
  for_sampled_nonzeros(pre, rb, nu, [&](const int64_t (&t)[kBucketUnroll], const int64_t (&e)[kBucketUnroll]) {
    int32_t c[kBucketUnroll], s[kBucketUnroll];
#pragma unroll
    for (int u = 0; u < kBucketUnroll; ++u) c[u] = t[u] >= 0 ? __ldcs(col + e[u]) : 0;
#pragma unroll
    for (int u = 0; u < kBucketUnroll; ++u) s[u] = t[u] >= 0 ? atomicAdd(cnt + c[u], 1) : 0;
#pragma unroll
    for (int u = 0; u < kBucketUnroll; ++u)
      if (t[u] >= 0) slot[e[u]] = s[u];
  });
}

// ---------------------------------------------------------------- exclusive scan of cnt
constexpr int kScanTile = 4096;   // 256 threads x 16
inline int64_t bucket_scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }

__global__ void __launch_bounds__(256) bucket_scan_sums(const int32_t* __restrict__ cnt, int64_t n,
                                                        int32_t* __restrict__ tsum, int32_t* __restrict__ off,
                                                        unsigned int* counter, int32_t* __restrict__ status) {
  __shared__ int32_t sh[33];
  if (dev_failed(status)) return;
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 16;
  int32_t s = 0;
  if (i0 + 16 <= n) {
    const int4* c4 = reinterpret_cast<const int4*>(cnt + i0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 v = __ldcg(c4 + q);
      s += v.x + v.y + v.z + v.w;
    }
  } else {
    for (int64_t i = i0; i < min64(n, i0 + 16); ++i) s += __ldcg(cnt + i);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) tsum[blockIdx.x] = s;
  // last CTA: exclusive scan of the tile sums (in place) and the grand total off[n]
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) *counter = 0;
  const int64_t nt = gridDim.x;
  int32_t run = 0;
  for (int64_t base = 0; base < nt; base += 256) {
    const int64_t i = base + threadIdx.x;
    const int32_t v = i < nt ? __ldcg(tsum + i) : 0;
    int32_t tot;
    const int32_t e = block_excl_scan(v, sh, &tot);
    if (i < nt) tsum[i] = run + e;
    run += tot;
  }
  if (threadIdx.x == 0) off[n] = run;
}

__global__ void __launch_bounds__(256) bucket_scan_write(int32_t* __restrict__ cnt, int64_t n,
                                                         const int32_t* __restrict__ tsum, int32_t* __restrict__ off,
                                                         const int32_t* __restrict__ status) {
  __shared__ int32_t sh[33];
  if (dev_failed(status)) return;
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 16;
  int32_t v[16];
  if (i0 + 16 <= n) {
    const int4* c4 = reinterpret_cast<const int4*>(cnt + i0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 x = __ldcg(c4 + q);
      v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = i0 + q < n ? __ldcg(cnt + i0 + q) : 0;
  }
  int32_t tot = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) tot += v[q];
  int32_t run = block_excl_scan(tot, sh, (int32_t*)nullptr) + tsum[blockIdx.x];
  if (i0 + 16 <= n) {
    int4* o4 = reinterpret_cast<int4*>(off + i0);
    int4* c4 = reinterpret_cast<int4*>(cnt + i0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int4 x;
      x.x = run; run += v[4 * q];
      x.y = run; run += v[4 * q + 1];
      x.z = run; run += v[4 * q + 2];
      x.w = run; run += v[4 * q + 3];
      o4[q] = x;
      c4[q] = make_int4(0, 0, 0, 0);   // buckets empty for the next plan
    }
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (i0 + q < n) {
        off[i0 + q] = run;
        cnt[i0 + q] = 0;
      }
      run += v[q];
    }
  }
}

// ---------------------------------------------------------------- bucket_fill
__global__ void __launch_bounds__(256) bucket_fill(const int32_t* __restrict__ col, const float* __restrict__ val,
                                                   const int64_t* __restrict__ pre, const int64_t* __restrict__ rb,
                                                   const int64_t* __restrict__ n_uniq_dev,
                                                   const int32_t* __restrict__ off, const int32_t* __restrict__ slot,
                                                   int2* __restrict__ ent, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t nu = *n_uniq_dev;
  if (nu <= 0) return;
  for_sampled_nonzeros(pre, rb, nu, [&](const int64_t (&t)[kBucketUnroll], const int64_t (&e)[kBucketUnroll]) {
    int32_t c[kBucketUnroll], s[kBucketUnroll];
    float a[kBucketUnroll];
#pragma unroll
    for (int u = 0; u < kBucketUnroll; ++u) {
      const bool ok = t[u] >= 0;
      c[u] = ok ? __ldcs(col + e[u]) : 0;
      s[u] = ok ? __ldcs(slot + e[u]) : 0;
      a[u] = ok ? __ldcs(val + e[u]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kBucketUnroll; ++u)
      if (t[u] >= 0) ent[__ldg(off + c[u]) + s[u]] = make_int2((int32_t)t[u], __float_as_int(a[u]));
  });
}

// ---------------------------------------------------------------- bucket_pull
// Y_s[r] = sum over bucket r of a_e Z[t_e] (Z[t] = omega_t f_{u_t}): one group of KP / 4 lanes per
// destination row, float4 gathers of Z (|U| x 4k bytes, L2 resident), each row written once.
template <int KP>
__global__ void __launch_bounds__(256) bucket_pull(const int32_t* __restrict__ off, const int2* __restrict__ ent,
                                                   const float4* __restrict__ Z, int64_t n, float4* __restrict__ Y,
                                                   const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  constexpr int LPR = KP / 4;
  const int li = threadIdx.x % LPR;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; r < n; r += ng) {
    const int32_t e0 = __ldg(off + r), e1 = __ldg(off + r + 1);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t e = e0;
    for (; e + 4 <= e1; e += 4) {
      int2 en[4];
      float4 z[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) en[u] = __ldcs(ent + e + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) z[u] = __ldg(Z + (int64_t)en[u].x * LPR + li);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float a = __int_as_float(en[u].y);
        acc.x = fmaf(a, z[u].x, acc.x); acc.y = fmaf(a, z[u].y, acc.y);
        acc.z = fmaf(a, z[u].z, acc.z); acc.w = fmaf(a, z[u].w, acc.w);
      }
    }
    for (; e < e1; ++e) {
      const int2 en = __ldcs(ent + e);
      const float4 z = __ldg(Z + (int64_t)en.x * LPR + li);
      const float a = __int_as_float(en.y);
      acc.x = fmaf(a, z.x, acc.x); acc.y = fmaf(a, z.y, acc.y);
      acc.z = fmaf(a, z.z, acc.z); acc.w = fmaf(a, z.w, acc.w);
    }
    Y[r * LPR + li] = acc;
  }
}

void launch_bucket_pull(const BucketWs& b, const float* Z, int64_t n, int k, float* Y, const int32_t* status,
                        cudaStream_t st) {
  const int64_t thr = n * (k / 4);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((thr + 255) / 256, 148 * 8));
  const float4* Z4 = reinterpret_cast<const float4*>(Z);
  float4* Y4 = reinterpret_cast<float4*>(Y);
  switch (k) {
    case 8: launch_pdl(bucket_pull<8>, grid, 256, 0, st, b.off, b.ent, Z4, n, Y4, status); break;
    case 16: launch_pdl(bucket_pull<16>, grid, 256, 0, st, b.off, b.ent, Z4, n, Y4, status); break;
    case 32: launch_pdl(bucket_pull<32>, grid, 256, 0, st, b.off, b.ent, Z4, n, Y4, status); break;
    default: launch_pdl(bucket_pull<64>, grid, 256, 0, st, b.off, b.ent, Z4, n, Y4, status); break;
  }
}

static int bucket_grid(int64_t cap_entries);

// ---------------------------------------------------------------- mirror marks (the default sampled product)
// Each sampled nonzero e = (i, c) of A (i in U) flags its mirror position m(e) -- the place of (c, i)
// in row c, precomputed once per A -- in a bitmap over the nonzeros; a pull over the rows of A then
// reads, in each destination row c, exactly the flagged entries (c, i), i in U, in column order:
// Y_s[c] = sum_i A[c, i] Z[slot(i)], deterministic and free of float atomics (spmm_nnz.cu).
__global__ void __launch_bounds__(256) mark_sampled(const int32_t* __restrict__ mirror, const int64_t* __restrict__ pre,
                                                    const int64_t* __restrict__ rb,
                                                    const int64_t* __restrict__ n_uniq_dev, uint32_t* __restrict__ bits,
                                                    const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t nu = *n_uniq_dev;
  if (nu <= 0) return;
  for_sampled_nonzeros(pre, rb, nu, [&](const int64_t (&t)[kBucketUnroll], const int64_t (&e)[kBucketUnroll]) {
    int32_t m[kBucketUnroll];
#pragma unroll
    for (int u = 0; u < kBucketUnroll; ++u) m[u] = t[u] >= 0 ? __ldcs(mirror + e[u]) : 0;
#pragma unroll
    for (int u = 0; u < kBucketUnroll; ++u)
      if (t[u] >= 0) atomicOr(bits + (m[u] >> 5), 1u << (m[u] & 31));
  });
}

// mirror[e] = position of (c, r) in row c for e = (r, c); *bad = 1 if A's pattern is not symmetric
__global__ void mirror_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, int64_t n,
                              int32_t* __restrict__ mirror, int32_t* __restrict__ bad) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= n) return;
  const int lane = threadIdx.x & 31;
  for (int64_t e = rowptr[r] + lane; e < rowptr[r + 1]; e += 32) {
    const int64_t c = col[e];
    int64_t lo = rowptr[c], hi = rowptr[c + 1];
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (col[m] < r) lo = m + 1; else hi = m;
    }
    if (lo < rowptr[c + 1] && col[lo] == r) mirror[e] = (int32_t)lo;
    else { mirror[e] = 0; atomicExch(bad, 1); }
  }
}

void launch_mirror(const symnmf_matrix& A, int32_t* mirror, int32_t* bad, cudaStream_t st) {
  if (A.n > 0) mirror_kernel<<<(unsigned)((A.n + 7) / 8), 256, 0, st>>>(A.rowptr, A.colidx, A.n, mirror, bad);
}

void launch_mark_sampled(const symnmf_matrix& A, const int32_t* uniq, const int64_t* n_uniq_dev, const BucketWs& b,
                         const int32_t* mirror, uint32_t* bits, int32_t* slot_of, unsigned int* counter,
                         int32_t* status, cudaStream_t st) {
  const int ptiles = (int)std::max<int64_t>(1, (b.cap + kPlanTile - 1) / kPlanTile);
  launch_pdl(plan_row_sums, ptiles, 256, 0, st, A.rowptr, uniq, n_uniq_dev, b.ptsum, b.pre, counter, status);
  launch_pdl(plan_row_write, ptiles, 256, 0, st, A.rowptr, uniq, n_uniq_dev, b.ptsum, b.pre, b.rb, slot_of, status);
  launch_pdl(mark_sampled, bucket_grid(A.nnz), 256, 0, st, mirror, b.pre, b.rb, n_uniq_dev, bits, status);
}

// ---------------------------------------------------------------- launchers
size_t bucket_ws_bytes(int64_t n, int64_t nnz, int64_t cap) {
  // pre, rb [cap + 1] int64; cnt, off [n + 1] int32; tsum; slot [nnz] int32; ent [nnz] int2
  return sizeof(int64_t) * 2 * (size_t)(cap + 1) + sizeof(int32_t) * 2 * (size_t)(n + 4) +
         sizeof(int32_t) * (size_t)(bucket_scan_tiles(n) + 4) + sizeof(int32_t) * (size_t)nnz +
         sizeof(int2) * (size_t)nnz + 6 * 256;
}

void mark_layout(Carver& c, int64_t n, int64_t nnz, int64_t cap, BucketWs* b) {   // plan-row offsets only
  (void)n; (void)nnz;
  *b = BucketWs{};
  b->cap = cap;
  b->ptsum = c.take<int64_t>((size_t)(cap + kPlanTile - 1) / kPlanTile + 4);
  b->pre = c.take<int64_t>((size_t)cap + 1);
  b->rb = c.take<int64_t>((size_t)cap + 1);
}

void bucket_layout(Carver& c, int64_t n, int64_t nnz, int64_t cap, BucketWs* b) {
  b->cap = cap;
  b->ptsum = c.take<int64_t>((size_t)(cap + kPlanTile - 1) / kPlanTile + 4);
  b->pre = c.take<int64_t>((size_t)cap + 1);
  b->rb = c.take<int64_t>((size_t)cap + 1);
  b->cnt = c.take<int32_t>((size_t)n + 4);
  b->off = c.take<int32_t>((size_t)n + 4);
  b->tsum = c.take<int32_t>((size_t)bucket_scan_tiles(n) + 4);
  b->slot = c.take<int32_t>((size_t)nnz);
  b->ent = c.take<int2>((size_t)nnz);
}

static int bucket_grid(int64_t cap_entries) {
  const int64_t warps = (cap_entries + kBucketChunk - 1) / kBucketChunk;
  return (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 148 * 8));
}

void launch_bucket_build(const symnmf_matrix& A, const int32_t* uniq, const int64_t* n_uniq_dev, const BucketWs& b,
                         unsigned int* counter, int32_t* status, cudaStream_t st) {
  const int64_t n = A.n;
  const int ptiles = (int)std::max<int64_t>(1, (b.cap + kPlanTile - 1) / kPlanTile);
  launch_pdl(plan_row_sums, ptiles, 256, 0, st, A.rowptr, uniq, n_uniq_dev, b.ptsum, b.pre, counter, status);
  launch_pdl(plan_row_write, ptiles, 256, 0, st, A.rowptr, uniq, n_uniq_dev, b.ptsum, b.pre, b.rb,
             (int32_t*)nullptr, status);
  const int grid = bucket_grid(A.nnz);
  launch_pdl(bucket_count, grid, 256, 0, st, A.colidx, b.pre, b.rb, n_uniq_dev, b.cnt, b.slot, status);
  const int tiles = (int)bucket_scan_tiles(n);
  launch_pdl(bucket_scan_sums, tiles, 256, 0, st, b.cnt, n, b.tsum, b.off, counter, status);
  launch_pdl(bucket_scan_write, tiles, 256, 0, st, b.cnt, n, b.tsum, b.off, status);
  launch_pdl(bucket_fill, grid, 256, 0, st, A.colidx, A.val, b.pre, b.rb, n_uniq_dev, b.off, b.slot, b.ent, status);
}

}  // namespace symnmf
