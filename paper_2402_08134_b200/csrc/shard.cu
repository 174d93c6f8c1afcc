// NEXT-4: row-sharded LvS / EXACT building blocks.  A shard owns the contiguous row
// block [row0, row0 + n_b) of A (CSR rows with global column indices), W and H; between the calls
// below the driver (paper_2402_08134_b200/shard.py) runs the collectives -- a k x k allreduce of
// Gram partials, an allgather of the shards' integer masses (whose exclusive scan places each
// shard's prefix inside the global one), an allgather of the shards' plan rows and scaled rows --
// over NCCL (one shard per GPU) or in-process (logical shards on one device).
//
//   symnmf_leverage_scores_gram  scores of a row block from the Gram of the whole factor
//   symnmf_hybrid_shard_sums     the block's integer mass W_b = sum floor(l 2^40) over I_R, |I_D ∩ b|,
//                                theta_b (readings Z1-Z6)
//   symnmf_hybrid_shard_plan     the block's part of the global plan: its I_D rows, and the global
//                                draws t = mulhi(u_j, W) that fall in [W_off, W_off + W_b), resolved in
//                                the block's own prefix; weights with the global W and s_R.  Integer
//                                arithmetic, so the concatenated shard plans equal the 1-shard plan
//                                bit for bit
//   symnmf_plan_rows_scaled      Z[t] = omega_t f_{u_t} for the block's plan rows (allgathered -> Z)
//   symnmf_sampled_ah_rows       Y_s rows of the block as a pull: Y_s[c] = sum_{i in U} a_ci Z[slot(i)]
//                                (row c of A holds a_ci = a_ic by symmetry), so the sampled
//                                product needs no exchange of A's rows
#include "kernels.cuh"

namespace symnmf {

constexpr double kTwo40s = 1099511627776.0;

// ---------------------------------------------------------------- shard sums (ordered, one CTA)
__global__ void __launch_bounds__(1024) shard_sums_kernel(const uint64_t* __restrict__ bw,
                                                          const uint32_t* __restrict__ bd,
                                                          const double* __restrict__ bt, int64_t nb,
                                                          uint64_t* __restrict__ W_out, int64_t* __restrict__ sD_out,
                                                          double* __restrict__ theta_out,
                                                          const int32_t* __restrict__ status) {
  __shared__ uint64_t shw[33];
  __shared__ uint32_t shd[33];
  __shared__ double sht[33];
  if (dev_failed(status)) return;
  uint64_t cw = 0;
  uint32_t cd = 0;
  double theta = 0.0;
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    uint64_t vw = i < nb ? bw[i] : 0ull;
    uint32_t vd = i < nb ? bd[i] : 0u;
    double vt = i < nb ? bt[i] : 0.0;
    vw = block_sum(vw, shw);
    vd = block_sum(vd, shd);
    vt = block_sum(vt, sht);
    cw += vw; cd += vd; theta += vt;   // valid in warp 0
    __syncthreads();
  }
  if (threadIdx.x == 0) { *W_out = cw; *sD_out = (int64_t)cd; *theta_out = theta; }
}

// ---------------------------------------------------------------- shard plan pieces
// After the local block scan: keep the local mass, publish the global s_R and W to the plan counts.
__global__ void shard_fix_kernel(int64_t* __restrict__ counts, uint64_t* __restrict__ wloc, int64_t s,
                                 int64_t sD_total, uint64_t W_total, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  *wloc = (uint64_t)counts[3];
  counts[1] = W_total == 0ull ? 0 : (s > sD_total ? s - sD_total : 0);   // reading Z2, global s_D
  counts[3] = (int64_t)W_total;
}

// Global draws j < s_R: t = mulhi(u_j, W) (Philox counter (j, 2 it + side), reading Z6); a draw in
// this block's mass range is resolved in the local inclusive prefix P: first i with P_i > t - W_off.
__global__ void samp_draws_shard(const uint64_t* __restrict__ P, int64_t n, uint64_t seed, uint32_t iteration,
                                 uint32_t side, const int64_t* __restrict__ counts, const uint64_t* __restrict__ wloc,
                                 uint64_t W_off, int32_t* __restrict__ cnt, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t sR = counts[1];
  const uint64_t W = (uint64_t)counts[3], Wb = *wloc;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < sR; j += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = philox4x32_10(make_uint4((uint32_t)j, (uint32_t)((uint64_t)j >> 32), 2u * iteration + side, 0u),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    const uint64_t u = ((uint64_t)x.y << 32) | (uint64_t)x.x;
    const uint64_t t = __umul64hi(u, W);
    if (t < W_off || t - W_off >= Wb) continue;
    const uint64_t tl = t - W_off;
    int64_t lo = 0, hi = n - 1;   // P[n-1] = Wb > tl
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (P[mid] > tl) hi = mid; else lo = mid + 1;
    }
    atomicAdd(cnt + lo, 1);
  }
}

__global__ void shift_rows_kernel(int32_t* __restrict__ uniq, const int64_t* __restrict__ counts, int64_t row0,
                                  const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t nu = counts[2];
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nu; t += (int64_t)gridDim.x * blockDim.x)
    uniq[t] = (int32_t)(uniq[t] + row0);
}

// ---------------------------------------------------------------- scaled plan rows, pull product
__global__ void plan_rows_scaled_kernel(const float* __restrict__ F, int64_t row0, int k,
                                        const int32_t* __restrict__ uniq, const double* __restrict__ w,
                                        const int64_t* __restrict__ counts, float* __restrict__ Z,
                                        const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t nu = counts[2];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nu * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / k;
    const int c = (int)(e - t * k);
    Z[e] = (float)w[t] * F[(uniq[t] - row0) * k + c];
  }
}

__global__ void slot_fill_kernel(int32_t* __restrict__ slot, int64_t n, const int32_t* __restrict__ uniq,
                                 const int64_t* __restrict__ n_uniq_dev, int phase, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t step = (int64_t)gridDim.x * blockDim.x, i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (phase == 0) {
    for (int64_t i = i0; i < n; i += step) slot[i] = -1;
  } else {
    const int64_t nu = *n_uniq_dev;
    for (int64_t t = i0; t < nu; t += step) slot[uniq[t]] = (int32_t)t;
  }
}

// Y[r] = sum over row r's nonzeros (c, a) with slot[c] >= 0 of a Z[slot[c]]; k/4 lanes per row.
template <int LPR>
__global__ void __launch_bounds__(256) pull_rows_v4(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                                    const float* __restrict__ val, int64_t nb,
                                                    const int32_t* __restrict__ slot, const float4* __restrict__ Z4,
                                                    float4* __restrict__ Y4, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int li = threadIdx.x % LPR;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; r < nb; r += ng) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
      const int t = __ldg(slot + __ldg(col + e));
      if (t < 0) continue;
      const float a = __ldg(val + e);
      const float4 z = __ldg(Z4 + (int64_t)t * LPR + li);
      acc.x = fmaf(a, z.x, acc.x); acc.y = fmaf(a, z.y, acc.y);
      acc.z = fmaf(a, z.z, acc.z); acc.w = fmaf(a, z.w, acc.w);
    }
    Y4[r * LPR + li] = acc;
  }
}

__global__ void __launch_bounds__(256) pull_rows_scalar(const int64_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ col, const float* __restrict__ val,
                                                        int64_t nb, const int32_t* __restrict__ slot,
                                                        const float* __restrict__ Z, int k, float* __restrict__ Y,
                                                        const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nb; r += nw) {
    float a0 = 0.f, a1 = 0.f;
    for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
      const int t = __ldg(slot + __ldg(col + e));
      if (t < 0) continue;
      const float a = __ldg(val + e);
      if (lane < k) a0 = fmaf(a, Z[(int64_t)t * k + lane], a0);
      if (lane + 32 < k) a1 = fmaf(a, Z[(int64_t)t * k + lane + 32], a1);
    }
    if (lane < k) Y[r * k + lane] = a0;
    if (lane + 32 < k) Y[r * k + lane + 32] = a1;
  }
}

static int grid_cap(int64_t threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((threads + 255) / 256, 148 * 16));
}

void launch_shard_sums(const float* lev, int64_t n, double T, const SamplerWs& w, uint64_t* W_out, int64_t* sD_out,
                       double* theta_out, int32_t* status, cudaStream_t st) {
  const int64_t nb = samp_blocks(n);
  launch_samp_block_sums(lev, n, T, w, status, st);
  shard_sums_kernel<<<1, 1024, 0, st>>>(w.bw, w.bd, w.bt, nb, W_out, sD_out, theta_out, status);
}

void launch_shard_plan(const float* lev, int64_t n, int64_t row0, int k, int64_t s, double T, uint64_t seed,
                       uint32_t iteration, uint32_t side, uint64_t W_off, uint64_t W_total, int64_t sD_total,
                       const symnmf_plan& plan, const SamplerWs& w, uint64_t* wloc, int32_t* status,
                       cudaStream_t st) {
  launch_samp_block_sums(lev, n, T, w, status, st);
  launch_samp_scan_blocks(n, s, k, plan, w, status, st);        // local offsets and local totals
  shard_fix_kernel<<<1, 1, 0, st>>>(plan.counts, wloc, s, sD_total, W_total, status);
  launch_samp_prefix(lev, n, T, w, plan, status, st);           // local inclusive prefix, local I_D
  samp_draws_shard<<<grid_cap(s), 256, 0, st>>>(w.P, n, seed, iteration, side, plan.counts, wloc, W_off, w.cnt,
                                                status);
  launch_samp_uniq(lev, n, T, w, plan, status, st);             // compaction, weights with the global W, s_R
  shift_rows_kernel<<<grid_cap(plan.cap), 256, 0, st>>>(plan.uniq_idx, plan.counts, row0, status);
}

void launch_plan_rows_scaled(const float* F, int64_t row0, int k, const symnmf_plan& plan, float* Z,
                             const int32_t* status, cudaStream_t st) {
  plan_rows_scaled_kernel<<<grid_cap(plan.cap * k), 256, 0, st>>>(F, row0, k, plan.uniq_idx, plan.uniq_w,
                                                                   plan.counts, Z, status);
}

void launch_sampled_rows_pull(const symnmf_matrix& Ab, int64_t n_total, const int32_t* uniq,
                              const int64_t* n_uniq_dev, int64_t cap, const float* Z, int k, float* Y, int32_t* slot,
                              const int32_t* status, cudaStream_t st) {
  slot_fill_kernel<<<grid_cap(n_total), 256, 0, st>>>(slot, n_total, uniq, n_uniq_dev, 0, status);
  slot_fill_kernel<<<grid_cap(cap), 256, 0, st>>>(slot, n_total, uniq, n_uniq_dev, 1, status);
  const int64_t nb = Ab.n;
  if (k % 4 == 0 && (k / 4 == 1 || k / 4 == 2 || k / 4 == 4 || k / 4 == 8 || k / 4 == 16)) {
    const float4* Z4 = reinterpret_cast<const float4*>(Z);
    float4* Y4 = reinterpret_cast<float4*>(Y);
    const int grid = grid_cap(nb * (k / 4));
    switch (k / 4) {
      case 1: pull_rows_v4<1><<<grid, 256, 0, st>>>(Ab.rowptr, Ab.colidx, Ab.val, nb, slot, Z4, Y4, status); return;
      case 2: pull_rows_v4<2><<<grid, 256, 0, st>>>(Ab.rowptr, Ab.colidx, Ab.val, nb, slot, Z4, Y4, status); return;
      case 4: pull_rows_v4<4><<<grid, 256, 0, st>>>(Ab.rowptr, Ab.colidx, Ab.val, nb, slot, Z4, Y4, status); return;
      case 8: pull_rows_v4<8><<<grid, 256, 0, st>>>(Ab.rowptr, Ab.colidx, Ab.val, nb, slot, Z4, Y4, status); return;
      default: pull_rows_v4<16><<<grid, 256, 0, st>>>(Ab.rowptr, Ab.colidx, Ab.val, nb, slot, Z4, Y4, status); return;
    }
  }
  pull_rows_scalar<<<grid_cap(nb * 32), 256, 0, st>>>(Ab.rowptr, Ab.colidx, Ab.val, nb, slot, Z, k, Y, status);
}

}  // namespace symnmf
