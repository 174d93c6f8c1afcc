// (a4)-(a7) Hybrid deterministic / random leverage-score sampling plan
// (Eq. 2.11), bit-exact by construction (readings Z1-Z6):
//   S1 per-block sums of the integer mass w_i = floor(l_i 2^40) (0 on I_D),
//      of the I_D indicator and of theta = sum_{I_D} l_i
//   S2 one-CTA exclusive scan of the block sums -> W, s_D, s_R, theta, xi
//   S3 per-block inclusive prefix P_i (uint64) and compaction of I_D
//   S4 draws: Philox4x32-10 -> u -> t = mulhi(u, W) -> first i with P_i > t
//   S5-S7 compaction of U = I_D u {drawn} with omega_i = c_i * (W / (s_R w_i))
// Integer sums are associative, so the parallel result equals the serial one.
#include "kernels.cuh"

namespace symnmf {

constexpr int ST = 256;                 // threads; 4 consecutive elements each
constexpr double kTwo40 = 1099511627776.0;

__device__ __forceinline__ void elem(const float* lev, int64_t i, int64_t n, double T, uint64_t& w, uint32_t& det,
                                     double& l) {
  if (i < n) {
    l = (double)lev[i];
    det = l >= T ? 1u : 0u;
    w = det ? 0ull : (uint64_t)__double2ull_rd(l * kTwo40);   // exact: power-of-two scaling then floor
  } else {
    l = 0.0; det = 0u; w = 0ull;
  }
}

__global__ void __launch_bounds__(ST) samp_block_sums(const float* __restrict__ lev, int64_t n, double T,
                                                      uint64_t* __restrict__ bw, uint32_t* __restrict__ bd,
                                                      double* __restrict__ bt, const int32_t* __restrict__ status) {
  __shared__ uint64_t shw[32];
  __shared__ uint32_t shd[32];
  __shared__ double sht[32];
  if (dev_failed(status)) return;
  const int64_t i0 = (int64_t)blockIdx.x * kSampBlock + threadIdx.x * 4;
  uint64_t sw = 0;
  uint32_t sd = 0;
  double stt = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    uint64_t w; uint32_t d; double l;
    elem(lev, i0 + e, n, T, w, d, l);
    sw += w; sd += d; stt += d ? l : 0.0;
  }
  sw = block_sum(sw, shw);
  sd = block_sum(sd, shd);
  stt = block_sum(stt, sht);
  if (threadIdx.x == 0) { bw[blockIdx.x] = sw; bd[blockIdx.x] = sd; bt[blockIdx.x] = stt; }
}

// One CTA of 1024 threads: exclusive offsets in place, totals into the plan.
__global__ void __launch_bounds__(1024) samp_scan_blocks(int64_t nb, uint64_t* __restrict__ bw,
                                                         uint32_t* __restrict__ bd, const double* __restrict__ bt,
                                                         int64_t s, int k, int64_t cap, int64_t* __restrict__ counts,
                                                         double* __restrict__ mass, int32_t* __restrict__ status) {
  __shared__ uint64_t shw[33];
  __shared__ uint32_t shd[33];
  __shared__ double sht[32];
  if (dev_failed(status)) return;
  uint64_t cw = 0;
  uint32_t cd = 0;
  double theta = 0.0;
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const uint64_t vw = i < nb ? bw[i] : 0ull;
    const uint32_t vd = i < nb ? bd[i] : 0u;
    const double vt = i < nb ? bt[i] : 0.0;
    uint64_t tw; uint32_t td;
    const uint64_t ew = block_excl_scan(vw, shw, &tw);
    const uint32_t ed = block_excl_scan(vd, shd, &td);
    const double st_ = block_sum(vt, sht);
    if (i < nb) { bw[i] = cw + ew; bd[i] = cd + ed; }
    cw += tw; cd += td;
    theta += st_;   // valid in warp 0, which writes the totals
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int64_t sD = (int64_t)cd;
    const int64_t sR = (cw == 0ull) ? 0 : (s > sD ? s - sD : 0);
    counts[0] = sD;
    counts[1] = sR;
    counts[3] = (int64_t)cw;
    mass[0] = theta;
    mass[1] = (double)k - theta;
    if (sD > cap) dev_fail(status, SYMNMF_ERR_CAPACITY);
  }
}

__global__ void __launch_bounds__(ST) samp_prefix(const float* __restrict__ lev, int64_t n, double T,
                                                  const uint64_t* __restrict__ bw, const uint32_t* __restrict__ bd,
                                                  uint64_t* __restrict__ P, int32_t* __restrict__ det_idx, int64_t cap,
                                                  const int32_t* __restrict__ status) {
  __shared__ uint64_t shw[33];
  __shared__ uint32_t shd[33];
  if (dev_failed(status)) return;
  const int64_t i0 = (int64_t)blockIdx.x * kSampBlock + threadIdx.x * 4;
  uint64_t w[4];
  uint32_t d[4];
  uint64_t tw = 0;
  uint32_t td = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    double l;
    elem(lev, i0 + e, n, T, w[e], d[e], l);
    tw += w[e]; td += d[e];
  }
  const uint64_t ew = block_excl_scan(tw, shw, (uint64_t*)nullptr) + bw[blockIdx.x];
  const uint32_t ed = block_excl_scan(td, shd, (uint32_t*)nullptr) + bd[blockIdx.x];
  uint64_t run = ew;
  uint32_t rd = ed;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t i = i0 + e;
    run += w[e];
    if (i < n) {
      P[i] = run;
      if (d[e]) { if ((int64_t)rd < cap) det_idx[rd] = (int32_t)i; ++rd; }
    }
  }
}

__global__ void samp_draws(const uint64_t* __restrict__ P, int64_t n, uint64_t seed, const int32_t* __restrict__ iter_dev,
                           uint32_t iteration, uint32_t side, const int64_t* __restrict__ counts,
                           int32_t* __restrict__ draw_idx, int32_t* __restrict__ cnt, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t sR = counts[1];
  if (j >= sR) return;
  const uint64_t W = (uint64_t)counts[3];
  const uint32_t it = iter_dev ? (uint32_t)*iter_dev : iteration;
  const uint4 x = philox4x32_10(make_uint4((uint32_t)j, (uint32_t)((uint64_t)j >> 32), 2u * it + side, 0u),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint64_t u = ((uint64_t)x.y << 32) | (uint64_t)x.x;
  const uint64_t t = __umul64hi(u, W);
  int64_t lo = 0, hi = n - 1;   // P[n-1] = W > t
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (P[mid] > t) hi = mid; else lo = mid + 1;
  }
  draw_idx[j] = (int32_t)lo;
  atomicAdd(cnt + lo, 1);
}

// Same draws; the search first locates the 1024-row block in the exclusive block offsets
// bw (staged in shared memory), then searches the block's slice of P (10 dependent loads).
// The index found is the same first i with P_i > t.
__global__ void samp_draws_2level(const uint64_t* __restrict__ P, const uint64_t* __restrict__ bw, int64_t nb,
                                  int64_t n, uint64_t seed, const int32_t* __restrict__ iter_dev, uint32_t iteration,
                                  uint32_t side, const int64_t* __restrict__ counts, int32_t* __restrict__ draw_idx,
                                  int32_t* __restrict__ cnt, const int32_t* __restrict__ status) {
  extern __shared__ uint64_t sbw[];
  if (dev_failed(status)) return;
  const int64_t sR = counts[1];
  if ((int64_t)blockIdx.x * blockDim.x >= sR) return;
  for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) sbw[i] = bw[i];
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= sR) return;
  const uint64_t W = (uint64_t)counts[3];
  const uint32_t it = iter_dev ? (uint32_t)*iter_dev : iteration;
  const uint4 x = philox4x32_10(make_uint4((uint32_t)j, (uint32_t)((uint64_t)j >> 32), 2u * it + side, 0u),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint64_t u = ((uint64_t)x.y << 32) | (uint64_t)x.x;
  const uint64_t t = __umul64hi(u, W);
  int64_t bl = 0, bh = nb - 1;          // largest b with bw[b] <= t (bw[0] = 0 <= t)
  while (bl < bh) {
    const int64_t mid = (bl + bh + 1) >> 1;
    if (sbw[mid] <= t) bl = mid; else bh = mid - 1;
  }
  int64_t lo = bl * kSampBlock, hi = min64(n, lo + kSampBlock) - 1;   // P[hi] > t
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (P[mid] > t) hi = mid; else lo = mid + 1;
  }
  draw_idx[j] = (int32_t)lo;
  atomicAdd(cnt + lo, 1);
}

// Same draws, one warp per draw: the search first locates the 1024-row block in the exclusive
// block offsets bw (staged in shared memory; lane-uniform), then the warp counts the entries P_i <= t of the block's slice with 32
// independent coalesced loads per lane instead of 10 dependent ones.  P is non-decreasing and
// P[block end] > t, so block start + that count is the same first i with P_i > t.
__global__ void __launch_bounds__(256) samp_draws_warp(const uint64_t* __restrict__ P, const uint64_t* __restrict__ bw,
                                                       int64_t nb, int64_t n, uint64_t seed,
                                                       const int32_t* __restrict__ iter_dev, uint32_t iteration,
                                                       uint32_t side, const int64_t* __restrict__ counts,
                                                       int32_t* __restrict__ draw_idx, int32_t* __restrict__ cnt,
                                                       const int32_t* __restrict__ status) {
  extern __shared__ uint64_t sbw[];
  if (dev_failed(status)) return;
  const int64_t sR = counts[1];
  const int64_t j0 = (int64_t)blockIdx.x * 8;
  if (j0 >= sR) return;
  for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) sbw[i] = bw[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t j = j0 + (threadIdx.x >> 5);
  if (j >= sR) return;
  const uint64_t W = (uint64_t)counts[3];
  const uint32_t it = iter_dev ? (uint32_t)*iter_dev : iteration;
  const uint4 x = philox4x32_10(make_uint4((uint32_t)j, (uint32_t)((uint64_t)j >> 32), 2u * it + side, 0u),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint64_t u = ((uint64_t)x.y << 32) | (uint64_t)x.x;
  const uint64_t t = __umul64hi(u, W);
  int64_t bl = 0, bh = nb - 1;          // largest b with bw[b] <= t (bw[0] = 0 <= t)
  while (bl < bh) {
    const int64_t mid = (bl + bh + 1) >> 1;
    if (sbw[mid] <= t) bl = mid; else bh = mid - 1;
  }
  const int64_t lo = bl * kSampBlock, len = min64(n, lo + kSampBlock) - lo;
  int c = 0;
#pragma unroll 8
  for (int q = 0; q < kSampBlock / 32; ++q) {
    const int64_t e = (int64_t)q * 32 + lane;
    if (e < len) c += (__ldcg(P + lo + e) <= t) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) {
    draw_idx[j] = (int32_t)(lo + c);
    atomicAdd(cnt + lo + c, 1);
  }
}

__global__ void __launch_bounds__(ST) samp_uniq_counts(const float* __restrict__ lev, int64_t n, double T,
                                                       const int32_t* __restrict__ cnt, uint32_t* __restrict__ bu,
                                                       const int32_t* __restrict__ status) {
  __shared__ uint32_t sh[32];
  if (dev_failed(status)) return;
  const int64_t i0 = (int64_t)blockIdx.x * kSampBlock + threadIdx.x * 4;
  uint32_t c = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t i = i0 + e;
    if (i < n) c += ((double)lev[i] >= T || cnt[i] > 0) ? 1u : 0u;
  }
  c = block_sum(c, sh);
  if (threadIdx.x == 0) bu[blockIdx.x] = c;
}

__global__ void __launch_bounds__(1024) samp_scan_uniq(int64_t nb, uint32_t* __restrict__ bu, int64_t cap,
                                                       int64_t* __restrict__ counts, int32_t* __restrict__ status) {
  __shared__ uint32_t sh[33];
  if (dev_failed(status)) return;
  uint32_t c = 0;
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < nb ? bu[i] : 0u;
    uint32_t tot;
    const uint32_t e = block_excl_scan(v, sh, &tot);
    if (i < nb) bu[i] = c + e;
    c += tot;
  }
  if (threadIdx.x == 0) {
    counts[2] = (int64_t)c;
    if ((int64_t)c > cap) dev_fail(status, SYMNMF_ERR_CAPACITY);
  }
}

__global__ void __launch_bounds__(ST) samp_uniq_write(const float* __restrict__ lev, int64_t n, double T,
                                                      int32_t* __restrict__ cnt, const uint32_t* __restrict__ bu,
                                                      const int64_t* __restrict__ counts, int32_t* __restrict__ uniq,
                                                      double* __restrict__ uw, int64_t cap,
                                                      const int32_t* __restrict__ status) {
  __shared__ uint32_t sh[33];
  if (dev_failed(status)) return;
  const int64_t i0 = (int64_t)blockIdx.x * kSampBlock + threadIdx.x * 4;
  uint32_t f[4];
  int32_t c[4];
  double l[4];
  uint32_t tf = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t i = i0 + e;
    if (i < n) {
      l[e] = (double)lev[i];
      c[e] = cnt[i];
      f[e] = (l[e] >= T || c[e] > 0) ? 1u : 0u;
    } else { l[e] = 0.0; c[e] = 0; f[e] = 0u; }
    tf += f[e];
  }
  uint32_t r = block_excl_scan(tf, sh, (uint32_t*)nullptr) + bu[blockIdx.x];
  const double W = (double)(uint64_t)counts[3];
  const double sR = (double)counts[1];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t i = i0 + e;
    if (!f[e]) continue;
    if ((int64_t)r < cap) {
      uniq[r] = (int32_t)i;
      double om;
      if (l[e] >= T) om = 1.0;
      else {
        const double wi = (double)(uint64_t)__double2ull_rd(l[e] * kTwo40);
        om = __dmul_rn((double)c[e], __ddiv_rn(W, __dmul_rn(sR, wi)));
      }
      uw[r] = om;
    }
    ++r;
    if (c[e]) cnt[i] = 0;   // leave the multiplicity buffer zeroed for the next plan
  }
}

void launch_samp_prefix(const float* lev, int64_t n, double T, const SamplerWs& w, const symnmf_plan& plan,
                        int32_t* status, cudaStream_t st) {
  launch_pdl(samp_prefix, (unsigned)samp_blocks(n), ST, 0, st, lev, n, T, w.bw, w.bd, w.P, plan.det_idx, plan.cap, status);
}

void launch_samp_draws(const SamplerWs& w, int64_t n, int64_t s, uint64_t seed, const int32_t* iter_dev,
                       uint32_t iteration, uint32_t side, const symnmf_plan& plan, int32_t* status, cudaStream_t st) {
  const int64_t dblocks = std::max<int64_t>(1, (s + 255) / 256);
  const int64_t nb = samp_blocks(n);
  // few draws over many prefix blocks: one warp per draw (c2: 8.0k -> 8.06k it/s); a one-block
  // prefix (c1, n = 1,000) is cheaper to binary-search (12.23k vs 12.54k it/s with the warp form)
  if (nb <= 6144 && nb >= 16 && s <= 8192) {
    launch_pdl(samp_draws_warp, (unsigned)std::max<int64_t>(1, (s + 7) / 8), 256, sizeof(uint64_t) * nb, st,
               w.P, w.bw, nb, n, seed, iter_dev, iteration, side, plan.counts, plan.draw_idx, w.cnt, status);
    return;
  }
  if (nb <= 6144) {   // many draws (c4: 18k): the warp form's 8 KB slice per draw costs more L2 than it saves
    launch_pdl(samp_draws_2level, (unsigned)dblocks, 256, sizeof(uint64_t) * nb, st,
               w.P, w.bw, nb, n, seed, iter_dev, iteration, side, plan.counts, plan.draw_idx, w.cnt, status);
    return;
  }
  launch_pdl(samp_draws, (unsigned)dblocks, 256, 0, st, w.P, n, seed, iter_dev, iteration, side, plan.counts, plan.draw_idx,
                                                w.cnt, status);
}

void launch_samp_uniq_write(const float* lev, int64_t n, double T, const SamplerWs& w, const symnmf_plan& plan,
                            int32_t* status, cudaStream_t st) {
  launch_pdl(samp_uniq_write, (unsigned)samp_blocks(n), ST, 0, st, lev, n, T, w.cnt, w.bu, plan.counts, plan.uniq_idx,
                                                           plan.uniq_w, plan.cap, status);
}

void launch_samp_block_sums(const float* lev, int64_t n, double T, const SamplerWs& w, int32_t* status,
                            cudaStream_t st) {
  samp_block_sums<<<(unsigned)samp_blocks(n), ST, 0, st>>>(lev, n, T, w.bw, w.bd, w.bt, status);
}

void launch_samp_scan_blocks(int64_t n, int64_t s, int k, const symnmf_plan& plan, const SamplerWs& w,
                             int32_t* status, cudaStream_t st) {
  samp_scan_blocks<<<1, 1024, 0, st>>>(samp_blocks(n), w.bw, w.bd, w.bt, s, k, plan.cap, plan.counts, plan.mass,
                                       status);
}

void launch_samp_uniq(const float* lev, int64_t n, double T, const SamplerWs& w, const symnmf_plan& plan,
                      int32_t* status, cudaStream_t st) {
  const int64_t nb = samp_blocks(n);
  samp_uniq_counts<<<(unsigned)nb, ST, 0, st>>>(lev, n, T, w.cnt, w.bu, status);
  samp_scan_uniq<<<1, 1024, 0, st>>>(nb, w.bu, plan.cap, plan.counts, status);
  samp_uniq_write<<<(unsigned)nb, ST, 0, st>>>(lev, n, T, w.cnt, w.bu, plan.counts, plan.uniq_idx, plan.uniq_w,
                                               plan.cap, status);
}

void launch_hybrid_sample(const float* lev, int64_t n, int k, int64_t s, double T, uint64_t seed,
                          const int32_t* iter_dev, uint32_t iteration, uint32_t side, const symnmf_plan& plan,
                          const SamplerWs& w, int32_t* status, cudaStream_t st) {
  const int64_t nb = samp_blocks(n);
  samp_block_sums<<<(unsigned)nb, ST, 0, st>>>(lev, n, T, w.bw, w.bd, w.bt, status);
  samp_scan_blocks<<<1, 1024, 0, st>>>(nb, w.bw, w.bd, w.bt, s, k, plan.cap, plan.counts, plan.mass, status);
  samp_prefix<<<(unsigned)nb, ST, 0, st>>>(lev, n, T, w.bw, w.bd, w.P, plan.det_idx, plan.cap, status);
  launch_samp_draws(w, n, s, seed, iter_dev, iteration, side, plan, status, st);
  samp_uniq_counts<<<(unsigned)nb, ST, 0, st>>>(lev, n, T, w.cnt, w.bu, status);
  samp_scan_uniq<<<1, 1024, 0, st>>>(nb, w.bu, plan.cap, plan.counts, status);
  samp_uniq_write<<<(unsigned)nb, ST, 0, st>>>(lev, n, T, w.cnt, w.bu, plan.counts, plan.uniq_idx, plan.uniq_w,
                                               plan.cap, status);
}

}  // namespace symnmf
