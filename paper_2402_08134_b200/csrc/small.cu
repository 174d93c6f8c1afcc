// Persistent LvS-SymNMF iteration for problems that fit one wave of CTAs (n <= 2^20):
// one cooperative launch runs a whole iteration (W-half then H-half, Alg. LvS-SymNMF
// P:673-700), with grid-wide barriers between the steps instead of kernel boundaries.
// At these sizes (BASELINE c1, c2) every step is a few microseconds of memory latency,
// so a kernel per step is dominated by launch and drain; here a step costs one barrier.
// Measured on B200 (c2, 148 CTAs x 256 threads): 149 us / iteration against 131 us for the
// multi-kernel graph -- one 8-warp CTA per SM leaves each step latency-bound (sweep 37 us,
// sampled products 28 us, Cholesky 11 us) -- so the solver uses it only on request
// (SYMNMF_SMALL=always, symnmf.h).
//
// Per half (F fixed, X updated), between barriers B1..B7:
//   P1  scores l_i = ||f_i R^{-1}||^2 (Eq. 2.10; forward substitution with the
//       CholeskyQR factor R of F^T F) and per-1024-row sums of the integer mass
//       w_i = floor(l_i 2^40) (0 on I_D), of the I_D indicator and of theta (readings Z1, Z3, Z6)
//   P2  every CTA scans the block sums (nb <= 1024) itself: W, s_D, s_R (Z2), block offsets
//   P3  inclusive prefix P_i of w and the I_D compaction
//   P4  s_R draws: Philox4x32-10 (seed; j, 2 it + side) -> t = mulhi(u, W) -> first i, P_i > t
//   P5  per-block |U| counts (U = I_D u {drawn})
//   P6  every CTA scans them; U and omega_i (1 on I_D, c_i W / (s_R w_i) drawn)
//   P7  G_s = sum omega f f^T and Y_s = (SA)^T (SF)
//   P8  HALS sweep with (G_s + alpha I, Y_s + alpha F) (Eq. 2.6), X^T X partials
//   P9  every CTA forms X^T X and its Cholesky factor (the next half's R) itself
// The arithmetic of every step is that of the multi-kernel path (sampler.cu, fused.cu), so
// plans are bit-identical given identical scores.  Data written by other CTAs during the
// launch is read through L2 (ld.global.cg): L1 is not coherent across SMs.
#include "fused_common.cuh"
#include "small_args.cuh"

namespace symnmf {

constexpr int SM_T = 256;             // threads per CTA
constexpr int SM_NBMAX = 1024;        // sampler blocks (n <= 2^20)
constexpr double kTwo40s = 1099511627776.0;


// Grid-wide barrier over co-resident CTAs (cooperative launch): arrival counter reset by the
// last arriver, which then bumps the generation word the others spin on.
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    __threadfence();
    const unsigned int arrived = atomicAdd(bar, 1u) + 1u;
    if (arrived == gridDim.x) {
      bar[0] = 0u;
      __threadfence();
      atomicExch(bar + 1, gen);
    } else {
      while ((int)(*(volatile unsigned int*)(bar + 1) - gen) < 0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void sm_elem(const float* lev, int64_t i, int64_t n, double T, uint64_t& w, uint32_t& d,
                                        double& l) {
  if (i < n) {
    l = (double)lev[i];
    d = l >= T ? 1u : 0u;
    w = d ? 0ull : (uint64_t)__double2ull_rd(l * kTwo40s);
  } else {
    l = 0.0; d = 0u; w = 0ull;
  }
}

// Block exclusive scan of nb <= SM_NBMAX values, result in shared memory (in place), total returned.
template <typename T>
__device__ T cta_scan_array(T* s, int nb, T* sh) {
  T run = T(0);
  for (int base = 0; base < nb; base += SM_T) {
    const int i = base + threadIdx.x;
    const T v = i < nb ? s[i] : T(0);
    T tot;
    const T e = block_excl_scan(v, sh, &tot);
    if (i < nb) s[i] = run + e;
    run += tot;
  }
  __syncthreads();
  return run;
}

// Cholesky of G = sum of the replicas of acc (k x k upper) -> fp32 R (KP x KP upper) + 1/diag.
template <int KP>
__device__ void cta_chol(const double* acc, int k, double* sG, double* scratch, float* sR, double* Gout, bool write,
                         int32_t* status) {
  for (int e = threadIdx.x; e < k * k; e += SM_T) {
    const int a = e / k, b = e - a * k;
    if (a > b) continue;
    double v = 0.0;
#pragma unroll
    for (int r = 0; r < kGramReplicas; ++r) v += __ldcg(acc + (size_t)r * k * k + e);
    sG[a * k + b] = v;
    sG[b * k + a] = v;
    if (write) { Gout[a * k + b] = v; Gout[b * k + a] = v; }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int fail;
    if constexpr (KP <= 16) {
      fail = warp_chol_col<KP>(sG, k, 0.0, sR, sR + KP * KP);
    } else {
      fail = warp_chol_inv(scratch, scratch + k * (k + 1), sG, k, 0.0, /*inverse=*/false);
      if (!fail) {
        for (int e = threadIdx.x; e < KP * KP; e += 32) {
          const int i = e / KP, c = e - i * KP;
          sR[e] = (i <= c && c < k) ? (float)scratch[i * (k + 1) + c] : 0.f;
        }
        for (int c = threadIdx.x; c < KP; c += 32) sR[KP * KP + c] = c < k ? (float)(1.0 / scratch[c * (k + 1) + c]) : 0.f;
      }
    }
    if (fail && threadIdx.x == 0) dev_fail(status, SYMNMF_ERR_NOT_PD);
  }
  __syncthreads();
}

template <int KP>
struct SmallSmem {
  static constexpr int ST = KP + 4;
  static constexpr size_t offw = 0;                                           // uint64 [NBMAX + 1]
  static constexpr size_t offd = offw + sizeof(uint64_t) * (SM_NBMAX + 1);    // uint32 [NBMAX + 1]
  static constexpr size_t offu = offd + sizeof(uint32_t) * (SM_NBMAX + 1);    // uint32 [NBMAX + 1]
  static constexpr size_t rbuf = (offu + sizeof(uint32_t) * (SM_NBMAX + 1) + 15) / 16 * 16;   // float KP*KP + KP
  static constexpr size_t gbuf = rbuf + sizeof(float) * (KP * KP + KP);       // double KP*KP
  static constexpr size_t chol = gbuf + sizeof(double) * KP * KP;             // double 2 KP (KP+1)
  static constexpr size_t work = (chol + sizeof(double) * 2 * KP * (KP + 1) + 15) / 16 * 16;   // phase scratch
  static constexpr size_t work_bytes = std::max(sizeof(float) * 2 * 256 * ST, sizeof(double) * 256 * 16);
  static constexpr size_t bytes = work + work_bytes;
};

template <int KP>
__global__ void __launch_bounds__(SM_T, 1) lvs_small_iteration(const SmallArgs a) {
  using L = SmallSmem<KP>;
  constexpr int ST = L::ST, Q = KP / 4;
  extern __shared__ __align__(16) unsigned char sms[];
  uint64_t* sOffW = reinterpret_cast<uint64_t*>(sms + L::offw);
  uint32_t* sOffD = reinterpret_cast<uint32_t*>(sms + L::offd);
  uint32_t* sOffU = reinterpret_cast<uint32_t*>(sms + L::offu);
  float* sR = reinterpret_cast<float*>(sms + L::rbuf);
  double* sGd = reinterpret_cast<double*>(sms + L::gbuf);
  double* sChol = reinterpret_cast<double*>(sms + L::chol);
  float* wk = reinterpret_cast<float*>(sms + L::work);
  __shared__ uint64_t shw[33];
  __shared__ uint32_t shd[33];
  __shared__ double sht[33];
  __shared__ __align__(16) float sG[KP * KP];
  __shared__ float sInv[KP];
  __shared__ int sOk[KP];
  __shared__ int64_t srow[64];
  __shared__ float swt[64];

  pdl_wait();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int64_t n = a.n;
  const int k = a.k;
  const int64_t nb = (n + kSampBlock - 1) / kSampBlock;
  unsigned int gen = *(volatile unsigned int*)(a.bar + 1);
  const uint32_t it = (uint32_t)*a.iter_dev;
  for (int e = tid; e < KP * KP + KP; e += SM_T) sR[e] = a.R32[e];
  __syncthreads();

  for (int side = 0; side < 2; ++side) {
    const float* F = side == 0 ? a.H : a.W;   // W-half: H fixed; H-half: W fixed
    float* X = side == 0 ? a.W : a.H;
    // ---------------- P1: scores + block sums
    for (int64_t b = blockIdx.x; b < nb; b += G) {
      uint64_t sw = 0;
      uint32_t sd = 0;
      double stt = 0.0;
      for (int sub = 0; sub < kSampBlock / 256; ++sub) {
        const int64_t r0 = b * kSampBlock + sub * 256;
        const int rows = (int)max64(0, min64(256, n - r0));
        __syncthreads();
        for (int e = tid; e < rows * Q; e += SM_T) {
          const int r = e / Q, c = e - r * Q;
          *reinterpret_cast<float4*>(wk + r * ST + 4 * c) = __ldcg(reinterpret_cast<const float4*>(F + r0 * KP) + e);
        }
        __syncthreads();
        if (tid < rows) {
          float f[KP];
#pragma unroll
          for (int c = 0; c < KP; c += 4) {
            const float4 v = *reinterpret_cast<const float4*>(wk + tid * ST + c);
            f[c] = v.x; f[c + 1] = v.y; f[c + 2] = v.z; f[c + 3] = v.w;
          }
          float l = 0.f;
#pragma unroll
          for (int c = 0; c < KP; ++c) {
            const float q = f[c] * sR[KP * KP + c];
            l = fmaf(q, q, l);
#pragma unroll
            for (int d = c + 1; d < KP; ++d) f[d] = fmaf(-q, sR[c * KP + d], f[d]);
          }
          a.lev[r0 + tid] = l;
          const double ld = (double)l;
          const bool det = ld >= a.T;                                    // reading Z1
          sw += det ? 0ull : (uint64_t)__double2ull_rd(ld * kTwo40s);   // reading Z6
          sd += det ? 1u : 0u;
          stt += det ? ld : 0.0;
        }
      }
      sw = block_sum(sw, shw);
      sd = block_sum(sd, shd);
      stt = block_sum(stt, sht);
      if (tid == 0) { a.bw[b] = sw; a.bd[b] = sd; a.bt[b] = stt; }
    }
    grid_barrier(a.bar, gen);                                                            // B1
    // ---------------- P2: block offsets, W, s_D, s_R (every CTA)
    for (int64_t i = tid; i < nb; i += SM_T) { sOffW[i] = __ldcg(a.bw + i); sOffD[i] = __ldcg(a.bd + i); }
    double th = 0.0;
    for (int64_t i = tid; i < nb; i += SM_T) th += __ldcg(a.bt + i);
    __syncthreads();
    const uint64_t Wt = cta_scan_array<uint64_t>(sOffW, (int)nb, shw);
    const uint32_t sDt = cta_scan_array<uint32_t>(sOffD, (int)nb, shd);
    th = block_sum(th, sht);
    const int64_t sD = (int64_t)sDt;
    const int64_t sR_ = (Wt == 0ull) ? 0 : (a.s > sD ? a.s - sD : 0);             // reading Z2
    if (blockIdx.x == 0) {
      if (tid == 0) {
        a.plan.counts[0] = sD;
        a.plan.counts[1] = sR_;
        a.plan.counts[3] = (int64_t)Wt;
        a.plan.mass[0] = th;
        a.plan.mass[1] = (double)k - th;
        if (sD > a.plan.cap) dev_fail(a.status, SYMNMF_ERR_CAPACITY);
      }
      for (int e = tid; e < kGramReplicas * k * k; e += SM_T) a.GAcc[e] = 0.0;   // read by all in P9 before B1
    }
    // ---------------- P3: prefix P and I_D compaction
    for (int64_t b = blockIdx.x; b < nb; b += G) {
      const int64_t i0 = b * kSampBlock + tid * 4;
      uint64_t w[4];
      uint32_t d[4];
      uint64_t tw = 0;
      uint32_t td = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        double l;
        sm_elem(a.lev, i0 + e, n, a.T, w[e], d[e], l);
        tw += w[e]; td += d[e];
      }
      const uint64_t ew = block_excl_scan(tw, shw, (uint64_t*)nullptr) + sOffW[b];
      const uint32_t ed = block_excl_scan(td, shd, (uint32_t*)nullptr) + sOffD[b];
      uint64_t run = ew;
      uint32_t rd = ed;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + e;
        run += w[e];
        if (i < n) {
          a.P[i] = run;
          if (d[e]) { if ((int64_t)rd < a.plan.cap) a.plan.det_idx[rd] = (int32_t)i; ++rd; }
        }
      }
    }
    grid_barrier(a.bar, gen);                                                            // B2
    // ---------------- P4: draws
    for (int64_t j = (int64_t)blockIdx.x * SM_T + tid; j < sR_; j += (int64_t)G * SM_T) {
      const uint4 x = philox4x32_10(make_uint4((uint32_t)j, (uint32_t)((uint64_t)j >> 32), 2u * it + side, 0u),
                                    make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32)));
      const uint64_t u = ((uint64_t)x.y << 32) | (uint64_t)x.x;
      const uint64_t t = __umul64hi(u, Wt);
      int64_t bl = 0, bh = nb - 1;            // largest b with offset <= t
      while (bl < bh) {
        const int64_t mid = (bl + bh + 1) >> 1;
        if (sOffW[mid] <= t) bl = mid; else bh = mid - 1;
      }
      int64_t lo = bl * kSampBlock, hi = min64(n, lo + kSampBlock) - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldcg(a.P + mid) > t) hi = mid; else lo = mid + 1;
      }
      a.plan.draw_idx[j] = (int32_t)lo;
      atomicAdd(a.cnt + lo, 1);
    }
    grid_barrier(a.bar, gen);                                                            // B3
    // ---------------- P5: |U| per block
    for (int64_t b = blockIdx.x; b < nb; b += G) {
      const int64_t i0 = b * kSampBlock + tid * 4;
      uint32_t c = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + e;
        if (i < n) c += ((double)a.lev[i] >= a.T || __ldcg(a.cnt + i) > 0) ? 1u : 0u;
      }
      c = block_sum(c, shd);
      if (tid == 0) a.bu[b] = c;
    }
    grid_barrier(a.bar, gen);                                                            // B4
    // ---------------- P6: U and omega
    for (int64_t i = tid; i < nb; i += SM_T) sOffU[i] = __ldcg(a.bu + i);
    __syncthreads();
    const uint32_t nU = cta_scan_array<uint32_t>(sOffU, (int)nb, shd);
    if (blockIdx.x == 0 && tid == 0) {
      a.plan.counts[2] = (int64_t)nU;
      if ((int64_t)nU > a.plan.cap) dev_fail(a.status, SYMNMF_ERR_CAPACITY);
      const int tt = (int)it - a.first_iter;
      if (a.stats && tt >= 0 && tt < a.max_iters) {
        symnmf_half_stats h;
        h.s_d = sD; h.s_r = sR_; h.n_uniq = (int64_t)nU; h.theta = th;
        a.stats[2 * tt + side] = h;
      }
    }
    const int64_t nu = min64((int64_t)nU, a.plan.cap);
    for (int64_t b = blockIdx.x; b < nb; b += G) {
      const int64_t i0 = b * kSampBlock + tid * 4;
      uint32_t f[4];
      int32_t c[4];
      double l[4];
      uint32_t tf = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + e;
        if (i < n) {
          l[e] = (double)a.lev[i];
          c[e] = __ldcg(a.cnt + i);
          f[e] = (l[e] >= a.T || c[e] > 0) ? 1u : 0u;
        } else { l[e] = 0.0; c[e] = 0; f[e] = 0u; }
        tf += f[e];
      }
      uint32_t r = block_excl_scan(tf, shd, (uint32_t*)nullptr) + sOffU[b];
      const double Wd = (double)Wt, sRd = (double)sR_;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + e;
        if (!f[e]) continue;
        if ((int64_t)r < a.plan.cap) {
          a.plan.uniq_idx[r] = (int32_t)i;
          double om;
          if (l[e] >= a.T) om = 1.0;
          else {
            const double wi = (double)(uint64_t)__double2ull_rd(l[e] * kTwo40s);
            om = __dmul_rn((double)c[e], __ddiv_rn(Wd, __dmul_rn(sRd, wi)));
          }
          a.plan.uniq_w[r] = om;
        }
        ++r;
        if (c[e]) a.cnt[i] = 0;
      }
    }
    grid_barrier(a.bar, gen);                                                            // B5
    // ---------------- P7: G_s partials and Y_s
    {
      GramThread gt;
      gt.init(tid, SM_T, KP / 4);
      const int64_t per = (nu + G - 1) / G;
      const int64_t u0 = blockIdx.x * per, u1 = min64(nu, u0 + per);
      for (int64_t r0 = u0; r0 < u1; r0 += 64) {
        const int rows = (int)min64(64, u1 - r0);
        __syncthreads();
        if (tid < 64) {
          const bool ok = tid < rows;
          srow[tid] = ok ? (int64_t)__ldcg(a.plan.uniq_idx + r0 + tid) : 0;
          swt[tid] = ok ? (float)__ldcg(a.plan.uniq_w + r0 + tid) : 0.f;
        }
        __syncthreads();
        for (int e = tid; e < rows * Q; e += SM_T) {
          const int r = e / Q, c = e - r * Q;
          *reinterpret_cast<float4*>(wk + r * ST + 4 * c) = __ldcg(reinterpret_cast<const float4*>(F + srow[r] * KP) + c);
        }
        __syncthreads();
        gt.accumulate(wk, ST, rows, swt);
      }
      gt.commit(a.GsAcc, k, reinterpret_cast<double*>(wk));
      if (a.kind == SYMNMF_CSR) {   // scatter omega_i A[i,c] f_i into row c of Y_s (vector red.add)
        const int li = lane % Q, sub = lane / Q, npw = 32 / Q;
        const int64_t nwarps = (int64_t)G * (SM_T / 32);
        for (int64_t u = (int64_t)blockIdx.x * (SM_T / 32) + wid; u < nu; u += nwarps) {
          const int64_t i = __ldcg(a.plan.uniq_idx + u);
          const float om = (float)__ldcg(a.plan.uniq_w + u);
          float4 f = __ldcg(reinterpret_cast<const float4*>(F + i * KP) + li);
          f.x *= om; f.y *= om; f.z *= om; f.w *= om;
          const int64_t e1 = a.rowptr[i + 1];
          for (int64_t e = a.rowptr[i] + sub; e < e1; e += npw) {
            const int64_t c = __ldg(a.colidx + e);
            const float v = __ldg(a.val + e);
            atomicAdd(reinterpret_cast<float4*>(a.Y + c * KP) + li, make_float4(v * f.x, v * f.y, v * f.z, v * f.w));
          }
        }
      } else {                      // dense: y_c = sum_u A[U_u, c] omega_u f_u, thread per (c, 4 columns)
        for (int64_t q = (int64_t)blockIdx.x * SM_T + tid; q < n * Q; q += (int64_t)G * SM_T) {
          const int64_t c = q / Q;
          const int cq = (int)(q - c * Q);
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          double4 acc64 = make_double4(0.0, 0.0, 0.0, 0.0);
          for (int64_t u = 0; u < nu; ++u) {
            const int64_t i = __ldcg(a.plan.uniq_idx + u);
            const float v = __ldg(a.val + i * a.lda + c) * (float)__ldcg(a.plan.uniq_w + u);
            const float4 f = __ldcg(reinterpret_cast<const float4*>(F + i * KP) + cq);
            acc.x = fmaf(v, f.x, acc.x); acc.y = fmaf(v, f.y, acc.y); acc.z = fmaf(v, f.z, acc.z); acc.w = fmaf(v, f.w, acc.w);
            if ((u & 31) == 31) {
              acc64.x += acc.x; acc64.y += acc.y; acc64.z += acc.z; acc64.w += acc.w;
              acc = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          reinterpret_cast<float4*>(a.Y + c * KP)[cq] =
              make_float4((float)(acc64.x + acc.x), (float)(acc64.y + acc.y), (float)(acc64.z + acc.z),
                          (float)(acc64.w + acc.w));
        }
      }
    }
    grid_barrier(a.bar, gen);                                                            // B6
    // ---------------- P8: sweep with G_s + alpha I, b = Y_s + alpha F; X^T X partials
    {
      for (int e = tid; e < KP * KP; e += SM_T) {
        const int i = e / KP, j = e - i * KP;
        double v = 0.0;
        if (i != j) {
#pragma unroll
          for (int r = 0; r < kGramReplicas; ++r) {
            const int aa = min(i, j), bb = max(i, j);
            v += __ldcg(a.GsAcc + (size_t)r * k * k + aa * k + bb);
          }
        }
        sG[e] = (float)v;   // symmetric: sG[i][j] = G_s[j][i]
      }
      for (int i = tid; i < KP; i += SM_T) {
        double g = 0.0;
#pragma unroll
        for (int r = 0; r < kGramReplicas; ++r) g += __ldcg(a.GsAcc + (size_t)r * k * k + i * k + i);
        const double den = g + a.alpha;
        sOk[i] = den > 0.0;
        sInv[i] = den > 0.0 ? (float)(1.0 / den) : 0.f;
      }
      __syncthreads();
      GramThread gt;
      gt.init(tid, SM_T, KP / 4);
      const float a32 = (float)a.alpha;
      float* sX = wk;
      float* sB = wk + 256 * ST;
      const int64_t tiles = (n + 255) / 256;
      for (int64_t t = blockIdx.x; t < tiles; t += G) {
        const int64_t r0 = t * 256;
        const int rows = (int)min64(256, n - r0);
        __syncthreads();
        for (int e = tid; e < rows * Q; e += SM_T) {
          const int r = e / Q, c = e - r * Q;
          const float4 y = __ldcg(reinterpret_cast<const float4*>(a.Y + r0 * KP) + e);
          const float4 f = __ldcg(reinterpret_cast<const float4*>(F + r0 * KP) + e);
          float4 b;
          b.x = fmaf(a32, f.x, y.x); b.y = fmaf(a32, f.y, y.y); b.z = fmaf(a32, f.z, y.z); b.w = fmaf(a32, f.w, y.w);
          *reinterpret_cast<float4*>(sB + r * ST + 4 * c) = b;
          *reinterpret_cast<float4*>(sX + r * ST + 4 * c) = __ldcg(reinterpret_cast<const float4*>(X + r0 * KP) + e);
          if (a.kind == SYMNMF_CSR) reinterpret_cast<float4*>(a.Y + r0 * KP)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        if (tid < rows) {
          float x[KP];
          const float* brow = sB + tid * ST;
#pragma unroll
          for (int j = 0; j < KP; j += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(sX + tid * ST + j);
            x[j] = xv.x; x[j + 1] = xv.y; x[j + 2] = xv.z; x[j + 3] = xv.w;
          }
#pragma unroll
          for (int i = 0; i < KP; ++i) {
            float s0 = brow[i], s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int j = 0; j < KP; j += 4) {
              const float4 g = *reinterpret_cast<const float4*>(sG + i * KP + j);
              s0 = fmaf(-x[j], g.x, s0);
              s1 = fmaf(-x[j + 1], g.y, s1);
              s2 = fmaf(-x[j + 2], g.z, s2);
              s3 = fmaf(-x[j + 3], g.w, s3);
            }
            const float sv = (s0 + s1) + (s2 + s3);
            if (sOk[i]) x[i] = fmaxf(0.f, sv * sInv[i]);
          }
#pragma unroll
          for (int j = 0; j < KP; j += 4)
            *reinterpret_cast<float4*>(sX + tid * ST + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
        }
        __syncthreads();
        for (int e = tid; e < rows * Q; e += SM_T) {
          const int r = e / Q, c = e - r * Q;
          reinterpret_cast<float4*>(X + r0 * KP)[e] = *reinterpret_cast<const float4*>(sX + r * ST + 4 * c);
        }
        gt.accumulate(sX, ST, rows, nullptr);
      }
      gt.commit(a.GAcc, k, reinterpret_cast<double*>(wk));
    }
    grid_barrier(a.bar, gen);                                                            // B7
    // ---------------- P9: X^T X and its Cholesky factor (every CTA); G_s accumulator reset
    cta_chol<KP>(a.GAcc, k, sGd, sChol, sR, a.Gout, blockIdx.x == 0, a.status);
    if (blockIdx.x == 0)
      for (int e = tid; e < kGramReplicas * k * k; e += SM_T) a.GsAcc[e] = 0.0;   // all CTAs read it before B7
  }
  if (blockIdx.x == 0) {
    for (int e = tid; e < KP * KP + KP; e += SM_T) a.R32[e] = sR[e];
    if (tid == 0) *a.iter_dev = (int32_t)it + 1;
  }
}

bool small_lvs_supported(const symnmf_matrix& A, int64_t n, int k) {
  if (kpad(k) != k || k > 32 || n > (int64_t)SM_NBMAX * kSampBlock) return false;
  if (A.kind == SYMNMF_CSR) return n <= (1 << 20);
  return n <= 4096;   // dense: the sampled gather is the hot spot beyond this (sampled_dense_v2)
}

template <int KP>
static bool launch_small_t(const SmallArgs& a, cudaStream_t st) {
  const size_t smem = SmallSmem<KP>::bytes;
  if (cudaFuncSetAttribute(lvs_small_iteration<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return false;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lvs_small_iteration<KP>, SM_T, smem) != cudaSuccess || occ < 1)
    return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);   // one CTA per SM: co-resident (cooperative launch)
  cfg.blockDim = dim3(SM_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, lvs_small_iteration<KP>, a) == cudaSuccess;
}

bool launch_small_lvs(const SmallArgs& a, cudaStream_t st) {
  switch (a.k) {
    case 8: return launch_small_t<8>(a, st);
    case 16: return launch_small_t<16>(a, st);
    case 32: return launch_small_t<32>(a, st);
    default: return false;
  }
}

}  // namespace symnmf
