// Fused kernels of the per-iteration hot loop (solver path):
//
//  gram_fused       G = F^T F (+ CholeskyQR factor R^{-1}) in ONE launch: per-CTA 4x4
//                   register-blocked partial Grams, fp64 red.add into a global accumulator,
//                   the last CTA to finish copies G out, re-zeroes the accumulator and (if
//                   asked) runs the one-warp fp64 Cholesky + triangular inverse.
//  sweep_fused      the HALS sweep (Eq. 2.6) of 256-row tiles staged with
//                   vectorised loads, fused with the Gram of the UPDATED factor (the next
//                   half's F^T F, P:420 / P:690) and its Cholesky in the last CTA; in LvS
//                   mode it also re-zeroes Y for the next sampled scatter.
//  leverage_fused   scores l_i = ||f_i R^{-1}||^2 fused with pass S1 of the
//                   sampler (integer mass / I_D counts per 1024-row block) and, in the last
//                   CTA, the block scan S2 (W, s_D, s_R, theta, xi, Z1-Z3).
//  uniq_count_fused pass S5 + block scan S6 of the plan compaction, and the per-half
//                   statistics record (s_D, s_R, |U|, theta).
//  sampled_gram_fused  G_s = sum_{i in U} omega_i f_i^T f_i over the compact plan.
// The "last CTA" pattern uses a per-call-site counter in the workspace that the last CTA
// resets, so the kernels are CUDA-graph replay safe.
#include <cstdlib>
#include "fused_common.cuh"


namespace symnmf {

// ---------------------------------------------------------------- gram_fused
constexpr int FT = 256;         // threads per CTA
constexpr size_t kRedBytes = sizeof(double) * 256 * 16;   // commit reduction scratch
constexpr int FROWS = 256;      // rows per staged tile

template <int KP>
__global__ void __launch_bounds__(FT) gram_fused(const float* __restrict__ F, int64_t n, int k, double* Gacc,
                                                 double* Gout, float* Rinv32, unsigned int* counter,
                                                 int32_t* status) {
  constexpr int ST = KP + 4;
  extern __shared__ __align__(16) unsigned char smf[];
  float* s = reinterpret_cast<float*>(smf);
  if (dev_failed(status)) return;
  GramThread gt;
  gt.init(threadIdx.x, FT, (k + 3) / 4);
  const int64_t tiles = (n + FROWS - 1) / FROWS;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t r0 = t * FROWS;
    const int rows = (int)min64(FROWS, n - r0);
    __syncthreads();
    if (k == KP) {
      const float4* src = reinterpret_cast<const float4*>(F + r0 * k);
      constexpr int Q = FROWS * KP / 4 / FT;   // float4 per thread
      float4 v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = threadIdx.x + q * FT;
        v[q] = (e < rows * (KP / 4)) ? __ldg(src + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = threadIdx.x + q * FT, r = e / (KP / 4), c = e - r * (KP / 4);
        *reinterpret_cast<float4*>(s + r * ST + 4 * c) = v[q];
      }
    } else {
      for (int e = threadIdx.x; e < FROWS * KP; e += FT) {
        const int r = e / KP, c = e - r * KP;
        s[r * ST + c] = (r < rows && c < k) ? F[(r0 + r) * k + c] : 0.f;
      }
    }
    __syncthreads();
    gt.accumulate(s, ST, rows, nullptr);
  }
  gt.commit(Gacc, k, reinterpret_cast<double*>(smf));
  if (arrive_last(counter)) {
    double* sa = reinterpret_cast<double*>(smf);
    finalize_gram<KP>(Gacc, Gout, k, Rinv32, sa, sa + k * (k + 1), status);
  }
}

// ---------------------------------------------------------------- sweep_fused
template <int KP>
__global__ void __launch_bounds__(FT, KP <= 32 ? 2 : 1) sweep_fused(const double* __restrict__ G, double alpha, float* __restrict__ Y,
                                                  const float* __restrict__ F, float* __restrict__ X, int64_t n, int k,
                                                  int zeroY, double* Gacc, double* Gout, float* Rinv32,
                                                  unsigned int* counter, int32_t* status) {
  constexpr int ST = KP + 4;
  constexpr int Q = KP / 4;       // float4 per lane per array (32-row warp tile)
  __shared__ __align__(16) float sG[KP * KP];     // sG[i*KP + j] = -G[j][i], 0 on the diagonal
  __shared__ float sInv[KP];
  __shared__ int sOk[KP];
  extern __shared__ __align__(16) unsigned char smw[];
  float* sX = reinterpret_cast<float*>(smw);        // [256][ST] updated rows (tile)
  float* sB = sX + FROWS * ST;                       // [256][ST] Y + alpha F
  if (dev_failed(status)) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < KP * KP; e += FT) {
    const int i = e / KP, j = e - i * KP;
    sG[e] = (i < k && j < k && i != j) ? -(float)G[j * k + i] : 0.f;
  }
  for (int i = tid; i < KP; i += FT) {
    const double den = i < k ? G[i * k + i] + alpha : 0.0;
    sOk[i] = den > 0.0;
    sInv[i] = den > 0.0 ? (float)(1.0 / den) : 0.f;
  }
  GramThread gt;
  gt.init(tid, FT, (k + 3) / 4);
  const float a32 = (float)alpha;
  __syncthreads();
  const int64_t tiles = (n + FROWS - 1) / FROWS;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t r0 = t * FROWS + wid * 32;          // this warp's 32 rows
    const int cnt = (int)max64(0, min64(32, n - r0));
    float* wX = sX + wid * 32 * ST;
    float* wB = sB + wid * 32 * ST;
    if (k == KP) {
      const float4* Y4 = reinterpret_cast<const float4*>(Y + r0 * k);
      const float4* F4 = reinterpret_cast<const float4*>(F + r0 * k);
      const float4* X4 = reinterpret_cast<const float4*>(X + r0 * k);
      float4 vy[Q], vf[Q], vx[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = lane + 32 * q;
        const bool ok = e < cnt * Q;
        vy[q] = ok ? __ldcs(Y4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        vf[q] = ok ? __ldg(F4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        vx[q] = ok ? X4[e] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = lane + 32 * q, r = e / Q, c = e - r * Q;
        float4 b;
        b.x = fmaf(a32, vf[q].x, vy[q].x); b.y = fmaf(a32, vf[q].y, vy[q].y);
        b.z = fmaf(a32, vf[q].z, vy[q].z); b.w = fmaf(a32, vf[q].w, vy[q].w);
        *reinterpret_cast<float4*>(wB + r * ST + 4 * c) = b;
        *reinterpret_cast<float4*>(wX + r * ST + 4 * c) = vx[q];
      }
    } else {
      for (int e = lane; e < 32 * KP; e += 32) {
        const int r = e / KP, c = e - r * KP;
        const bool ok = r < cnt && c < k;
        const int64_t gidx = (r0 + r) * k + c;
        wB[r * ST + c] = ok ? fmaf(a32, F[gidx], Y[gidx]) : 0.f;
        wX[r * ST + c] = ok ? X[gidx] : 0.f;
      }
    }
    __syncwarp();
    if (lane < cnt) {
      float2 x[KP / 2];   // column pairs (packed FFMA2); b = Y + alpha F stays in shared memory
      const float* brow = wB + lane * ST;
#pragma unroll
      for (int j = 0; j < KP; j += 4) {
        const float4 xv = *reinterpret_cast<const float4*>(wX + lane * ST + j);
        x[j / 2] = make_float2(xv.x, xv.y); x[j / 2 + 1] = make_float2(xv.z, xv.w);
      }
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        if (i < k) {
          // two independent packed partial sums: the column update is a short dependency chain
          float2 s01 = make_float2(brow[i], 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < KP; j += 4) {
            const float4 g = *reinterpret_cast<const float4*>(sG + i * KP + j);
            s01 = ffma2(x[j / 2], make_float2(g.x, g.y), s01);
            s23 = ffma2(x[j / 2 + 1], make_float2(g.z, g.w), s23);
          }
          const float s = (s01.x + s01.y) + (s23.x + s23.y);
          if (sOk[i]) {
            const float v = fmaxf(0.f, s * sInv[i]);
            if (i & 1) x[i / 2].y = v; else x[i / 2].x = v;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < KP; j += 4)
        *reinterpret_cast<float4*>(wX + lane * ST + j) = make_float4(x[j / 2].x, x[j / 2].y, x[j / 2 + 1].x, x[j / 2 + 1].y);
    } else {
#pragma unroll
      for (int j = 0; j < KP; j += 4)
        *reinterpret_cast<float4*>(wX + lane * ST + j) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();
    if (k == KP) {
      float4* X4 = reinterpret_cast<float4*>(X + r0 * k);
      float4* Y4 = reinterpret_cast<float4*>(Y + r0 * k);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = lane + 32 * q, r = e / Q, c = e - r * Q;
        if (e < cnt * Q) {
          X4[e] = *reinterpret_cast<const float4*>(wX + r * ST + 4 * c);
          if (zeroY) __stcs(Y4 + e, make_float4(0.f, 0.f, 0.f, 0.f));
        }
      }
    } else {
      for (int e = lane; e < cnt * k; e += 32) {
        const int r = e / k, c = e - r * k;
        X[(r0 + r) * k + c] = wX[r * ST + c];
        if (zeroY) Y[(r0 + r) * k + c] = 0.f;
      }
    }
    __syncthreads();
    if (Gacc) gt.accumulate(sX, ST, (int)min64(FROWS, n - t * FROWS), nullptr);
    __syncthreads();
  }
  if (!Gacc) return;
  gt.commit(Gacc, k, reinterpret_cast<double*>(smw));
  if (arrive_last(counter)) {
    double* sa = reinterpret_cast<double*>(smw);
    finalize_gram<KP>(Gacc, Gout, k, Rinv32, sa, sa + k * (k + 1), status);
  }
}

// ---------------------------------------------------------------- leverage_fused (+ S1, S2)
constexpr double kTwo40f = 1099511627776.0;

// Constant-bank copies of the CholeskyQR factor (R upper KP x KP | 1 / diag R), one per (solver
// slot, half), as for the sweep's G (sweep.cu): the forward substitution's R operands come from
// the constant cache into uniform registers instead of shared memory.
constexpr int kLevTabs = 8;
constexpr int kLevTab = 32 * 32 + 32;
__constant__ float cLev[kLevTabs][kLevTab];

template <int KP, int TAB>
struct LevR {
  const float* sR;
  const float* sRd;
  __device__ __forceinline__ float4 r4(int a, int c) const {
    if constexpr (TAB < 0) return *reinterpret_cast<const float4*>(sR + a * KP + c);
    else return make_float4(cLev[TAB][a * KP + c], cLev[TAB][a * KP + c + 1], cLev[TAB][a * KP + c + 2],
                            cLev[TAB][a * KP + c + 3]);
  }
  __device__ __forceinline__ float rd(int a) const {
    if constexpr (TAB < 0) return sRd[a]; else return cLev[TAB][KP * KP + a];
  }
};

// Scores of the sampler block's 1024 rows in four 256-row sub-tiles, staged with cp.async into a
// double-buffered shared-memory ring (16 B chunks XOR-swizzled by row, so a thread reading its own
// row is conflict free); with R in the constant bank three CTAs fit an SM.
template <int KP>
__device__ __forceinline__ int lev_swz(int c, int r) {
  constexpr int C = KP / 4, RPL = 8 / (C < 8 ? C : 8);
  return c ^ ((r / RPL) % C);
}

template <int KP, int TAB = -1>
__global__ void __launch_bounds__(FT, TAB >= 0 && KP <= 32 ? 3 : 1) leverage_fused(
    const float* __restrict__ F, int64_t n, int k, const float* __restrict__ Rinv, float* __restrict__ lev, double T,
    uint64_t* __restrict__ bw, uint32_t* __restrict__ bd, double* __restrict__ bt, int64_t s, int64_t cap,
    int64_t* __restrict__ counts, double* __restrict__ mass, unsigned int* counter, int32_t* status) {
  constexpr int C = KP / 4;
  __shared__ __align__(16) float sR[TAB < 0 ? KP * KP : 4];
  __shared__ float sRd[TAB < 0 ? KP : 1];
  __shared__ uint64_t shw[33];
  __shared__ uint32_t shd[33];
  __shared__ double sht[33];
  extern __shared__ __align__(16) unsigned char sml[];
  float* sF = reinterpret_cast<float*>(sml);          // k == KP: [2][256][KP] swizzled; else [256][KP + 4]
  if (dev_failed(status)) return;
  const int tid = threadIdx.x;
  if constexpr (TAB < 0) {
    for (int e = tid; e < KP * KP + KP; e += FT) {   // Rf = [R (KP x KP upper) | 1 / diag(R)]
      if (e < KP * KP) sR[e] = Rinv[e]; else sRd[e - KP * KP] = Rinv[e];
    }
  }
  const int64_t b = blockIdx.x;                       // sampler block: rows [1024 b, 1024 b + 1024)
  uint64_t sw = 0;
  uint32_t sd = 0;
  double stt = 0.0;
  constexpr int NSUB = kSampBlock / FROWS;
  const bool full = k == KP;
  auto issue = [&](int sub) {                         // cp.async of sub-tile `sub` into buffer sub & 1
    const int64_t r0 = b * kSampBlock + sub * FROWS;
    const int rows = (int)max64(0, min64(FROWS, n - r0));
    float* dst = sF + (sub & 1) * FROWS * KP;
    for (int q = tid; q < FROWS * C; q += FT) {
      const int r = q / C, c = q - r * C;
      const bool ok = r < rows;
      cp_async16(dst + r * KP + 4 * lev_swz<KP>(c, r), ok ? F + (r0 + r) * KP + 4 * c : F, ok);
    }
    cp_async_commit();
  };
  if (full) { issue(0); issue(1); }
  for (int sub = 0; sub < NSUB; ++sub) {
    const int64_t r0 = b * kSampBlock + sub * FROWS;
    const int rows = (int)max64(0, min64(FROWS, n - r0));
    const float* cur = sF + (full ? (sub & 1) * FROWS * KP : 0);
    if (full) {
      cp_async_wait<1>();                             // this sub-tile's group has landed
      __syncthreads();
    } else {
      __syncthreads();
      for (int e = tid; e < FROWS * KP; e += FT) {
        const int r = e / KP, c = e - r * KP;
        sF[r * (KP + 4) + c] = (r < rows && c < k) ? F[(r0 + r) * k + c] : 0.f;
      }
      __syncthreads();
    }
    if (tid < rows) {
      float2 f[KP / 2];   // column pairs: the substitution runs on packed FFMA2
#pragma unroll
      for (int a = 0; a < KP; a += 4) {
        const float4 v = full ? *reinterpret_cast<const float4*>(cur + tid * KP + 4 * lev_swz<KP>(a / 4, tid))
                              : *reinterpret_cast<const float4*>(sF + tid * (KP + 4) + a);
        f[a / 2] = make_float2(v.x, v.y); f[a / 2 + 1] = make_float2(v.z, v.w);
      }
      // q = f R^{-1} by forward substitution q R = f (R upper, rd = 1 / diag R), l = ||q||^2.
      // Row a of R is read as float4 groups from the aligned group holding column a: entries
      // c <= a of f are dead once q_a is formed, so updating them too is harmless (R is stored
      // with zeros below the diagonal).
      const LevR<KP, TAB> rsrc{sR, sRd};
      float l = 0.f;
#pragma unroll
      for (int a = 0; a < KP; ++a) {
        const float q = ((a & 1) ? f[a / 2].y : f[a / 2].x) * rsrc.rd(a);
        l = fmaf(q, q, l);
        const float2 nq = make_float2(-q, -q);
#pragma unroll
        for (int c = (a + 1) & ~3; c < KP; c += 4) {
          const float4 r4 = rsrc.r4(a, c);
          f[c / 2] = ffma2(nq, make_float2(r4.x, r4.y), f[c / 2]);
          f[c / 2 + 1] = ffma2(nq, make_float2(r4.z, r4.w), f[c / 2 + 1]);
        }
      }
      lev[r0 + tid] = l;
      const double ld = (double)l;
      const bool det = ld >= T;                                     // reading Z1
      sw += det ? 0ull : (uint64_t)__double2ull_rd(ld * kTwo40f);  // reading Z6
      sd += det ? 1u : 0u;
      stt += det ? ld : 0.0;
    }
    if (full) {
      __syncthreads();                                // buffer sub & 1 free
      if (sub + 2 < NSUB) issue(sub + 2); else cp_async_commit();   // keep one group per step
    }
  }
  sw = block_sum(sw, shw);
  sd = block_sum(sd, shd);
  stt = block_sum(stt, sht);
  if (tid == 0) { bw[b] = sw; bd[b] = sd; bt[b] = stt; }
  if (!arrive_last(counter)) return;
  // S2: exclusive scan of the block sums, totals into the plan
  const int64_t nb = gridDim.x;
  uint64_t cw = 0;
  uint32_t cd = 0;
  double theta = 0.0;
  for (int64_t base = 0; base < nb; base += FT) {
    const int64_t i = base + tid;
    const uint64_t vw = i < nb ? __ldcg(bw + i) : 0ull;
    const uint32_t vd = i < nb ? __ldcg(bd + i) : 0u;
    const double vt = i < nb ? __ldcg(bt + i) : 0.0;
    uint64_t tw; uint32_t td;
    const uint64_t ew = block_excl_scan(vw, shw, &tw);
    const uint32_t ed = block_excl_scan(vd, shd, &td);
    const double st_ = block_sum(vt, sht);
    if (i < nb) { bw[i] = cw + ew; bd[i] = cd + ed; }
    cw += tw; cd += td;
    theta += st_;
  }
  if (tid == 0) {
    const int64_t sD = (int64_t)cd;
    const int64_t sR_ = (cw == 0ull) ? 0 : (s > sD ? s - sD : 0);   // reading Z2
    counts[0] = sD;
    counts[1] = sR_;
    counts[3] = (int64_t)cw;
    mass[0] = theta;
    mass[1] = (double)k - theta;
    if (sD > cap) dev_fail(status, SYMNMF_ERR_CAPACITY);
  }
}

// ---------------------------------------------------------------- uniq_count_fused (S5 + S6 + stats)
__global__ void __launch_bounds__(256) uniq_count_fused(const float* __restrict__ lev, int64_t n, double T,
                                                        const int32_t* __restrict__ cnt, uint32_t* __restrict__ bu,
                                                        int64_t cap, int64_t* __restrict__ counts,
                                                        const double* __restrict__ mass, const int32_t* iter_dev,
                                                        int32_t first_iter, int32_t max_iters, int side,
                                                        symnmf_half_stats* stats, unsigned int* counter,
                                                        int32_t* status) {
  __shared__ uint32_t sh[33];
  if (dev_failed(status)) return;
  const int64_t i0 = (int64_t)blockIdx.x * kSampBlock + threadIdx.x * 4;
  uint32_t c = 0;
  if (i0 + 3 < n) {
    const float4 l4 = *reinterpret_cast<const float4*>(lev + i0);
    const int4 c4 = *reinterpret_cast<const int4*>(cnt + i0);
    c = ((double)l4.x >= T || c4.x > 0) + ((double)l4.y >= T || c4.y > 0) + ((double)l4.z >= T || c4.z > 0) +
        ((double)l4.w >= T || c4.w > 0);
  } else {
    for (int e = 0; e < 4; ++e)
      if (i0 + e < n) c += ((double)lev[i0 + e] >= T || cnt[i0 + e] > 0) ? 1u : 0u;
  }
  c = block_sum(c, sh);
  if (threadIdx.x == 0) bu[blockIdx.x] = c;
  if (!arrive_last(counter)) return;
  const int64_t nb = gridDim.x;
  uint32_t run = 0;
  for (int64_t base = 0; base < nb; base += 256) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < nb ? __ldcg(bu + i) : 0u;
    uint32_t tot;
    const uint32_t e = block_excl_scan(v, sh, &tot);
    if (i < nb) bu[i] = run + e;
    run += tot;
  }
  if (threadIdx.x == 0) {
    counts[2] = (int64_t)run;
    if ((int64_t)run > cap) dev_fail(status, SYMNMF_ERR_CAPACITY);
    if (stats) {
      const int t = *iter_dev - first_iter;
      if (t >= 0 && t < max_iters) {
        symnmf_half_stats h;
        h.s_d = counts[0]; h.s_r = counts[1]; h.n_uniq = (int64_t)run; h.theta = mass[0];
        stats[2 * t + side] = h;
      }
    }
  }
}

// ---------------------------------------------------------------- sampled_gram_fused
template <int KP>
__global__ void __launch_bounds__(FT) sampled_gram_fused(const float* __restrict__ F, int k,
                                                         const int32_t* __restrict__ uniq,
                                                         const double* __restrict__ w,
                                                         const int64_t* __restrict__ n_uniq_dev, double* Gacc,
                                                         double* Gout, unsigned int* counter, int32_t* status) {
  constexpr int ST = KP + 4;
  constexpr int ROWS = 64;
  __shared__ __align__(16) float s[ROWS * ST];
  extern __shared__ double red[];   // 32 KB: row-group reduction of the commit
  __shared__ float sw[ROWS];
  __shared__ int64_t srow[ROWS];
  if (dev_failed(status)) return;
  const int64_t nu = *n_uniq_dev;
  GramThread gt;
  gt.init(threadIdx.x, FT, (k + 3) / 4);
  for (int64_t r0 = (int64_t)blockIdx.x * ROWS; r0 < nu; r0 += (int64_t)gridDim.x * ROWS) {
    const int rows = (int)min64(ROWS, nu - r0);
    __syncthreads();
    if (threadIdx.x < ROWS) {
      const bool ok = threadIdx.x < rows;
      srow[threadIdx.x] = ok ? (int64_t)uniq[r0 + threadIdx.x] : 0;
      sw[threadIdx.x] = ok ? (float)w[r0 + threadIdx.x] : 0.f;
    }
    __syncthreads();
    if (k == KP) {       // gathered rows: one float4 per (row, 4 columns), all loads in flight
      constexpr int NV = ROWS * KP / 4, Q = (NV + FT - 1) / FT;
      float4 v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = threadIdx.x + q * FT, r = e / (KP / 4), c = e - r * (KP / 4);
        v[q] = (e < NV && r < rows) ? __ldg(reinterpret_cast<const float4*>(F + srow[r] * k) + c)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = threadIdx.x + q * FT, r = e / (KP / 4), c = e - r * (KP / 4);
        if (e < NV) *reinterpret_cast<float4*>(s + r * ST + 4 * c) = v[q];
      }
    } else {
      for (int e = threadIdx.x; e < ROWS * KP; e += FT) {
        const int r = e / KP, c = e - r * KP;
        s[r * ST + c] = (r < rows && c < k) ? __ldg(F + srow[r] * k + c) : 0.f;
      }
    }
    __syncthreads();
    gt.accumulate(s, ST, rows, sw);
  }
  gt.commit(Gacc, k, red);
  if (arrive_last(counter)) finalize_gram<KP>(Gacc, Gout, k, nullptr, nullptr, nullptr, status);
}

// ---------------------------------------------------------------- launchers
static int fused_grid(int64_t tiles, int per_sm) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 148 * per_sm));
}

template <int KP>
static void gram_fused_t(const float* F, int64_t n, int k, double* Gacc, double* Gout, float* Rinv32,
                         unsigned int* counter, int32_t* status, cudaStream_t st) {
  const size_t smem = std::max({sizeof(float) * FROWS * (KP + 4), sizeof(double) * 2 * k * (k + 1), kRedBytes});
  cudaFuncSetAttribute(gram_fused<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gram_fused<KP><<<fused_grid((n + FROWS - 1) / FROWS, 2), FT, smem, st>>>(F, n, k, Gacc, Gout, Rinv32, counter,
                                                                            status);
}

void launch_gram_fused(const float* F, int64_t n, int k, double* Gacc, double* Gout, float* Rinv32,
                       unsigned int* counter, int32_t* status, cudaStream_t st) {
  switch (kpad(k)) {
    case 8: gram_fused_t<8>(F, n, k, Gacc, Gout, Rinv32, counter, status, st); break;
    case 16: gram_fused_t<16>(F, n, k, Gacc, Gout, Rinv32, counter, status, st); break;
    case 32: gram_fused_t<32>(F, n, k, Gacc, Gout, Rinv32, counter, status, st); break;
    default: gram_fused_t<64>(F, n, k, Gacc, Gout, Rinv32, counter, status, st); break;
  }
}

template <int KP>
static void sweep_fused_t(const double* G, double alpha, float* Y, const float* F, float* X, int64_t n, int k,
                          bool zeroY, double* Gacc, double* Gout, float* Rinv32, unsigned int* counter,
                          int32_t* status, cudaStream_t st) {
  const size_t smem = std::max({sizeof(float) * 2 * FROWS * (KP + 4), sizeof(double) * 2 * k * (k + 1), kRedBytes});
  cudaFuncSetAttribute(sweep_fused<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  sweep_fused<KP><<<fused_grid((n + FROWS - 1) / FROWS, KP <= 32 ? 2 : 1), FT, smem, st>>>(
      G, alpha, Y, F, X, n, k, zeroY ? 1 : 0, Gacc, Gout, Rinv32, counter, status);
}

void launch_sweep_fused(const double* G, double alpha, float* Y, const float* F, float* X, int64_t n, int k,
                        bool zeroY, double* Gacc, double* Gout, float* Rinv32, unsigned int* counter,
                        int32_t* status, cudaStream_t st) {
  switch (kpad(k)) {
    case 8: sweep_fused_t<8>(G, alpha, Y, F, X, n, k, zeroY, Gacc, Gout, Rinv32, counter, status, st); break;
    case 16: sweep_fused_t<16>(G, alpha, Y, F, X, n, k, zeroY, Gacc, Gout, Rinv32, counter, status, st); break;
    case 32: sweep_fused_t<32>(G, alpha, Y, F, X, n, k, zeroY, Gacc, Gout, Rinv32, counter, status, st); break;
    default: sweep_fused_t<64>(G, alpha, Y, F, X, n, k, zeroY, Gacc, Gout, Rinv32, counter, status, st); break;
  }
}

template <int KP, int TAB>
static void leverage_fused_t(const float* F, int64_t n, int k, const float* Rinv, float* lev, double T,
                             const SamplerWs& w, int64_t s, const symnmf_plan& plan, unsigned int* counter,
                             int32_t* status, cudaStream_t st) {
  const size_t smem = k == KP ? sizeof(float) * 2 * FROWS * KP : sizeof(float) * FROWS * (KP + 4);
  cudaFuncSetAttribute(leverage_fused<KP, TAB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  leverage_fused<KP, TAB><<<(unsigned)samp_blocks(n), FT, smem, st>>>(F, n, k, Rinv, lev, T, w.bw, w.bd, w.bt, s,
                                                                      plan.cap, plan.counts, plan.mass, counter,
                                                                      status);
}

template <int KP>
static void leverage_tab_dispatch(int tab, const float* F, int64_t n, int k, const float* Rinv, float* lev, double T,
                                  const SamplerWs& w, int64_t s, const symnmf_plan& plan, unsigned int* counter,
                                  int32_t* status, cudaStream_t st) {
#define LV_CASE(T_) case T_: leverage_fused_t<KP, T_>(F, n, k, Rinv, lev, T, w, s, plan, counter, status, st); break;
  switch (tab) {
    LV_CASE(0) LV_CASE(1) LV_CASE(2) LV_CASE(3) LV_CASE(4) LV_CASE(5) LV_CASE(6) LV_CASE(7)
    default: leverage_fused_t<KP, -1>(F, n, k, Rinv, lev, T, w, s, plan, counter, status, st); break;
  }
#undef LV_CASE
}

// tab >= 0 (k == kpad(k) <= 32): R copied from Rinv to constant table tab first.
void launch_leverage_fused(const float* F, int64_t n, int k, const float* Rinv, float* lev, double T,
                           const SamplerWs& w, int64_t s, const symnmf_plan& plan, unsigned int* counter,
                           int32_t* status, cudaStream_t st, int tab) {
  const int kp = kpad(k);
  if (tab >= 0 && kp == k && kp <= 32) {
    cudaMemcpyToSymbolAsync(cLev, Rinv, sizeof(float) * (kp * kp + kp), sizeof(float) * kLevTab * tab,
                            cudaMemcpyDeviceToDevice, st);
  } else {
    tab = -1;
  }
  switch (kp) {
    case 8: leverage_tab_dispatch<8>(tab, F, n, k, Rinv, lev, T, w, s, plan, counter, status, st); break;
    case 16: leverage_tab_dispatch<16>(tab, F, n, k, Rinv, lev, T, w, s, plan, counter, status, st); break;
    case 32: leverage_tab_dispatch<32>(tab, F, n, k, Rinv, lev, T, w, s, plan, counter, status, st); break;
    default: leverage_fused_t<64, -1>(F, n, k, Rinv, lev, T, w, s, plan, counter, status, st); break;
  }
}

void launch_uniq_count_fused(const float* lev, int64_t n, double T, const SamplerWs& w, const symnmf_plan& plan,
                             const int32_t* iter_dev, int32_t first_iter, int32_t max_iters, int side,
                             symnmf_half_stats* stats, unsigned int* counter, int32_t* status, cudaStream_t st) {
  launch_pdl(uniq_count_fused, (unsigned)samp_blocks(n), 256, 0, st, lev, n, T, w.cnt, w.bu, plan.cap, plan.counts,
                                                             plan.mass, iter_dev, first_iter, max_iters, side, stats,
                                                             counter, status);
}

void launch_sampled_gram_fused(const float* F, int k, const symnmf_plan& plan, double* Gacc, double* Gout,
                               unsigned int* counter, int32_t* status, cudaStream_t st) {
  const int grid = fused_grid((plan.cap + 63) / 64, 1);
  switch (kpad(k)) {
    case 8: launch_pdl(sampled_gram_fused<8>, grid, FT, kRedBytes, st, F, k, plan.uniq_idx, plan.uniq_w, plan.counts + 2, Gacc, Gout, counter, status); break;
    case 16: launch_pdl(sampled_gram_fused<16>, grid, FT, kRedBytes, st, F, k, plan.uniq_idx, plan.uniq_w, plan.counts + 2, Gacc, Gout, counter, status); break;
    case 32: launch_pdl(sampled_gram_fused<32>, grid, FT, kRedBytes, st, F, k, plan.uniq_idx, plan.uniq_w, plan.counts + 2, Gacc, Gout, counter, status); break;
    default: launch_pdl(sampled_gram_fused<64>, grid, FT, kRedBytes, st, F, k, plan.uniq_idx, plan.uniq_w, plan.counts + 2, Gacc, Gout, counter, status); break;
  }
}

}  // namespace symnmf
